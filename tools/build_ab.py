"""Builds A/B variants of the product library for same-box comparisons:
gemv_batch.cu recompiled with extra defines (e.g. the per-tile duty
assignment, BITLUT_SUM_WARP) and linked with the
product objects into _ab/libbitlut_ab_<name>.so.  Select a variant with
BITLUT_B200_LIB (tools/batch_ab.py, tools/batch_groups.py).

    python tools/build_ab.py "s0:-DBITLUT_SUM_WARP=0" "s2:-DBITLUT_SUM_WARP=2"
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_00088_b200 import build as B  # noqa: E402

B.build_lib()
objdir = os.path.join(B.PKG, "_lib", "obj")
outdir = os.path.join(ROOT, "_ab")
os.makedirs(outdir, exist_ok=True)
flags = [f for f in B.NVCC_FLAGS if f not in ("-shared", "-Xptxas", "-v")]
VARIANT_TUS = ["gemv_batch.cu"]
for n in sys.argv[1:]:
    # n = "<name>" or "<name>:-DX=1,-DY=2" (extra defines for the variant TUs)
    extra = []
    if ":" in n:
        n, defs = n.split(":", 1)
        extra = defs.split(",")
    objs = []
    for src in B.SOURCES:
        if src in VARIANT_TUS:
            o = os.path.join(outdir, f"{src[:-3]}_ab{n}.o")
            subprocess.run([B.nvcc(), *flags, *(extra or [f"-DBITLUT_AB={n}"]), "-c", "-o", o,
                            os.path.join(B.PKG, "csrc", src)], check=True)
            objs.append(o)
        else:
            objs.append(os.path.join(objdir, src.replace(".cu", ".o")))
    out = os.path.join(outdir, f"libbitlut_ab_{n}.so")
    subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs], check=True)
    print(out)
