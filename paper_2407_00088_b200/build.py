"""In-tree build of the CUDA library (nvcc, sm_100a) and the C oracle.

    python -m paper_2407_00088_b200.build

Outputs: paper_2407_00088_b200/_lib/libbitlut_b200.so (product) and, via
oracle/Makefile, oracle/_build/liboracle.so (test-only checker).  Built
files are git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SOURCES = ["weight_prep.cu", "lut.cu", "gemv.cu", "gemv_b1.cu", "gemv_batch.cu", "pipeline.cu", "host_api.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def lib_path(checks: bool = False) -> str:
    return os.path.join(PKG, "_lib", "libbitlut_b200_checks.so" if checks else "libbitlut_b200.so")


def needs_build(checks: bool = False) -> bool:
    out = lib_path(checks)
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(PKG, "csrc", f) for f in os.listdir(os.path.join(PKG, "csrc"))]
    deps.append(os.path.join(ROOT, "include", "bitlut_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """nvcc each translation unit (in parallel), then link the shared library.
    checks=True builds the diagnostic libbitlut_b200_checks.so with the
    device-side bounds checks (BL_CHECK, common.cuh) compiled in; select it
    with BITLUT_B200_LIB."""
    from concurrent.futures import ThreadPoolExecutor
    out = lib_path(checks)
    if not force and not needs_build(checks):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objdir = os.path.join(os.path.dirname(out), "obj_checks" if checks else "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DBITLUT_CHECKS=1"] if checks else [])

    csrc = os.path.join(PKG, "csrc")
    headers = [os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "bitlut_b200.h"))
    newest_header = max(os.path.getmtime(h) for h in headers)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        srcp = os.path.join(csrc, src)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(srcp), newest_header)):
            return obj, None                       # up to date (incremental rebuild)
        cmd = [nvcc(), *flags, "-c", "-o", obj, srcp]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for obj, res in results:
        if res is None:
            continue
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(obj)}")
        if verbose:
            sys.stderr.write(res.stderr)
    tmp = out + ".tmp"
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp]
                         + [o for o, _ in results], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed linking {os.path.basename(out)}")
    os.replace(tmp, out)
    return out


def build_oracle() -> None:
    mk = os.path.join(ROOT, "oracle", "Makefile")
    if os.path.exists(mk):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


if __name__ == "__main__":
    print(build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv, checks="--checks" in sys.argv))
    build_oracle()
