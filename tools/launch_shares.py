"""Per-kernel launch counts, total/mean device time and share of the step
from an ncu launch list (ncu --metrics gpu__time_duration.sum --csv
--log-file X).  ncu serialises launches and flushes caches, so absolute
times are cold-cache; the SHARES are what to compare with bench.py.

    python tools/launch_shares.py gpurun_out/launches.csv --header "..." --out profiles/x.txt"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--header", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--exclude", default="distribution_elementwise,vectorized_elementwise,fill,copy,unrolled")
    ap.add_argument("--include", default="gemv,build_lut,pipeline_kernel",
                    help="comma list: keep only kernels whose name contains one of these")
    args = ap.parse_args()
    rows = [r for r in csv.reader(open(args.csv)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    excl = [e for e in args.exclude.split(",") if e]
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        if any(e in name for e in excl):
            continue
        if args.include and not any(i in name for i in args.include.split(",")):
            continue
        v = float(r[vi].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    lines = [l for l in args.header.split("\\n") if l]
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{name[:60]:60s} launches {cnt[name]:5d}  total {t / 1e3:10.1f} us  "
                     f"mean {t / cnt[name] / 1e3:7.2f} us  share {100 * t / allt:5.1f}%")
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
