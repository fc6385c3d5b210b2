"""Summarize an ncu report for profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py gpurun_out/prof.ncu-rep --bytes B --out profiles/x.json

Pulls the per-launch DRAM bytes, duration, throughput and occupancy metrics
of each profiled kernel; --bytes gives the algorithmic bytes per launch so
the JSON records traffic / algorithmic."""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__t_bytes.sum": "l2_bytes",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--bytes", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            if k in d:
                u = units[hdr.index(k)]
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if u == "Kbyte":
                    v *= 1e3
                elif u == "Mbyte":
                    v *= 1e6
                elif u == "Gbyte":
                    v *= 1e9
                elif u in ("usecond", "us"):
                    v *= 1e3
                elif u == "msecond":
                    v *= 1e6
                e[name] = v
        if "dram_read" in e:
            e["dram_bytes_per_launch"] = e["dram_read"] + e.get("dram_write", 0.0)
            if args.bytes:
                e["algorithmic_bytes"] = args.bytes
                e["traffic_over_algorithmic"] = e["dram_bytes_per_launch"] / args.bytes
        out.append(e)
    with open(args.out, "w") as f:
        json.dump({"report": args.rep, "launches": out, "units": "bytes, ns"}, f, indent=1)
    for e in out:
        print(json.dumps(e))


if __name__ == "__main__":
    main()
