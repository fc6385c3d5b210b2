"""ncu raw-page CSV (exported on the box: ncu -i X --page raw --csv) ->
profiles/*.json with the metrics DESIGN.md quotes, per launch.

    python tools/ncu_to_json.py raw.csv --bytes B1,B2 --command "..." --out profiles/x.json
"""
import argparse
import csv
import json

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
         "byte": 1, "nsecond": 1, "ns": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--bytes", default="", help="comma list: algorithmic bytes per launch, in launch order")
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.raw)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, data = rows[start], rows[start + 1], rows[start + 2:]
    algo = [float(x) for x in a.bytes.split(",") if x]
    out = []
    for i, r in enumerate(data):
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:160]}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                u = units[hdr.index(k)]
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                e[k] = v * SCALE.get(u, 1)
        if i < len(algo):
            e["algorithmic_bytes"] = algo[i]
            e["dram_over_algorithmic"] = round(
                (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / algo[i], 4)
        out.append(e)
    json.dump({"command": a.command, "note": a.note, "units": "bytes, ns", "launches": out},
              open(a.out, "w"), indent=1)
    for e in out:
        print(json.dumps(e))


if __name__ == "__main__":
    main()
