"""Summarise an ncu report (.ncu-rep) into a short text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 12] > profiles/rNN_name.txt
    [--traffic-json profiles/ncu_traffic.json --workload W --key decode_attention --match decode_attn]

--traffic-json records dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the
launches whose name contains --match) for bench.py's roofline `traffic` field.

Per kernel: duration, DRAM bytes read/written (traffic), DRAM / L2 / SM / tensor-pipe utilisation,
registers, achieved occupancy; then the hottest SASS lines by warp-stall samples.
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "hmma_inst_%"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--traffic-json")
    ap.add_argument("--workload")
    ap.add_argument("--key")
    ap.add_argument("--match")
    a = ap.parse_args()
    raw = list(csv.reader(io.StringIO(ncu(["-i", a.report, "--page", "raw", "--csv", "--print-units", "base"]))))
    hdr, units = raw[0], raw[1]
    name_i = hdr.index("Kernel Name")
    print(f"# ncu summary of {a.report}")
    for row in raw[2:]:
        print(f"\n## kernel: {row[name_i][:140]}")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {label:16s} {row[i]:>14s} {units[i]}")
    if a.traffic_json:
        rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        vals = [float(r[rd].replace(",", "")) + float(r[wr].replace(",", "")) for r in raw[2:] if a.match in r[name_i]]
        assert vals, f"no launch matching {a.match}"
        db = json.load(open(a.traffic_json)) if os.path.exists(a.traffic_json) else {}
        db.setdefault(a.workload, {})[a.key] = {"dram_bytes_per_launch": round(sum(vals) / len(vals)),
                                                "launches": len(vals), "source": os.path.basename(a.report)}
        json.dump(db, open(a.traffic_json, "w"), indent=1)
    src = ncu(["-i", a.report, "--page", "source", "--csv", "--print-source", "sass"])
    blocks, cur = [], None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    for b in blocks:
        rows = b["rows"]
        if len(rows) < 2:
            continue
        h = rows[0]
        try:
            si, ti = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        except ValueError:
            continue
        data = [r for r in rows[1:] if len(r) > si and r[si]]
        tot = sum(float(r[si]) for r in data) or 1.0
        print(f"\n## hottest SASS (warp-stall samples) — {b['name'][:100]}")
        for r in sorted(data, key=lambda r: -float(r[si]))[:a.top]:
            print(f"  {100 * float(r[si]) / tot:5.1f}%  {r[ti][:110]}")


if __name__ == "__main__":
    main()
