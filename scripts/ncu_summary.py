"""Summarise ncu reports (.ncu-rep) and a launch list (.csv) into profiles/<tag>_ncu_summary.json.

    python scripts/ncu_summary.py <tag> gpurun_out/<tag>_gemm.ncu-rep gpurun_out/<tag>_stream.ncu-rep \
        [--launches gpurun_out/<tag>_launches.csv]

Per captured kernel: duration, DRAM bytes, throughputs, tensor-pipe activity, registers, shared
bank conflicts and the top issue-stall reasons (share of PC samples). With --launches, the
launch list's per-kernel-family share of device time over the captured steps.
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, body = rows[0], rows[2:]  # rows[1] = units
    return [dict(zip(header, r)) for r in body]


def summarise(rep: str):
    res = []
    for r in raw_rows(rep):
        d = {"Kernel Name": r.get("Kernel Name", "")[:160]}
        for m in METRICS:
            if m in r:
                d[m] = r[m]
        stalls = {k[len(STALL):]: float(v.replace(",", "")) for k, v in r.items()
                  if k.startswith(STALL) and not k.endswith("_not_issued") and v}
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in
                               sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        d["report"] = Path(rep).name
        res.append(d)
    return res


def family(name: str) -> str:
    for key in ("slice_gemm_tc2", "k_stream<0", "k_stream<1", "k_stream<2", "k_stream<3",
                "k_sum_partials", "k_token"):
        if key in name:
            return key
    return name[:60]


def launch_shares(path: str):
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    t = defaultdict(float)
    n = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        f = family(r["Kernel Name"])
        t[f] += float(r["Metric Value"].replace(",", ""))
        n[f] += 1
    tot = sum(t.values()) or 1.0
    return {f: {"launches": n[f], "total_ns": t[f], "share": round(t[f] / tot, 4)}
            for f in sorted(t, key=lambda k: -t[k])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--launches")
    args = ap.parse_args()
    out = {"kernels": [k for rep in args.reports for k in summarise(rep)]}
    if args.launches:
        out["launch_shares"] = launch_shares(args.launches)
    dst = Path(__file__).resolve().parent.parent / "profiles" / f"{args.tag}_ncu_summary.json"
    dst.write_text(json.dumps(out, indent=1))
    print(dst)


if __name__ == "__main__":
    main()
