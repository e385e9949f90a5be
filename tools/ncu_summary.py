#!/usr/bin/env python3
"""Summarise ncu reports into profiles/ (tracked).

  tools/ncu_summary.py OUT.json --launches launches.csv rep1.ncu-rep [rep2 ...]

For every --set full report: per-kernel duration, DRAM bytes (read/write),
tensor-pipe and DRAM utilisation, registers, grid, occupancy limiters.  For the
launch list (--metrics gpu__time_duration.sum): per-kernel count, total, mean
and share of the captured step.
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": "tc_inst_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_xu.sum": "xu_inst",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_sectors_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_throughput_pct",
    "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed": "sm_memory_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def short(name):
    n = name.replace("<unnamed>::", "").split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    return n.replace("unnamed>::", "").replace("fsvd::", "").strip()


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        k = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                k[key] = v * SCALE.get(units[i], 1)
        k["duration_us"] = k.pop("duration", None)
        out[k["kernel"]] = k
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5 and not r[0].startswith("==")]
    hdr, data = rows[0], rows[1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1)
        agg[short(r[ik])][0] += 1
        agg[short(r[ik])][1] += v
    tot = sum(t for _, t in agg.values())
    return {k: {"count": n, "total_us": round(t, 2), "mean_us": round(t / n, 2),
                "share": round(t / tot, 4)} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}


def main():
    if len(sys.argv) < 2 or sys.argv[1] in ("-h", "--help"):
        print(__doc__)
        sys.exit(0 if len(sys.argv) >= 2 else 2)
    out = sys.argv[1]
    args = sys.argv[2:]
    res = {"kernels": {}, "launch_list": None}
    if args and args[0] == "--launches":
        res["launch_list"] = launches(args[1])
        args = args[2:]
    for p in args:
        res["kernels"].update(full_report(p))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
