"""Summarise the ncu evidence of one bench profile run into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_materialize.ncu-rep \
        gpurun_out/launches_bench.csv profiles/materialize_ncu_summary.json

Reads the `--set full` capture of fdy_materialize_kernel (ncu -i ... --page raw)
and the launch list of the same bench command, and writes the per-launch
DRAM traffic bench.py reports as roofline.traffic, next to the kernel's
share of the step from the launch list.
"""
from __future__ import annotations

import csv
import io
import json
import statistics
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_per_cta_bytes",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def unit_scale(unit: str) -> float:
    unit = unit.split("/")[0]
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
            "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
            "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(unit, 1)


def raw_page(rep: str, kernel: str = "fdy_materialize_kernel") -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for row in rows[2:]:
        if kernel not in ",".join(row):
            continue
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    res[key] = float(row[i].replace(",", "")) * unit_scale(units[i])
                except ValueError:
                    pass
        break
    return res


def launch_list(path: str) -> dict:
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    per = defaultdict(dict)
    for r in rows:
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    by_kernel = defaultdict(list)
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("<unnamed>::", "")
        by_kernel[short].append(m)
    return {k: {"launches": len(v),
                "mean_ns": statistics.mean(x.get("gpu__time_duration.sum", 0.0) for x in v),
                "mean_dram_bytes": statistics.mean(x.get("dram__bytes_read.sum", 0.0)
                                                   + x.get("dram__bytes_write.sum", 0.0) for x in v)}
            for k, v in by_kernel.items()}


def main() -> None:
    rep, launches, out = sys.argv[1:4]
    kernel = sys.argv[4] if len(sys.argv) > 4 else "fdy_materialize_kernel"
    full = raw_page(rep, kernel)
    ll = launch_list(launches)
    mat = ll.get("fdy_materialize_kernel", {}).get("mean_ns", 0.0)
    rel = ll.get("fdy_relocate_templates_kernel", {}).get("mean_ns", 0.0)
    summary = {
        "kernel": kernel,
        "command": "python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline --skip-tier-s (tools/gpu_profile_bench.sh)",
        "source": {"full_set": rep, "launch_list": launches},
        **{k: v for k, v in full.items()},
        # one fdy_materialize launch = the template relocation grid (delta != 0,
        # launch-list bytes) + the member grid (full-set bytes)
        "dram_bytes_per_launch": full.get("dram_bytes_read", 0) + full.get("dram_bytes_write", 0)
        + ll.get("fdy_relocate_templates_kernel", {}).get("mean_dram_bytes", 0.0),
        "note": "ncu replays with a cache flush; DRAM writes below the 147 MB of member images "
                "are lines still dirty in the 126 MB L2 when the kernel ends",
        "launch_list_mean_ns": ll,
        "materialize_share_of_launch": mat / (mat + rel) if mat + rel else None,
    }
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
