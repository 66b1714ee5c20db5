"""Summaries of ncu outputs for profiles/ (run in the dev container).

  python scripts/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
  python scripts/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/rNN_<kernel>.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    unit = None
    for r in data:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[ui]
        agg[r[ki]].append(v)
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none\n")
    print("Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n")
    print("| launches | avg us | share | kernel |\n|---:|---:|---:|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {len(v)} | {sum(v) / len(v) * scale:.1f} | {100 * sum(v) / tot:.1f}% | `{k[:110]}` |")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
           "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_wait",
           "smsp__pcsamp_warps_issue_stalled_lg_throttle",
           "smsp__pcsamp_warps_issue_stalled_mio_throttle",
           "smsp__pcsamp_warps_issue_stalled_membar",
           "smsp__pcsamp_warps_issue_stalled_sleeping",
           "smsp__pcsamp_warps_issue_stalled_selected"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name") if "Kernel Name" in h else None
    print(f"# ncu --set full summary ({path})\n")
    for j, r in enumerate(data):
        print(f"## launch {j}: `{r[name_i][:100] if name_i is not None else ''}`\n")
        print("| metric | value | unit |\n|---|---:|---|")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                print(f"| {m} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
