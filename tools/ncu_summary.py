"""Summarise ncu captures for profiles/ (run here, on the CPU box, on reports brought back by gpurun).

    python tools/ncu_summary.py gpurun_out/prof_gather.ncu-rep [...] > profiles/r01_ncu_summary.md
    python tools/ncu_summary.py --launches gpurun_out/launches_L8.csv >> profiles/r01_ncu_summary.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("pcie__read_bytes.sum.per_second", "PCIe read bytes/s (link, incl. protocol)"),
    ("pcie__write_bytes.sum.per_second", "PCIe write bytes/s"),
    ("syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum", "sysmem read sectors (32 B)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (avg SM, elapsed)"),
    ("sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed", "tensor pipe % (busiest SM)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def summarise(rep):
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"\n### `{rep.split('/')[-1]}`\n")
    for row in data:
        name = row[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
        print(f"**{name[:110]}**\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in idx:
                print(f"| {label} (`{k}`) | {row[idx[k]]} | {units[idx[k]]} |")
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(row[i].replace(",", "")), h))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            print("\ntop warp stall reasons (cycles per issued instruction): " +
                  ", ".join(f"{h.split('stalled_')[1].split('.')[0]} {v:.2f}" for v, h in stalls[:6]))
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = defaultdict(list)
    unit = ""
    for r in rows[start + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    tot = sum(sum(v) for v in d.values())
    print(f"\n### launch list `{path.split('/')[-1]}` (ncu --metrics gpu__time_duration.sum, serialised, cold)\n")
    print(f"| kernel | launches | mean ({unit}) | share of summed time |\n|---|---|---|---|")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k[-70:]}` | {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            launches(p)
    else:
        for p in args:
            summarise(p)
