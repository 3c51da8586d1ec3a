"""Per-launch DRAM and PCIe traffic of the dominant kernels from committed ncu captures, for bench.py's
roofline.traffic field:  python tools/ncu_traffic.py gather=gpurun_out/prof_gather.ncu-rep \
    attn=gpurun_out/prof_attn_M7.ncu-rep > profiles/ncu_traffic.json"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
        "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, row = rows[0], rows[1], rows[2]
    get = lambda k: float(row[hdr.index(k)].replace(",", "")) * UNIT.get(units[hdr.index(k)], 1)  # noqa: E731
    dur = get("gpu__time_duration.sum")
    return {"kernel": row[hdr.index("Kernel Name")][:80], "duration_s": dur,
            "dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
            "pcie_read_bytes": get("pcie__read_bytes.sum.per_second") * dur,
            "pcie_write_bytes": get("pcie__write_bytes.sum.per_second") * dur, "source": rep.split("/")[-1]}


if __name__ == "__main__":
    print(json.dumps({k: metrics(v) for k, v in (a.split("=", 1) for a in sys.argv[1:])}, indent=1))
