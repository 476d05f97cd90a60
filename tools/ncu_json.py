"""Per-launch DRAM traffic and headline metrics of one ncu --set full capture
as the JSON bench.py reads (profiles/<tag>_epoch_kernel_cfg<N>.json).

    python tools/ncu_json.py report.ncu-rep "source description" > out.json
"""
import csv
import json
import subprocess
import sys

rep, source = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
m = {n: [val, unit] for n, unit, val in zip(h, u, v) if n in want}
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def num(key, table):
    val, unit = m[key]
    return float(val.replace(",", "")) * table[unit]


rd = num("dram__bytes_read.sum", scale)
wr = num("dram__bytes_write.sum", scale)
kernel = [r for r in rows[2:3]][0][h.index("Kernel Name")] if "Kernel Name" in h else "epoch_kernel"
print(json.dumps({
    "source": source,
    "kernel": kernel,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "traffic_bytes_per_launch": rd + wr,
    "duration_ms_under_ncu": num("gpu__time_duration.sum", tscale),
    "metrics": m,
}, indent=1))
