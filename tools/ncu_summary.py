"""Summarise ncu --set full captures (.ncu-rep) into one line of key metrics per kernel."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "smem_tensor%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64cyc%"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__cycles_active.avg", "cyc_active"),
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data"
    h, u = rows[0], rows[1]
    lines = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        units = dict(zip(h, u))
        name = d.get("Kernel Name", "?").split("(")[0]
        parts = [name]
        for k, lab in KEYS:
            if k in d and d[k] != "":
                parts.append(f"{lab}={d[k]}{units.get(k, '')}")
        lines.append("  ".join(parts))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
