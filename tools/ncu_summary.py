"""Summarise an ncu report (``ncu -i X --page raw --csv``) into the markdown
table kept under profiles/.   python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "blocks/SM limit (regs)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    stall = [i for i, c in enumerate(h) if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        print(f"### `{name}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {label} | {r[i]} {units[i]} |")
        st = sorted(((float(r[i].replace(",", "") or 0), h[i]) for i in stall), reverse=True)[:4]
        s = ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}" for v, n in st)
        print(f"| top stalls (warps per issue) | {s} |\n")


if __name__ == "__main__":
    main(sys.argv[1])
