"""Summarise an ncu launch list (``ncu --metrics gpu__time_duration.sum --csv
--log-file X``) into the markdown table kept under profiles/.
    python tools/launch_table.py launches.csv[.xz]"""
import collections
import csv
import lzma
import statistics
import sys


def main(path):
    rows = list(csv.reader(lzma.open(path, "rt") if path.endswith(".xz") else open(path)))
    i = 0
    while not rows[i] or rows[i][0] != "ID":
        i += 1
    h = rows[i]
    k_name, k_metric, k_value = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    us = collections.defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > k_value and r[k_metric] == "gpu__time_duration.sum":
            us[r[k_name].split("(")[0].replace("void ", "")].append(float(r[k_value].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in us.values())
    print("| kernel | launches | working (>5 us) | total ms | median us (working) | share |")
    print("|---|---|---|---|---|---|")
    for name, v in sorted(us.items(), key=lambda kv: -sum(kv[1])):
        if sum(v) / total < 0.001:
            continue
        w = [x for x in v if x > 5]
        med = statistics.median(w) if w else 0.0
        print(f"| `{name}` | {len(v)} | {len(w)} | {sum(v) / 1e3:.2f} | {med:.1f} | {sum(v) / total * 100:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
