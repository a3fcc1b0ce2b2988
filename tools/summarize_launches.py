"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
per kernel name: total time, share, launches, mean time, DRAM GB/s.
Usage: python tools/summarize_launches.py launches.csv [top_n]"""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[ui]
        if unit in ("usecond",):
            v *= 1e3
        elif unit in ("msecond",):
            v *= 1e6
        elif unit in ("Kbyte",):
            v *= 1e3
        elif unit in ("Mbyte",):
            v *= 1e6
        elif unit in ("Gbyte",):
            v *= 1e9
        per[r[idi]][r[mi]] = v
        names[r[idi]] = r[ki]
    agg = defaultdict(lambda: [0.0, 0, 0.0])
    total = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i][:90]]
        a[0] += t
        a[1] += 1
        a[2] += b
        total += t
    print(f"# {path}: total kernel time {total / 1e6:.2f} ms over {len(per)} launches (ncu: serialised, cold caches)")
    for name, (t, n, b) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        gbs = b / t if t else 0.0
        print(f"{t / 1e3:10.1f} us {100 * t / total:5.1f}%  n={n:5d}  mean {t / n / 1e3:8.1f} us  {gbs:7.0f} GB/s  {name}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
