"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel shares: python tools/launch_summary.py launches.csv [header lines]."""
import collections
import csv
import re
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ik, ig, iv, iu = (hdr.index("Kernel Name"), hdr.index("Grid Size") if "Grid Size" in hdr else None,
                  hdr.index("Metric Value"), hdr.index("Metric Unit"))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iv or not r[iv]:
        continue
    v = float(r[iv].replace(",", ""))
    us = v / 1e3 if r[iu] == "ns" else (v * 1e3 if r[iu] == "ms" else v)
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
    name = re.sub(r"<([^>]*)>", lambda m: "<" + m.group(1).replace("__nv_bfloat16", "bf16") + ">", name)
    if ig is not None and "tc_gemm" in name:
        name += " grid" + r[ig]
    agg[name][0] += 1
    agg[name][1] += us
total = sum(t for _, t in agg.values())
for h in sys.argv[2:]:
    print("# " + h)
print(f"# launches {sum(n for n, _ in agg.values())}, summed device time {total / 1e3:.2f} ms")
print("share  launches  avg_us  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{100 * t / total:5.1f}%  {n:7d}  {t / n:7.2f}  {k}")
