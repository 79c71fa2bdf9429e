"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
totals and shares.  python tools/launch_share.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[i], rows[i + 1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "second": 1e3, "s": 1e3}
tot, cnt = collections.Counter(), collections.Counter()
for r in data:
    name = r[ik].split("(")[0].replace("void ", "")
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':62s} {'launches':>8s} {'total ms':>9s} {'avg us':>9s} {'share':>6s}")
for k, v in tot.most_common():
    print(f"{k[:62]:62s} {cnt[k]:8d} {v:9.3f} {v / cnt[k] * 1e3:9.1f} {v / T * 100:5.1f}%")
print(f"{'TOTAL':62s} {sum(cnt.values()):8d} {T:9.3f}")
