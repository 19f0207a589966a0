"""Per-kernel-family share of one training step from an `ncu --metrics gpu__time_duration.sum` launch list."""
import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/train_launches.csv"
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
fam = collections.Counter()
n = collections.Counter()
for r in rows[1:]:
    name = r[ki]
    v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(r[ui], 1.0)
    key = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0]
    fam[key] += v
    n[key] += 1
tot = sum(fam.values())
print(f"total {tot/1e3:.2f} ms over {sum(n.values())} launches (ncu, serialised, cold caches)")
for k, v in fam.most_common(20):
    print(f"{k:40s} {v/1e3:9.3f} ms  {100*v/tot:5.1f}%  launches {n[k]}")
