"""Summarise an ncu launch list of `bench.py` (per kernel family: launches, total
and mean duration, share of the listed time, DRAM bytes) into JSON."""
import collections, csv, json, sys

path, out = sys.argv[1], sys.argv[2]
rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
lau = collections.OrderedDict()
for r in rows:
    lau.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = \
        float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
fam = collections.defaultdict(list)
for (_, name), m in lau.items():
    f = "ff_chain_pair_kernel" if "ff_chain_pair" in name else ("ff_chain_kernel" if "ff_chain_kernel" in name else name[:60])
    fam[f].append(m)
tot = sum(m.get("gpu__time_duration.sum", 0) for ms in fam.values() for m in ms)
doc = {"source": path, "launches": len(lau), "total_ns": tot, "families": {}}
for f, ms in sorted(fam.items(), key=lambda x: -sum(m.get("gpu__time_duration.sum", 0) for m in x[1])):
    t = sum(m.get("gpu__time_duration.sum", 0) for m in ms)
    dram = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ms]
    doc["families"][f] = {"launches": len(ms), "total_ns": t, "share": round(t / tot, 4), "mean_ns": t / len(ms),
                          "mean_dram_bytes": sum(dram) / len(dram)}
json.dump(doc, open(out, "w"), indent=1)
for f, v in doc["families"].items():
    print(f"{f[:60]:60s} n={v['launches']:4d} mean {v['mean_ns']/1e3:8.1f} us share {v['share']:.3f} dram {v['mean_dram_bytes']/1e6:8.1f} MB")
