"""Summarise an ncu launch-list CSV of tests/_profile_run.py into
profiles/ncu_summary.json (DRAM bytes, kernel time and tensor-pipe share of the
fused chain vs the cuBLAS unfused chain, per workload)."""
import csv, json, sys
path, names, out = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
launches = []
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    if not launches or launches[-1]["key"] != key:
        launches.append({"key": key, "name": r["Kernel Name"], "m": {}})
    v = r["Metric Value"].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        pass
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
    launches[-1]["m"][r["Metric Name"]] = v * scale if isinstance(v, float) else v
doc = {"round": "r01 (session 5)", "method": "ncu --cache-control all --clock-control none --metrics gpu__time_duration.sum,"
       "dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed "
       "python tests/_profile_run.py (FF_NO_COOPERATIVE=1); per-launch values are cold-cache and serialised"}
i = 0
for name in names:
    while i < len(launches) and "ff_chain" not in launches[i]["name"]:
        i += 1  # workspace zero-fill of a fresh (larger) workspace
    fused = []
    while i < len(launches) and "ff_chain" in launches[i]["name"]:
        fused.append(launches[i]); i += 1
    chain = []
    while i < len(launches) and "ff_chain" not in launches[i]["name"] and "FillFunctor" not in launches[i]["name"]:
        chain.append(launches[i]); i += 1
    f = fused[-1]
    per = len(chain) // 2
    last = chain[per:]
    dram = lambda L: L["m"].get("dram__bytes_read.sum", 0) + L["m"].get("dram__bytes_write.sum", 0)
    doc[name] = {
        "dram_bytes_per_launch": int(dram(f)),
        "fused_chain_dram_bytes": int(dram(f)),
        "fused_chain_ns": int(f["m"].get("gpu__time_duration.sum", 0)),
        "fused_kernels": [f["name"][:60]],
        "fused_tensor_pipe_pct": round(f["m"].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0), 2),
        "cublas_dram_bytes": int(sum(dram(L) for L in last)),
        "cublas_chain_ns": int(sum(L["m"].get("gpu__time_duration.sum", 0) for L in last)),
        "cublas_kernels": [L["name"][:60] for L in last],
        "cublas_tensor_pipe_pct": [round(L["m"].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0), 2) for L in last],
    }
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc, indent=1))
