"""Summarise an `ncu --metrics ... --csv --log-file` launch list: one line per
launch, kernel name + every metric (development aid)."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
by = collections.OrderedDict()
for r in csv.DictReader(lines):
    d = by.setdefault(r["ID"], {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
short = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rdGB", "dram__bytes_write.sum": "wrGB",
         "lts__t_sector_hit_rate.pct": "L2hit", "launch__grid_size": "grid",
         "launch__cluster_size": "clus", "launch__block_size": "blk",
         "launch__shared_mem_per_block_dynamic": "smem",
         "launch__registers_per_thread": "regs",
         "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor%",
         "sm__cycles_elapsed.avg.per_second": "clk"}
for k, d in by.items():
    out = []
    for m, vu in d.items():
        if m == "name":
            continue
        v, u = vu
        v = float(v.replace(",", "")) if v.replace(",", "").replace(".", "").isdigit() else v
        if m == "gpu__time_duration.sum":
            v = v / 1e3 if u == "ns" else v * 1e3 if u == "msecond" else v
        if m.startswith("dram__bytes"):
            v = v / {"byte": 1e9, "Kbyte": 1e6, "Mbyte": 1e3, "Gbyte": 1}.get(u, 1e9)
        out.append(f"{short.get(m, m)}={v:.4g}" if isinstance(v, float) else f"{short.get(m, m)}={v}")
    print(k, d["name"][:90])
    print("    " + " ".join(out))
