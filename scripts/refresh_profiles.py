"""Turn a GPU session's raw outputs (gpurun_out/) into the committed profile
summaries under profiles/ (development aid, runs in the build container):

    python scripts/refresh_profiles.py [round]     # default r01

Reads  gpurun_out/prof_decode.ncu-rep, prof_gemm.ncu-rep, prof_router.ncu-rep
       (ncu --set full), gpurun_out/launches.csv (ncu gpu__time_duration list of
       one bench.py run), gpurun_out/bench.json, bench_ref.json
Writes profiles/<round>/ncu_full_summary.json, ncu_launches_share.json,
       ncu_launches_bench.csv, bench.json, bench_reference.json and
       profiles/ncu_decode_summary.json (the `traffic` bench.py reports).
"""
import csv
import json
import shutil
import sys
from collections import OrderedDict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarise  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
DECODE_BYTES = 704_774_144


def num(v):
    return float(str(v).split()[0].replace(",", ""))


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    dst = ROOT / "profiles" / rnd
    dst.mkdir(parents=True, exist_ok=True)
    full = {}
    for name in ("decode", "gemm", "router", "attn_prefill", "skinny", "attention", "ep"):
        rep = OUT / f"prof_{name}.ncu-rep"
        if rep.exists():
            full[name] = summarise(str(rep))
    if full:
        (dst / "ncu_full_summary.json").write_text(json.dumps(full, indent=1))
    dec = full.get("decode")
    if dec:
        k = dec[0]
        rd = num(k["dram__bytes_read.sum"]) * (1e6 if "Mbyte" in k["dram__bytes_read.sum"] else 1e9 if "Gbyte" in k["dram__bytes_read.sum"] else 1)
        wr = num(k["dram__bytes_write.sum"]) * (1e6 if "Mbyte" in k["dram__bytes_write.sum"] else 1e9 if "Gbyte" in k["dram__bytes_write.sum"] else 1)
        (ROOT / "profiles" / "ncu_decode_summary.json").write_text(json.dumps({
            "kernel": k["Kernel Name"],
            "source": f"profiles/{rnd}/ncu_full_summary.json (ncu --set full, one launch)",
            "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
            "algorithmic_bytes_per_launch": DECODE_BYTES}, indent=1))
    lc = OUT / "launches.csv"
    if lc.exists():
        shutil.copy(lc, dst / "ncu_launches_bench.csv")
        rows = list(csv.reader(open(lc)))
        i = [j for j, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[i]
        ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
        agg = OrderedDict()
        for r in rows[i + 1:]:
            if r[mi] != "gpu__time_duration.sum":
                continue
            name = r[ki].split("(")[0]
            a = agg.setdefault(name, [0, 0.0])
            a[0] += 1
            a[1] += num(r[vi])
        tot = sum(v[1] for v in agg.values())
        (dst / "ncu_launches_share.json").write_text(json.dumps({
            "unit": "ns (gpu__time_duration.sum; ncu --clock-control none, serialised, cold caches)",
            "kernels": {n: {"launches": c, "total_ns": t, "mean_ns": t / c, "share": t / tot}
                        for n, (c, t) in agg.items()}}, indent=1))
    for src, name in (("bench.json", "bench.json"), ("bench_ref.json", "bench_reference.json")):
        p = OUT / src
        if p.exists() and p.stat().st_size:
            shutil.copy(p, dst / name)
    print("profiles refreshed under", dst)


if __name__ == "__main__":
    main()
