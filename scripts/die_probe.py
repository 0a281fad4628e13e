"""SM -> die map of the B200 (csrc/topology.cu): the timing probe's raw
first-access latencies, the slow fraction per SM and the library's
classification; with a die_pair.csv from scripts/die_pair_probe.py (ncu fabric
counter, same box) it also prints the agreement (development aid, GPU box)."""
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_10375_b200 import _lib  # noqa: E402

sms = torch.cuda.get_device_properties(0).multi_processor_count
nl, stride = 64, 160
for rep in range(2):
    buf = torch.zeros(sms * nl * stride, dtype=torch.int32, device="cuda")
    lat = torch.zeros((sms, nl), dtype=torch.int32, device="cuda")
    smid = torch.zeros(sms, dtype=torch.int32, device="cuda")
    _lib.call("daop_die_probe", buf.data_ptr(), nl, stride, sms, lat.data_ptr(), smid.data_ptr(), 0)
    torch.cuda.synchronize()
    L = lat.cpu().numpy().astype(np.int64)
    S = smid.cpu().numpy()
    L = L[np.argsort(S)]
    print("latency percentiles (clk) 5/25/50/75/95:", np.percentile(L, [5, 25, 50, 75, 95]))
    h, e = np.histogram(L.ravel(), bins=24)
    print("histogram:", [(int(a), int(b)) for a, b in zip(e[:-1], h)])
    thr = np.percentile(L, 87.5)
    f = (L >= thr).mean(axis=1)
    print("slow frac (>= p87.5):", " ".join(f"{i}:{x:.2f}" for i, x in enumerate(f)))
d = np.zeros(sms, dtype=np.int32)
nd = np.zeros(1, dtype=np.int32)
_lib.call("daop_die_map", d.ctypes.data, sms, nd.ctypes.data)
print("n_die", int(nd[0]), "die_of_sm:", "".join(str(x) for x in d))
if len(sys.argv) > 1 and Path(sys.argv[1]).exists():
    lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
    v = {}
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "lts__t_sectors_srcunit_ltcfabric.sum":
            v[int(r["ID"])] = float(r["Metric Value"].replace(",", ""))
    vals = [v[i] for i in sorted(v)]
    base = vals[0]
    truth = np.array([0] + [1 if x > 1.5 * base else 0 for x in vals[1:]])
    print("ncu truth:   ", "".join(str(x) for x in truth))
    print("agreement with the ncu fabric map:", float((truth == d).mean()), "n_die", int(nd[0]))
