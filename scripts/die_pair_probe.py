"""SM -> die map from the die-to-die fabric counter (run under ncu:
    ncu --metrics lts__t_sectors_srcunit_ltcfabric.sum -k regex:die_pair --csv ...
launch i: SM 0 reads a 16 MB buffer, then SM test_i reads it; the first launch
has SM 0 read it twice).  Development aid, GPU box."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2501_10375_b200 import _lib  # noqa: E402

n = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.randint(0, 1 << 30, (4 << 20,), dtype=torch.int32, device="cuda")  # 16 MB
flag = torch.zeros(4, dtype=torch.int32, device="cuda")
tests = [0] + list(range(1, n))
for t in tests:
    # flush L2 between launches: read a 256 MB buffer
    junk = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    junk.fill_(1)
    del junk
    _lib.call("daop_die_pair_probe", buf.data_ptr(), buf.numel() * 4, 0, t, flag.data_ptr(), 0)
    torch.cuda.synchronize()
print("tests", tests)
