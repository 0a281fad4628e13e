"""Small invocations of each hot-path kernel for compute-sanitizer
(racecheck / synccheck / memcheck; scripts/sanitize.sh runs every case under
every tool and keeps the logs under profiles/).  Shapes are small so a
sanitizer's ~100x slowdown stays in seconds, but each case crosses the code
paths that matter: several tiles / chunks per CTA, ragged expert groups,
the self-resetting workspaces run twice.

    python scripts/sanitize_cases.py CASE
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2501_10375_b200 as P  # noqa: E402
from paper_2501_10375_b200 import ops  # noqa: E402
from paper_2501_10375_b200.engine import MoEBlockEngine  # noqa: E402
from paper_2501_10375_b200.model import MoEModel  # noqa: E402


def model(d=512, ffn=1024, E=8, k=2, L=2):
    return MoEModel(P.ModelShape(L, E, k), d, ffn, seed=1, device="cuda", resident_layers=[0])


def case_permute():
    # T*k in (256, 4096]: the single-CTA count/scan/scatter kernel over
    # several 256-row tiles (the ADVICE r01 race), then the multi-chunk path
    for T in (700, 2048, 5000):
        ids = torch.stack([torch.randperm(8)[:2] for _ in range(T)]).to(torch.int32).cuda()
        x = torch.randn(T, 64, device="cuda").to(torch.bfloat16)
        ops.permute(ids, 8, x)


def case_router():
    m = model()
    for T in (3, 64, 1000):
        h = m.input_hidden(T, stream=1)
        hist = torch.zeros((1, 2, 8), dtype=torch.int32, device="cuda")
        ops.router(h, m.norm[0], m.gate[0], m.gate[1], 2, hist=hist[:, 0], tokens_per_seq=T,
                   hist_seq_stride=16)


def case_decode():
    m = model()
    eng = MoEBlockEngine(m)
    for s in range(3):  # dataflow counters reset themselves between launches
        eng.decode(m.input_hidden(1, stream=2, step=s)[0])


def case_prefill():
    m = model()
    eng = MoEBlockEngine(m)
    for T in (64, 900):  # skinny GEMMs, then the CTA-pair grouped GEMMs
        eng.prefill(m.input_hidden(T, stream=3), 0)


def case_prefill_die():
    # enough rows for the per-die schedule (>= 16 pair m-tiles): the die probe,
    # the cluster ranks and the die-split tiles of both GEMMs, staged epilogue
    m = model()
    eng = MoEBlockEngine(m)
    eng.prefill(m.input_hidden(4608, stream=4), 0)


def case_attention_fused():
    # the attention core + O-proj cooperative kernel (off by default)
    from paper_2501_10375_b200 import _lib
    from paper_2501_10375_b200.attention import AttentionStack
    att = AttentionStack(1, 512, 4, 2, max_seq=256, seed=1, device="cuda")
    _lib.call("daop_set_attn_fused", 1)
    for pos in range(60, 63):
        att.decode(torch.randn(512, device="cuda"), 0, pos)
    _lib.call("daop_set_attn_fused", 0)


def case_ep():
    from paper_2501_10375_b200.ep import PeerEP, ep_model
    G = 2
    models = [ep_model(P.ModelShape(2, 8, 2), 512, 1024, r, G, seed=1) for r in range(G)]
    ranks = PeerEP.emulated(models, 0, t_cap=300)
    for step in range(2):
        hs = [models[0].input_hidden(300 - 100 * r, stream=9 + r, step=step) for r in range(G)]
        for r in range(G):
            ranks[r].route(hs[r])
        for r in range(G):
            ranks[r].publish()
        for r in range(G):
            ranks[r].dispatch()
        for r in range(G):
            ranks[r].experts()
        for r in range(G):
            ranks[r].finish()
    torch.cuda.synchronize()
    for r in ranks:
        r.check()


def case_attention():
    from paper_2501_10375_b200.attention import AttentionStack
    att = AttentionStack(1, 512, 4, 2, max_seq=256, seed=1, device="cuda")
    h = torch.randn(100, 512, device="cuda")
    att.prefill(h, 0, 0)
    for pos in range(100, 103):
        att.decode(torch.randn(512, device="cuda"), 0, pos)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
    torch.cuda.synchronize()
    print("ok", names)
