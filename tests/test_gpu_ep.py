"""Expert-parallel layer on the GPU path (NCCL, world size 1 on the one-GPU
box): dispatch -> local tcgen05 grouped GEMMs -> reverse all-to-all ->
combine must reproduce the single-GPU prefill layer bit-for-bit (row results
of the expert GEMMs do not depend on which rows share a tile)."""

import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_ep_world1_equals_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.distributed as dist
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.ep import ep_model, gpu_ep_layer
    from paper_2501_10375_b200.model import MoEModel

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m = MoEModel(P.ModelShape(2, 8, 2), 512, 1024, seed=4, resident_layers=[0])
        h = m.input_hidden(300, stream=6)
        ref = MoEBlockEngine(m).prefill(h, 0)
        out, sel, w, plan = gpu_ep_layer(m, 0, h)
        torch.cuda.synchronize()
        assert torch.equal(sel, ref["topk_idx"])
        assert torch.equal(out, ref["out"])
        assert plan.local_offsets == ref["offsets"].tolist()
        # a rank model holding only its own experts (world 1: all of them)
        me = ep_model(P.ModelShape(2, 8, 2), 512, 1024, 0, 1, seed=4)
        out2, _, _, _ = gpu_ep_layer(me, 0, h)
        assert torch.equal(out2, ref["out"])
    finally:
        dist.destroy_process_group()


def _single_gpu_reference(P, E, d, ffn, seed):
    from paper_2501_10375_b200.engine import MoEBlockEngine
    from paper_2501_10375_b200.model import MoEModel
    m = MoEModel(P.ModelShape(2, E, 2), d, ffn, seed=seed, resident_layers=[0])
    return m, MoEBlockEngine(m)


def test_peer_ep_world1_equals_single_gpu():
    """Peer-memory EP without peers: dispatch kernel = permutation gather,
    fused-return down GEMM = plain down GEMM -> bit-identical prefill."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.ep import PeerEP, ep_model
    m, eng = _single_gpu_reference(P, 8, 512, 1024, 5)
    me = ep_model(P.ModelShape(2, 8, 2), 512, 1024, 0, 1, seed=5)
    ctx = PeerEP(me, 0, t_cap=700)
    for step, t in enumerate((700, 129, 1)):  # several epochs, both count slots
        h = m.input_hidden(t, stream=7, step=step)
        ref = eng.prefill(h, 0)
        out, sel, w = ctx.layer(h)
        torch.cuda.synchronize()
        ctx.check()
        assert torch.equal(sel, ref["topk_idx"])
        assert torch.equal(out, ref["out"])
        assert ctx.local_offsets().tolist() == ref["offsets"].tolist()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_peer_ep_emulated_ranks_equal_single_gpu(G):
    """G ranks in one process on one GPU, each with its own workspace, its
    own E/G experts and its own tokens; the peer tables point at each
    other's workspaces, so dispatch (remote row stores), the expert-major
    receive layout, the fused-return GEMM epilogue (stores into the source's
    y_back) and the epoch flags run exactly as across G GPUs.  Every rank's
    output must equal the single-GPU prefill of its tokens bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2501_10375_b200 as P
    from paper_2501_10375_b200.ep import PeerEP, ep_model
    E, d, ffn = 8, 512, 1024
    m, eng = _single_gpu_reference(P, E, d, ffn, 6)
    models = [ep_model(P.ModelShape(2, E, 2), d, ffn, r, G, seed=6) for r in range(G)]
    ranks = PeerEP.emulated(models, 0, t_cap=400)
    tok = [400, 1, 257, 33, 400, 2, 64, 300][:G]
    for step in range(3):
        hs = [m.input_hidden(tok[r], stream=20 + r, step=step) for r in range(G)]
        for r in range(G):
            ranks[r].route(hs[r])
        for r in range(G):
            ranks[r].publish()
        for r in range(G):
            ranks[r].dispatch()
        for r in range(G):
            ranks[r].experts()
        outs = [ranks[r].finish() for r in range(G)]
        torch.cuda.synchronize()
        for r in range(G):
            ranks[r].check()
            ref = eng.prefill(hs[r], 0)
            assert torch.equal(outs[r][1], ref["topk_idx"])
            assert torch.equal(outs[r][0], ref["out"]), (G, step, r)
        # every row was received exactly once by its owner
        total = sum(int(ranks[r].local_offsets()[-1]) for r in range(G))
        assert total == 2 * sum(tok)
