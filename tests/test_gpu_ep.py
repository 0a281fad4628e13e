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
