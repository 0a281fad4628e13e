"""Expert-parallel dispatch/combine with world_size 2 on CPU (gloo).

The expert and router computations are the oracle's (numpy) -- this test
covers the EP host logic: ownership, stable ordering, count exchange,
payload all-to-all (incl. bf16 bits), reverse all-to-all and the fixed-order
combine.  EP(2) must equal the single-process oracle layer over all tokens.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numerics as N

D, FFN, E, K, T_PER = 64, 128, 8, 2, 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_10375_b200.ep import ep_moe_layer, local_experts
    om = N.OracleModel(2, E, K, D, FFN, seed=9)
    mine = local_experts(rank, E, world)
    W = {e: (om.w1(0, e), om.w3(0, e), om.w2(0, e)) for e in mine}
    h_all = N.input_hidden(9, 3, 0, T_PER * world, D)
    h = torch.from_numpy(h_all[rank * T_PER:(rank + 1) * T_PER].copy())

    def router_fn(hh):
        x = N.rmsnorm(hh.numpy(), om.norm(0))
        p, _ = N.router(x, om.gate(0), om.gate(1))
        from oracle.decisions import topk_rows
        sel = topk_rows(p.astype(np.float64), K)
        w = N.renorm_weights(p, sel)
        xb = torch.from_numpy(x).to(torch.bfloat16)
        return xb, torch.from_numpy(sel), torch.from_numpy(w)

    def permute_fn(sel_t, x):
        offsets, perm, inv = N.permutation(sel_t.numpy(), E)
        return torch.from_numpy(offsets), x[torch.from_numpy(perm // K)], torch.from_numpy(inv)

    def expert_fn(xr, local_offsets):
        out = np.zeros((xr.shape[0], D), dtype=np.float32)
        xs = xr.to(torch.float32).numpy()
        for e in range(E):
            a, b = local_offsets[e], local_offsets[e + 1]
            if b > a:
                assert e in mine, f"rank {rank} received expert {e}"
                out[a:b] = N.expert_ffn(xs[a:b], *W[e])
        return torch.from_numpy(out)

    def combine_fn(hh, y_perm, inv, w):
        return torch.from_numpy(N.combine(hh.numpy(), y_perm.numpy(), inv.numpy(), w.numpy()))

    out, sel, w, plan = ep_moe_layer(h, router_fn, permute_fn, expert_fn, combine_fn, E)
    # every row this rank sent came back, and the receive buffer is expert-major
    assert plan.local_offsets[-1] == plan.recv_rows
    assert sum(n for _, n in plan.send) == T_PER * K
    q.put((rank, out.numpy(), sel.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, out, sel = q.get(timeout=60)
        res[r] = (out, sel)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = np.concatenate([res[r][0] for r in range(world)])
    sel = np.concatenate([res[r][1] for r in range(world)])
    om = N.OracleModel(2, E, K, D, FFN, seed=9)
    h_all = N.input_hidden(9, 3, 0, T_PER * world, D)
    ref = N.moe_layer(om, 0, h_all)
    assert np.array_equal(sel, ref["sel"])
    assert np.abs(out - ref["out"]).max() <= 1e-5 * (1 + np.abs(ref["out"]).max())


def test_ownership_partition():
    from paper_2501_10375_b200.ep import local_experts, owner_of
    for G in (1, 2, 4, 8):
        parts = [local_experts(r, 8, G) for r in range(G)]
        assert sorted(sum(parts, [])) == list(range(8))
        assert all(len(p) == 8 // G for p in parts)
        assert owner_of(torch.arange(8), 8, G).tolist() == [e * G // 8 for e in range(8)]


def test_plan_exchange_expert_major():
    """Receive buffer groups rows by local expert, then by source rank."""
    from paper_2501_10375_b200.ep import plan_exchange
    # world 2, E 4: rank 1 owns experts 2, 3; sources send (5, 7) and (1, 0) rows
    plan = plan_exchange([0, 3, 4, 9, 16], [[5, 7], [1, 0]], 1, 2, 4)
    assert plan.send == [(0, 3), (3, 1), (4, 5), (9, 7)]
    assert plan.recv == {(0, 2): (0, 5), (1, 2): (5, 1), (0, 3): (6, 7), (1, 3): (13, 0)}
    assert plan.local_offsets == [0, 0, 0, 6, 13]
    assert plan.recv_rows == 13


def test_plan_exchange_properties():
    """Random count matrices: every source segment is sent once, every owner
    receives exactly the rows addressed to its experts, receive segments tile
    [0, recv_rows) expert-major without gaps, and non-local experts are empty."""
    from hypothesis import given, settings
    from hypothesis import strategies as st
    from paper_2501_10375_b200.ep import local_experts, plan_exchange

    @settings(max_examples=200, deadline=None)
    @given(st.sampled_from([(1, 8), (2, 8), (4, 8), (8, 8), (2, 4), (4, 16)]),
           st.data())
    def check(ge, data):
        G, E = ge
        counts = [[data.draw(st.integers(0, 50)) for _ in range(E)] for _ in range(G)]
        for r in range(G):
            offs = [0]
            for e in range(E):
                offs.append(offs[-1] + counts[r][e])
            mine = local_experts(r, E, G)
            recv = [[counts[s][e] for e in mine] for s in range(G)]
            plan = plan_exchange(offs, recv, r, G, E)
            assert [n for _, n in plan.send] == counts[r]
            assert plan.recv_rows == sum(counts[s][e] for s in range(G) for e in mine)
            pos = 0
            for e in range(E):
                assert plan.local_offsets[e] == pos
                if e in mine:
                    for s in range(G):
                        a, n = plan.recv[(s, e)]
                        assert a == pos and n == counts[s][e]
                        pos += n
                assert plan.local_offsets[e + 1] == pos
            assert pos == plan.recv_rows

    check()
