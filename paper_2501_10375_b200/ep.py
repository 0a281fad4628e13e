"""Expert parallelism over several GPUs.

Experts are independent units: expert e of every layer lives on rank
owner(e) = floor(e * G / E); tokens are sharded data-parallel.  One MoE layer:

  1. router on the rank's own tokens (fused router kernel): x, top-k, weights
  2. assignments (t, j) sorted stably by (owner, expert, t, j)
  3. count exchange (all_to_all of G ints), then payload all_to_all of the
     bf16 x rows and their expert ids with those split sizes
  4. the owner runs its local experts on what it received (permutation +
     tcgen05 grouped GEMMs on its slab)
  5. reverse all_to_all of the fp32 expert outputs
  6. combine on the token's rank: h' = h + sum_j w_j y_j in fixed j order

Row results of the expert GEMMs do not depend on which other rows share a
tile, so the EP output equals the single-GPU output.  The collectives are
NCCL (NVLink/NVSwitch) on GPUs and gloo in the CPU tests; decisions are made
before dispatch, so they are identical to the single-GPU decisions.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def owner_of(expert: torch.Tensor, num_experts: int, world: int) -> torch.Tensor:
    return (expert * world) // num_experts


def local_experts(rank: int, num_experts: int, world: int):
    return [e for e in range(num_experts) if (e * world) // num_experts == rank]


def ep_moe_layer(h: torch.Tensor, router_fn, expert_fn, num_experts: int, k: int,
                 group=None):
    """One expert-parallel MoE layer.

    router_fn(h) -> (x, sel, w): x (T, d) rows fed to experts, sel (T, k)
      int64 expert ids, w (T, k) fp32 combine weights.
    expert_fn(expert_ids (R,), x_rows (R, d)) -> (R, d) fp32 outputs of this
      rank's local experts.
    Returns (h', sel, w).
    """
    G = dist.get_world_size(group)
    T, d = h.shape
    x, sel, w = router_fn(h)
    sel = sel.to(torch.int64)
    flat_e = sel.reshape(-1)
    dest = owner_of(flat_e, num_experts, G)
    order = torch.argsort(dest * num_experts + flat_e, stable=True)
    send_counts = torch.bincount(dest, minlength=G).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    s_split = send_counts.tolist()
    r_split = recv_counts.tolist()
    send_x = x[order // k].contiguous()
    send_e = flat_e[order].contiguous()
    R = int(sum(r_split))
    recv_x = torch.empty((R, x.shape[1]), dtype=x.dtype, device=x.device)
    recv_e = torch.empty((R,), dtype=send_e.dtype, device=send_e.device)
    _a2a(recv_x, send_x, r_split, s_split, group)
    _a2a(recv_e, send_e, r_split, s_split, group)
    y_recv = expert_fn(recv_e, recv_x).to(torch.float32).contiguous()
    y_back = torch.empty((T * k, d), dtype=torch.float32, device=h.device)
    _a2a(y_back, y_recv, s_split, r_split, group)
    y = torch.empty_like(y_back)
    y[order] = y_back
    if h.is_cuda:
        # same fixed-order fused combine kernel as the single-GPU path
        from . import ops
        inv = torch.arange(T * k, dtype=torch.int32, device=h.device).view(T, k)
        out = ops.combine(h.to(torch.float32).contiguous(), y, inv,
                          w.to(torch.float32).contiguous())
        return out, sel, w
    y = y.view(T, k, d)
    out = h.to(torch.float32).clone()
    for j in range(k):
        out = out + w[:, j:j + 1].to(torch.float32) * y[:, j]
    return out, sel, w


def _a2a(out, inp, out_split, in_split, group):
    dist.all_to_all_single(out, inp, out_split, in_split, group=group)


def gpu_router_fn(model, layer: int):
    """Fused router kernel as the EP router (device tensors)."""
    from . import ops

    def fn(h):
        nxt = model.gate[layer + 1] if layer + 1 < model.shape.num_layers else None
        r = ops.router(h, model.norm[layer], model.gate[layer], nxt, model.shape.top_k)
        return r["x"], r["topk_idx"].to(torch.int64), r["topk_w"]

    return fn


def gpu_expert_fn(model, layer: int):
    """This rank's experts on received rows: permutation + tcgen05 grouped
    GEMMs over the local slab (experts without a local slot get no tiles)."""
    from . import ops

    def fn(expert_ids, x_rows):
        if x_rows.shape[0] == 0:
            return torch.empty((0, model.d), dtype=torch.float32, device=x_rows.device)
        ids = expert_ids.to(torch.int32).view(-1, 1).contiguous()
        pr = ops.permute(ids, model.shape.num_experts, x_rows.contiguous())
        so = model.slot_of[layer]
        act = ops.expert_gemm_up(pr["x_perm"], pr["offsets"], so, model.slab, model.n_slots,
                                 model.slot_elems, model.d, model.ffn)
        y = ops.expert_gemm_down(act, pr["offsets"], so, model.slab, model.n_slots,
                                 model.slot_elems, model.d, model.ffn)
        return y[pr["inv"].view(-1).to(torch.int64)]

    return fn
