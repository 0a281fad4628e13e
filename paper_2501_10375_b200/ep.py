"""Expert parallelism over several GPUs.

Experts are independent units: expert e of every layer lives on rank
owner(e) = floor(e * G / E) (E/G consecutive experts per rank); tokens are
sharded data-parallel.  One MoE layer on rank r:

  1. router on the rank's own tokens (fused router kernel): x, top-k, weights
  2. stable permutation by (expert, t, j) -- the same histogram + scan +
     scatter + gather kernels as the single-GPU prefill.  owner() is monotone
     in e, so x_perm is already grouped by destination rank: it IS the send
     buffer, segment e = rows [offsets[e], offsets[e+1])
  3. count exchange: all_to_all of the (G, E/G) per-expert counts, so every
     owner knows how many rows of each of its experts each source sends
  4. payload exchange as one batch of point-to-point transfers (NCCL groups
     them into a single launch, like all_to_all): source segment (src, e)
     lands in the owner's receive buffer at an EXPERT-MAJOR position
     (expert, then source rank), so the received rows are already grouped by
     expert and the tcgen05 grouped GEMMs run on them directly (no re-permute)
  5. up / down grouped GEMMs on the owner's slab (offsets over all E experts,
     zero rows for non-local experts)
  6. reverse exchange of the fp32 expert outputs straight into the source's
     permuted order, then the fixed-order combine kernel with the
     permutation's inverse -- the single-GPU combine, unchanged

Row results of the expert GEMMs do not depend on which other rows share a
tile, so the EP output equals the single-GPU output bit for bit.  Decisions
are made before dispatch, so they are identical too.  The collectives are
NCCL over NVLink/NVSwitch on GPUs; the CPU tests run the same exchange over
gloo (world size 2) with the oracle's permutation / experts / combine
injected -- this module does no arithmetic of its own.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

# SKINNY_MAX_ROWS: receive capacity up to which the skinny (weights-as-M) GEMMs
# run -- the single-GPU crossover (scripts/skinny_crossover.py)
from .engine import SKINNY_MAX_ROWS


def owner_of(expert: torch.Tensor, num_experts: int, world: int) -> torch.Tensor:
    return (expert * world) // num_experts


def local_experts(rank: int, num_experts: int, world: int):
    return [e for e in range(num_experts) if (e * world) // num_experts == rank]


@dataclass
class ExchangePlan:
    """Row segments of one layer's dispatch on one rank (host integers).

    send[e] = (start, rows) of expert e in this rank's permuted buffer;
    recv[(src, e)] = (start, rows) of source src's rows of local expert e in
    the expert-major receive buffer; local_offsets (E+1) = row offsets of
    every expert in the receive buffer (zero rows for non-local experts)."""
    rank: int
    world: int
    num_experts: int
    send: list
    recv: dict
    local_offsets: list
    recv_rows: int


def plan_exchange(send_offsets, recv_counts, rank: int, world: int,
                  num_experts: int) -> ExchangePlan:
    """send_offsets: (E+1) host ints of the permuted buffer; recv_counts:
    (G, E/G) host ints, recv_counts[src][i] = rows of local expert i from src."""
    E, G = num_experts, world
    per = E // G
    send = [(int(send_offsets[e]), int(send_offsets[e + 1] - send_offsets[e])) for e in range(E)]
    mine = local_experts(rank, E, G)
    recv, local = {}, [0] * (E + 1)
    pos = 0
    for e in range(E):
        local[e] = pos
        if e in mine:
            i = e - mine[0]
            for src in range(G):
                n = int(recv_counts[src][i])
                recv[(src, e)] = (pos, n)
                pos += n
    local[E] = pos
    assert per * G == E
    return ExchangePlan(rank, G, E, send, recv, local, pos)


def _p2p(ops_list, group):
    if ops_list:
        for req in dist.batch_isend_irecv(ops_list):
            req.wait()


def dispatch(plan: ExchangePlan, x_perm: torch.Tensor, group=None) -> torch.Tensor:
    """Source-permuted rows -> owner's expert-major receive buffer."""
    E, G, r = plan.num_experts, plan.world, plan.rank
    if G == 1:
        return x_perm
    out = torch.empty((plan.recv_rows,) + tuple(x_perm.shape[1:]), dtype=x_perm.dtype,
                      device=x_perm.device)
    ops_list = []
    for e in range(E):  # sends in expert order; each owner receives in the same order
        dst = e * G // E
        a, n = plan.send[e]
        if n and dst != r:
            ops_list.append(dist.P2POp(dist.isend, x_perm[a:a + n], _peer(dst, group), group))
    for (src, e), (a, n) in sorted(plan.recv.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        if not n:
            continue
        if src == r:
            s, _ = plan.send[e]
            out[a:a + n].copy_(x_perm[s:s + n])
        else:
            ops_list.append(dist.P2POp(dist.irecv, out[a:a + n], _peer(src, group), group))
    _p2p(ops_list, group)
    return out


def gather_back(plan: ExchangePlan, y_recv: torch.Tensor, group=None) -> torch.Tensor:
    """Owner's expert-major outputs -> source's permuted order."""
    E, G, r = plan.num_experts, plan.world, plan.rank
    if G == 1:
        return y_recv
    rows = plan.send[-1][0] + plan.send[-1][1] if plan.send else 0
    out = torch.empty((rows,) + tuple(y_recv.shape[1:]), dtype=y_recv.dtype,
                      device=y_recv.device)
    ops_list = []
    for (src, e), (a, n) in sorted(plan.recv.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        if n and src != r:
            ops_list.append(dist.P2POp(dist.isend, y_recv[a:a + n], _peer(src, group), group))
    for e in range(E):
        owner = e * G // E
        s, n = plan.send[e]
        if not n:
            continue
        if owner == r:
            a, _ = plan.recv[(r, e)]
            out[s:s + n].copy_(y_recv[a:a + n])
        else:
            ops_list.append(dist.P2POp(dist.irecv, out[s:s + n], _peer(owner, group), group))
    _p2p(ops_list, group)
    return out


def _peer(rank_in_group, group):
    return rank_in_group if group is None else dist.get_global_rank(group, rank_in_group)


def exchange_counts(send_offsets: torch.Tensor, world: int, group=None):
    """all_to_all of per-expert row counts: returns (G, E/G) host ints."""
    counts = (send_offsets[1:] - send_offsets[:-1]).to(torch.int64)
    E = counts.numel()
    if world == 1:
        return counts.view(1, E).tolist()
    recv = torch.empty_like(counts)
    dist.all_to_all_single(recv, counts, group=group)
    return recv.view(world, E // world).tolist()


def ep_moe_layer(h: torch.Tensor, router_fn, permute_fn, expert_fn, combine_fn,
                 num_experts: int, group=None, timings=None):
    """One expert-parallel MoE layer on this rank's tokens h (T, d).

    router_fn(h) -> (x (T,d), sel (T,k), w (T,k))
    permute_fn(sel, x) -> (offsets (E+1), x_perm (T*k, d), inv (T,k))
    expert_fn(x_recv (R,d), local_offsets (E+1) host ints) -> (R, d) fp32
      outputs of this rank's experts, rows grouped by expert
    combine_fn(h, y_perm, inv, w) -> h'
    Returns (h', sel, w, plan).  `timings` (optional list) receives
    (name, event) pairs around the phases when h is on a GPU."""
    if dist.is_available() and dist.is_initialized():
        G, r = dist.get_world_size(group), dist.get_rank(group)
    else:  # one GPU, no process group: the same path without a collective
        G, r = 1, 0
    mark = _marker(h, timings)
    x, sel, w = router_fn(h)
    offsets, x_perm, inv = permute_fn(sel, x)
    mark("route+permute")
    recv_counts = exchange_counts(offsets, G, group)
    plan = plan_exchange(offsets.tolist(), recv_counts, r, G, num_experts)
    x_recv = dispatch(plan, x_perm, group)
    mark("dispatch")
    y_recv = expert_fn(x_recv, plan.local_offsets)
    mark("experts")
    y_perm = gather_back(plan, y_recv, group)
    mark("gather")
    out = combine_fn(h, y_perm, inv, w)
    mark("combine")
    return out, sel, w, plan


def _marker(h, timings):
    if timings is None or not h.is_cuda:
        return lambda name: None
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    timings.append(("start", ev))

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        timings.append((name, e))
    return mark


# ------------------------------------------------------------------ GPU functions


def gpu_router_fn(model, layer: int):
    """Fused router kernel as the EP router (device tensors)."""
    from . import ops

    def fn(h):
        nxt = model.gate[layer + 1] if layer + 1 < model.shape.num_layers else None
        r = ops.router(h, model.norm[layer], model.gate[layer], nxt, model.shape.top_k)
        return r["x"], r["topk_idx"], r["topk_w"]

    return fn


def gpu_permute_fn(num_experts: int):
    from . import ops

    def fn(sel, x):
        pr = ops.permute(sel, num_experts, x)
        return pr["offsets"], pr["x_perm"], pr["inv"]

    return fn


def gpu_expert_fn(model, layer: int):
    """This rank's experts on the expert-major receive buffer: tcgen05
    grouped GEMMs over the local slab, no re-permutation."""
    from . import ops

    def fn(x_recv, local_offsets):
        if x_recv.shape[0] == 0:
            return torch.empty((0, model.d), dtype=torch.float32, device=x_recv.device)
        off = torch.tensor(local_offsets, dtype=torch.int64).to(x_recv.device, non_blocking=True)
        so = model.slot_of[layer]
        act = ops.expert_gemm_up(x_recv, off, so, model.slab, model.n_slots,
                                 model.slot_elems, model.d, model.ffn)
        return ops.expert_gemm_down(act, off, so, model.slab, model.n_slots,
                                    model.slot_elems, model.d, model.ffn)

    return fn


def gpu_combine_fn():
    from . import ops

    def fn(h, y_perm, inv, w):
        return ops.combine(h, y_perm, inv, w)

    return fn


def gpu_ep_layer(model, layer: int, h: torch.Tensor, group=None, timings=None):
    """EP MoE layer with every phase on the B200 path."""
    return ep_moe_layer(h, gpu_router_fn(model, layer), gpu_permute_fn(model.shape.num_experts),
                        gpu_expert_fn(model, layer), gpu_combine_fn(),
                        model.shape.num_experts, group=group, timings=timings)


def ep_model(shape, d_model: int, d_ff: int, rank: int, world: int, layers=(0,), seed: int = 0,
             device="cuda"):
    """A MoEModel holding only this rank's experts (E/G slots per layer)."""
    from .model import MoEModel
    E = shape.num_experts
    mine = local_experts(rank, E, world)
    m = MoEModel(shape, d_model, d_ff, seed=seed, device=device,
                 n_slots=len(mine) * len(layers), resident_layers=[])
    for l in layers:
        for e in mine:
            m.load_expert(l, e)
    return m


def open_peer_table(ws: torch.Tensor, rank: int, world: int, group=None):
    """Exchange this rank's workspace by CUDA IPC over the process group and
    open every peer's: returns (device table of the G workspace addresses as
    seen from this GPU, opened IPC bases to close)."""
    import ctypes

    from . import _lib
    torch.cuda.synchronize()  # the zeroed workspace must exist before any peer flags it
    handle = ctypes.create_string_buffer(64)
    off = torch.zeros(1, dtype=torch.int64)
    _lib.call("daop_ep_ipc_handle", ws.data_ptr(), ctypes.addressof(handle), off.data_ptr())
    allh = [None] * world
    dist.all_gather_object(allh, (bytes(handle.raw), int(off[0])), group=group)
    ptrs, bases, err = [], [], ""
    for s, (hb, o) in enumerate(allh):
        if s == rank:
            ptrs.append(ws.data_ptr())
            continue
        hbuf = ctypes.create_string_buffer(hb, 64)
        base, ptr = ctypes.c_void_p(), ctypes.c_void_p()
        try:
            _lib.call("daop_ep_ipc_open", ctypes.addressof(hbuf), o, ctypes.byref(base),
                      ctypes.byref(ptr))
        except Exception as exc:  # every rank must learn about it (no half-open group)
            err = f"rank {rank}: peer {s}: {exc}"
            break
        bases.append(base.value)
        ptrs.append(ptr.value)
    _all_ok(not err, group, err or "a peer could not open this rank's workspace", bases)
    return torch.tensor(ptrs, dtype=torch.int64, device=ws.device), bases


def _all_ok(ok: bool, group, what: str, bases=()):
    """Collective success check: every rank raises if any rank failed, so the
    ranks never diverge into mismatched collectives."""
    from . import _lib
    from .errors import DeviceError
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                        device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:
        for b in bases:
            try:
                _lib.call("daop_ep_ipc_close", b)
            except Exception:
                pass
        raise DeviceError(f"peer-memory EP setup failed: {what}")


def _check_ws(ws: torch.Tensor, what: str, world: int = 1, group=None):
    """Raise if any cross-GPU wait of this workspace timed out -- on every
    rank when world > 1 (the flag is reduced over the group)."""
    from . import _lib
    from .errors import DeviceError
    err = torch.zeros(1, dtype=torch.int32)
    _lib.call("daop_ep_status", ws.data_ptr(), err.data_ptr())
    bad = int(err[0])
    if world > 1 and dist.is_available() and dist.is_initialized():
        flag = torch.tensor([bad], dtype=torch.int32,
                            device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        bad = int(flag.item())
    if bad:
        raise DeviceError(f"{what}: a cross-GPU wait timed out (peer not progressing)")


# ------------------------------------------------------------------ peer-memory EP


class PeerEP:
    """Expert-parallel MoE layer over NVLink peer memory (csrc/ep_p2p.cu).

    Replaces the NCCL exchanges of `ep_moe_layer` with kernels that store
    straight into the peers' symmetric workspaces: the permutation gather IS
    the dispatch (x rows go from token order to the owner's expert-major
    receive buffer in one pass), and the down GEMM's epilogue IS the return
    all-to-all (each fp32 output tile is stored into the source rank's
    y_back as it leaves TMEM).  Ranks synchronise through epoch flags in the
    workspaces; nothing on the path waits for the host, so a layer is one
    stream of launches (graph-capturable).

    `model` holds this rank's experts (ep_model); `t_cap` bounds the tokens
    per rank per call.  With world > 1 the workspaces are exchanged by CUDA
    IPC over the process group (one process per GPU)."""

    def __init__(self, model, layer: int, t_cap: int, rank: int = 0, world: int = 1,
                 group=None, _peer_table=None):
        from . import _lib
        self.m, self.layer_idx, self.rank, self.world = model, layer, rank, world
        self.E, self.k, self.d, self.ffn = (model.shape.num_experts, model.shape.top_k,
                                            model.d, model.ffn)
        self.t_cap = t_cap
        self.cap_send = t_cap * self.k
        self.cap_recv = world * t_cap * self.k
        out = [torch.zeros(1, dtype=torch.int64) for _ in range(4)]
        _lib.call("daop_ep_ws_layout", world, self.E, self.d, self.cap_recv, self.cap_send,
                  *[o.data_ptr() for o in out])
        total, self.recv_off, self.yback_off, self.local_off = (int(o[0]) for o in out)
        dev = model.device
        self.ws = torch.zeros(total, dtype=torch.uint8, device=dev)
        self.recv_x = self.ws[self.recv_off: self.recv_off + self.cap_recv * self.d * 2] \
            .view(torch.bfloat16).view(self.cap_recv, self.d)
        self.y_back = self.ws[self.yback_off: self.yback_off + self.cap_send * self.d * 4] \
            .view(torch.float32).view(self.cap_send, self.d)
        self.act = torch.empty((self.cap_recv, self.ffn), dtype=torch.bfloat16, device=dev)
        self.epoch = 0
        self._ipc_bases = []
        self._group = group
        if _peer_table is not None:
            self.peers = _peer_table
        elif world == 1:
            self.peers = torch.tensor([self.ws.data_ptr()], dtype=torch.int64, device=dev)
        else:
            self.peers = self._open_peers(group)

    def _open_peers(self, group):
        table, self._ipc_bases = open_peer_table(self.ws, self.rank, self.world, group)
        return table

    @classmethod
    def emulated(cls, models, layer: int, t_cap: int):
        """G ranks in ONE process on one GPU (test harness): every rank's
        peer table points at the G workspaces, so the kernels run the exact
        multi-rank data movement; the caller interleaves the phases."""
        G = len(models)
        ranks = [cls(m, layer, t_cap, r, G, _peer_table=torch.zeros(1)) for r, m in
                 enumerate(models)]
        table = torch.tensor([c.ws.data_ptr() for c in ranks], dtype=torch.int64,
                             device=models[0].device)
        for c in ranks:
            c.peers = table
        return ranks

    def close(self):
        from . import _lib
        for b in self._ipc_bases:
            _lib.call("daop_ep_ipc_close", b)
        self._ipc_bases = []

    # -- phases (one layer = route, publish, dispatch, experts, finish) -----
    def route(self, h):
        from . import ops
        m, l = self.m, self.layer_idx
        t = h.shape[0]
        if t > self.t_cap:
            raise ValueError(f"{t} tokens exceed the workspace capacity {self.t_cap}")
        nxt = m.gate[l + 1] if l + 1 < m.shape.num_layers else None
        r = ops.router(h, m.norm[l], m.gate[l], nxt, self.k)
        pr = ops.permute(r["topk_idx"], self.E)
        self.epoch += 1
        self._cur = dict(h=h, x=r["x"], sel=r["topk_idx"], w=r["topk_w"], perm=pr["perm"],
                         inv=pr["inv"], offsets=pr["offsets"], t=t)
        return self._cur

    def publish(self):
        from . import _lib, ops
        _lib.call("daop_ep_publish", self.peers.data_ptr(), self.rank, self.world, self.E,
                  self._cur["offsets"].data_ptr(), self.epoch, ops._s())

    def dispatch(self):
        from . import _lib, ops
        c = self._cur
        _lib.call("daop_ep_dispatch", self.peers.data_ptr(), self.rank, self.world, self.E,
                  self.k, self.d, c["x"].data_ptr(), c["perm"].data_ptr(), c["t"] * self.k,
                  self.recv_off, self.epoch, ops._s())

    def experts(self):
        from . import _lib, ops
        m, l = self.m, self.layer_idx
        s = ops._s()
        _lib.call("daop_ep_recv", self.peers.data_ptr(), self.rank, self.world, self.E, self.d,
                  self.yback_off, self.epoch, s)
        if self.cap_recv <= SKINNY_MAX_ROWS:  # batched decode: weights as the M side
            nt = ops.skinny_nt(self.cap_recv, self.E)  # ~1.25x the mean rows per expert
            _lib.call("daop_expert_gemm_up_skinny", self.recv_x.data_ptr(), self.cap_recv, self.d,
                      self.ffn, m.slab.data_ptr(), m.n_slots, m.slot_elems,
                      self.ws.data_ptr() + self.local_off, m.slot_of[l].data_ptr(), self.E,
                      self.act.data_ptr(), nt, s)
            _lib.call("daop_ep_expert_gemm_down_skinny", self.act.data_ptr(), self.cap_recv,
                      self.d, self.ffn, m.slab.data_ptr(), m.n_slots, m.slot_elems,
                      m.slot_of[l].data_ptr(), self.E, self.peers.data_ptr(), self.ws.data_ptr(),
                      self.rank, self.world, self.epoch, nt, s)
            return
        _lib.call("daop_expert_gemm_up", self.recv_x.data_ptr(), self.cap_recv, self.d, self.ffn,
                  m.slab.data_ptr(), m.n_slots, m.slot_elems, self.ws.data_ptr() + self.local_off,
                  m.slot_of[l].data_ptr(), self.E, self.act.data_ptr(), 0, s)
        _lib.call("daop_ep_expert_gemm_down", self.act.data_ptr(), self.cap_recv, self.d,
                  self.ffn, m.slab.data_ptr(), m.n_slots, m.slot_elems, m.slot_of[l].data_ptr(),
                  self.E, self.peers.data_ptr(), self.ws.data_ptr(), self.rank, self.world,
                  self.epoch, 0, s)

    def finish(self):
        from . import _lib, ops
        c = self._cur
        _lib.call("daop_ep_wait_back", self.ws.data_ptr(), self.world, self.epoch, ops._s())
        out = ops.combine(c["h"], self.y_back[: c["t"] * self.k], c["inv"], c["w"])
        return out, c["sel"], c["w"]

    def layer(self, h):
        """One EP MoE layer on this rank's tokens: (h', sel, w)."""
        self.route(h)
        self.publish()
        self.dispatch()
        self.experts()
        return self.finish()

    def local_offsets(self):
        return self.ws[self.local_off: self.local_off + 8 * (self.E + 1)].view(torch.int64)

    def check(self):
        """Raise (on every rank) if any cross-GPU wait timed out."""
        _check_ws(self.ws, "peer-memory EP", self.world, self._group)


class PeerEPDecode:
    """Expert-parallel decode of one token (b = 1) over NVLink peer memory.

    The residual stream is replicated on every rank.  Per layer each rank runs
    the fused decode kernel (router + selection + HBM-streaming SwiGLU GEMV)
    with ITS experts as the resident set -- the selection is the true top-k
    and identical on every rank, and each pick is streamed by exactly one
    GPU, so a token's 2 experts are read by 2 GPUs in parallel.  The owners
    store their picks' outputs into every peer's decode workspace
    (daop_ep_decode_share), and every rank combines h + sum_j w_j y_j in
    fixed j order -- bit-identical to the single-GPU decode layer.  DAOP
    PLAN mode (prediction-driven selection with degradation) is a
    single-GPU / host-tier feature: here every expert is in some GPU's HBM."""

    def __init__(self, model, rank: int = 0, world: int = 1, group=None, _peer_table=None):
        from . import _lib, ops
        self.m, self.rank, self.world = model, rank, world
        self.E, self.k, self.d, self.ffn = (model.shape.num_experts, model.shape.top_k,
                                            model.d, model.ffn)
        nb = torch.zeros(1, dtype=torch.int64)
        _lib.call("daop_ep_decode_ws_bytes", self.k, self.d, nb.data_ptr())
        dev = model.device
        self.ws = torch.zeros(int(nb[0]), dtype=torch.uint8, device=dev)
        self.ygather = self.ws[1024:].view(torch.float32).view(2, self.k, self.d)
        self.bufs = ops.DecodeBuffers(self.d, self.ffn, self.E, self.k, dev)
        self.out = [torch.empty(self.d, dtype=torch.float32, device=dev) for _ in range(2)]
        self.epoch = 0
        self._ipc_bases = []
        self._group = group
        if _peer_table is not None:
            self.peers = _peer_table
        elif world == 1:
            self.peers = torch.tensor([self.ws.data_ptr()], dtype=torch.int64, device=dev)
        else:
            self.peers, self._ipc_bases = open_peer_table(self.ws, rank, world, group)

    @classmethod
    def emulated(cls, models):
        """G ranks in one process on one GPU (test harness), see PeerEP.emulated."""
        ranks = [cls(m, r, len(models), _peer_table=torch.zeros(1)) for r, m in enumerate(models)]
        table = torch.tensor([c.ws.data_ptr() for c in ranks], dtype=torch.int64,
                             device=models[0].device)
        for c in ranks:
            c.peers = table
        return ranks

    def close(self):
        from . import _lib
        for b in self._ipc_bases:
            _lib.call("daop_ep_ipc_close", b)
        self._ipc_bases = []

    def stream(self, h: torch.Tensor, layer: int = 0):
        """Decode kernel on this rank's experts; its phase-2 reduction stores
        the local picks' outputs into every peer's workspace and its last CTA
        flags them (daop_ep_decode_layer)."""
        from . import _lib, ops
        m, b = self.m, self.bufs
        self.epoch += 1
        nxt = m.gate[layer + 1] if layer + 1 < m.shape.num_layers else None
        _lib.call("daop_ep_decode_layer", self.peers.data_ptr(), self.rank, self.world,
                  self.epoch, h.data_ptr(), m.norm[layer].data_ptr(), m.gate[layer].data_ptr(),
                  0 if nxt is None else nxt.data_ptr(), m.fast[layer].data_ptr(),
                  m.slot_of[layer].data_ptr(), m.slab.data_ptr(), m.slot_elems, self.d, self.ffn,
                  self.E, self.k, float(ops.RMS_EPS), b.x.data_ptr(), b.p.data_ptr(),
                  b.p_pred.data_ptr(), b.sel.data_ptr(), b.w.data_ptr(), b.is_fast.data_ptr(),
                  b.deg.data_ptr(), b.y.data_ptr(), b.h_out.data_ptr(), b.ws.data_ptr(), ops._s())
        self._h = h

    def finish(self) -> torch.Tensor:
        """Wait for every owner's outputs and combine (one kernel) -> the
        next residual."""
        from . import _lib, ops
        out = self.out[self.epoch & 1]
        _lib.call("daop_ep_decode_finish", self.ws.data_ptr(), self.world, self.k, self.d,
                  self._h.data_ptr(), self.bufs.w.data_ptr(), out.data_ptr(), self.epoch,
                  ops._s())
        return out

    def layer(self, h: torch.Tensor, layer: int = 0) -> torch.Tensor:
        self.stream(h, layer)
        return self.finish()

    def check(self):
        _check_ws(self.ws, "peer-memory EP decode", self.world, self._group)


def nccl_ep_decode_layer(model, layer: int, h: torch.Tensor, bufs, y_sum: torch.Tensor,
                         out: torch.Tensor, group=None):
    """Baseline of PeerEPDecode with a collective: every rank runs the decode
    kernel on its own experts, zeroes the outputs of picks it does not own,
    and an all_reduce (NCCL over NVLink) sums the k x d outputs -- each pick
    has exactly one non-zero contribution, so the sum is exact -- then the
    fixed-order combine.  Bit-identical to the single-GPU decode layer."""
    from . import _lib, ops
    m = model
    nxt = m.gate[layer + 1] if layer + 1 < m.shape.num_layers else None
    ops.decode_layer(h, m.norm[layer], m.gate[layer], nxt, m.fast[layer], m.slot_of[layer],
                     m.slab, m.slot_elems, m.d, m.ffn, m.shape.top_k, bufs)
    torch.mul(bufs.y, bufs.is_fast.view(-1, 1).to(torch.float32), out=y_sum)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y_sum, group=group)
    _lib.call("daop_combine_dense", h.data_ptr(), y_sum.data_ptr(), bufs.w.data_ptr(),
              m.shape.top_k, m.d, out.data_ptr(), ops._s())
    return out
