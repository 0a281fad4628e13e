"""Oracle (TEST INFRASTRUCTURE ONLY): restatement of the reference decision path.

Plain numpy / Python, deliberately written independently of the product code.
Citations are ``file:line`` into ``/root/reference/pkg/src/moesim``.
Placements are ``list[set[int]]`` (one set of GPU-resident experts per layer).
Plans are ``list`` of per-layer dicts ``{"executed": [(expert, device,
input_source, precalc), ...], "degraded": [(dropped, dscore, sub, sscore), ...]}``.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


class OracleError(Exception):
    """Raised where the reference raises a MoesimError; ``kind`` names the class."""

    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------- _kernels.py


def topk_rows(scores, k: int) -> np.ndarray:
    """_kernels.py:32-40 (numpy backend) == :63-79 (numba): stable argsort of
    -score, i.e. highest score first, ties to the lower index."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    order = np.argsort(-s, axis=-1, kind="stable")
    return order[:, :k].astype(np.int64)


def topk_scan(row, k: int) -> list[int]:
    """_kernels.py:63-79 literally: k passes of a strict '>' scan."""
    taken = [False] * len(row)
    out = []
    for _ in range(k):
        best = -1
        for c in range(len(row)):
            if taken[c]:
                continue
            if best < 0 or row[c] > row[best]:
                best = c
        out.append(best)
        taken[best] = True
    return out


def activation_counts(topk: np.ndarray, num_experts: int) -> np.ndarray:
    """_kernels.py:52-58: (T, L, k) ids -> (L, E) float64 counts."""
    t, l, _ = topk.shape
    out = np.zeros((l, num_experts), dtype=np.float64)
    layer_idx = np.broadcast_to(np.arange(l)[None, :, None], topk.shape)
    np.add.at(out, (layer_idx, topk), 1.0)
    return out


def pair_overlap(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """_kernels.py:43-49: per-row |a ∩ b| for rows of distinct ids."""
    hits = a[:, :, None] == b[:, None, :]
    return hits.any(axis=2).sum(axis=1).astype(np.int64)


# ----------------------------------------------------------------- metrics.py


def expert_counts(true_scores: np.ndarray, k: int) -> np.ndarray:
    """metrics.py:64-71 via _phase_topk :55-61: (T, L, E) true scores of one
    phase -> (L, E) int64 counts of true top-k membership."""
    t, l, e = true_scores.shape
    if t == 0:
        raise OracleError("EmptyPhaseError", "no tokens")
    top = topk_rows(true_scores.reshape(-1, e), k).reshape(t, l, k)
    return activation_counts(top, e).astype(np.int64)


def prediction_accuracy(decode_true: np.ndarray, decode_pred: np.ndarray, k: int):
    """metrics.py:120-143: entry l = mean over tokens of
    |topk(pred carried on l-1) ∩ topk(true l)| / k; entry 0 is NaN."""
    n, l, e = decode_true.shape
    out = np.full(l, np.nan)
    true_top = topk_rows(decode_true.reshape(-1, e), k).reshape(n, l, k)
    for layer in range(1, l):
        pred_top = topk_rows(decode_pred[:, layer - 1, :], k)
        out[layer] = pair_overlap(pred_top, true_top[:, layer, :]).mean() / k
    return out


def pooled_decode_probabilities(decode_true_list, k: int) -> np.ndarray:
    """experiment.py:132-142: summed decode counts / total decode tokens."""
    total = None
    tokens = 0
    for dt in decode_true_list:
        c = expert_counts(dt, k)
        total = c if total is None else total + c
        tokens += dt.shape[0]
    return total / tokens


# --------------------------------------------------------------- placement.py


def slot_budget_for_ecr(ecr: float, num_layers: int, num_experts: int) -> int:
    """placement.py:123-125: floor(ECR * L * E), evaluated left to right."""
    return math.floor(ecr * num_layers * num_experts)


def init_from_calibration(calib, ecr: float):
    """placement.py:128-185.  Returns (sets, budget)."""
    v = np.asarray(calib, dtype=np.float64)
    l, e = v.shape
    if not 0.0 < ecr <= 1.0:
        raise OracleError("BudgetError", f"ecr {ecr}")
    budget = slot_budget_for_ecr(ecr, l, e)
    if budget < l:
        raise OracleError("BudgetError", f"budget {budget} < {l}")
    base = budget // l
    rem = budget - base * l
    sets = []
    for layer in range(l):  # :167-169 per-layer top-`base` by (-v, j)
        order = sorted(range(e), key=lambda j: (-v[layer, j], j))
        sets.append(set(order[:base]))
    if rem:  # :171-183 global remainder, at most one extra per layer
        cands = sorted(
            ((i, j) for i in range(l) for j in range(e) if j not in sets[i]),
            key=lambda ij: (-v[ij[0], ij[1]], ij[0], ij[1]),
        )
        granted = set()
        for i, j in cands:
            if len(granted) == rem:
                break
            if i in granted:
                continue
            sets[i].add(j)
            granted.add(i)
    return sets, budget


def allocate_for_sequence(sets, counts, swap_in_out: float = 1.05):
    """placement.py:188-237 (Alg. 1).  Returns (new_sets, events) with events
    (layer, swapped_in, swapped_out, hot_tokens, cold_tokens)."""
    c = np.asarray(counts)
    if np.any(c < 0) or not np.all(c == np.floor(c)):
        raise OracleError("ShapeMismatchError", "counts")
    c = c.astype(np.int64)
    thr = Fraction(str(float(swap_in_out)))  # :211
    l, e = c.shape
    swap_num = e // 2  # :213
    new_sets, events = [], []
    for layer in range(l):
        cached = set(sets[layer])
        slow = [j for j in range(e) if j not in cached]
        fast = sorted(cached)
        act = c[layer]
        hot = sorted(slow, key=lambda j: (-act[j], j))[:swap_num]  # :221
        cold = sorted(fast, key=lambda j: (act[j], j))[:swap_num]  # :222
        for h, cc in zip(hot, cold):
            if Fraction(int(act[h])) >= thr * int(act[cc]):  # :224 inclusive
                cached.discard(cc)
                cached.add(h)
                events.append((layer, h, cc, int(act[h]), int(act[cc])))
        new_sets.append(cached)
    return new_sets, events


# ---------------------------------------------------------------- policies.py


def degrade_selection(scores, selection, fast):
    """policies.py:264-296."""
    fast = set(fast)
    sel = list(selection)
    deg = []
    while True:
        slow_sel = [x for x in sel if x not in fast]
        if len(slow_sel) < 2:
            break
        alts = [x for x in sorted(fast) if x not in sel]
        if not alts:
            break
        drop = min(slow_sel, key=lambda x: (scores[x], x))
        sub = max(alts, key=lambda x: (scores[x], -x))
        sel[sel.index(drop)] = sub
        deg.append((drop, float(scores[drop]), sub, float(scores[sub])))
    return sel, deg


def plan_token(true_le, pred_le, pred_mask, sets, k, engine="daop", start=4,
               degrade=True):
    """policies.py:248-261 (fiddler) and :299-336 (daop).

    true_le: (L, E) true scores; pred_le: (L, E) predicted scores carried on
    layer l for layer l+1; pred_mask: (L,) bool.
    """
    l_count = true_le.shape[0]
    top = topk_rows(true_le, k)
    plans = []
    for l in range(l_count):
        res = lambda e: "fast" if e in sets[l] else "slow"  # noqa: E731
        if engine == "fiddler" or l < start:
            plans.append({
                "executed": [(int(e), res(int(e)), "current", False) for e in top[l]],
                "degraded": [],
            })
            continue
        if not pred_mask[l - 1]:
            raise OracleError("PredictionMissingError", f"layer {l - 1}")
        s = pred_le[l - 1]
        sel = [int(x) for x in topk_rows(s[None, :], k)[0]]
        deg = []
        if degrade:
            sel, deg = degrade_selection(s, sel, sets[l])
        ex = []
        for e in sel:
            if res(e) == "slow":
                ex.append((e, "slow", "stale", True))
            else:
                ex.append((e, "fast", "current", False))
        plans.append({"executed": ex, "degraded": deg})
    return plans


class LruCaches:
    """policies.py:103-140 (_LayerCache / CacheState): one LRU cache per layer
    seeded with the placement's set (identical recency 0, capacity = size);
    one global step counter, ticked once per (token, layer)."""

    def __init__(self, sets):
        self.last_use = [{int(e): 0 for e in sorted(s)} for s in sets]
        self.capacity = [len(s) for s in sets]
        self.step = 0

    def insert(self, l, e, step):
        """policies.py:120-127: evict the least recently used (ties -> lower id)."""
        lu = self.last_use[l]
        if e not in lu and len(lu) >= self.capacity[l]:
            if not lu:
                raise OracleError("ConfigError", f"layer {l} cache has no capacity")
            ev = min(lu, key=lambda x: (lu[x], x))
            del lu[ev]
        lu[e] = step


def plan_token_lru(true_le, pred_le, pred_mask, caches: LruCaches, k, engine, start=4):
    """policies.py:173-194 (OnDemandPlanner) and :197-245 (PrefetchPlanner).

    Mutates ``caches`` like the reference planner (state persists across
    tokens; a PredictionMissingError leaves the updates already made)."""
    l_count = true_le.shape[0]
    top = topk_rows(true_le, k)
    plans = []
    for l in range(l_count):
        caches.step += 1
        step = caches.step
        lu = caches.last_use[l]
        need = [int(e) for e in top[l]]
        absent = sorted(e for e in need if e not in lu)
        for e in need:
            if e in lu:
                lu[e] = step
        for e in absent:
            caches.insert(l, e, step)
        issues = []
        if engine == "prefetch" and l + 1 < l_count and l + 1 >= start:
            if not pred_mask[l]:
                raise OracleError("PredictionMissingError", f"layer {l}")
            pred_top = [int(x) for x in topk_rows(pred_le[l][None, :], k)[0]]
            nlu = caches.last_use[l + 1]
            issues = sorted(e for e in pred_top if e not in nlu)
            for e in issues:
                caches.insert(l + 1, e, step)
        plans.append({"executed": [(e, "fast", "current", False) for e in need],
                      "migrations": absent, "prefetch_issues": issues, "degraded": []})
    return plans


def decode_counters(plans_per_token, engine="daop", start=4):
    """simulator.py:297-389 counter semantics: slow_executions = current slow
    picks + precalc picks; stale_inputs = precalc picks; degradations =
    len(plan.degraded); migrations = demand migrations; prefetches = early
    migrations, wasted when the expert is not executed at layer l+1."""
    c = {"migrations": 0, "prefetches": 0, "wasted_prefetches": 0,
         "slow_executions": 0, "degradations": 0, "stale_inputs": 0}
    for plans in plans_per_token:
        l_count = len(plans)
        for l, p in enumerate(plans):
            c["migrations"] += len(p.get("migrations", ()))
            for e in p.get("prefetch_issues", ()):
                c["prefetches"] += 1
                if e not in [x[0] for x in plans[l + 1]["executed"]]:
                    c["wasted_prefetches"] += 1
            cur_slow = [x for x in p["executed"] if x[1] == "slow" and not x[3]]
            c["slow_executions"] += len(cur_slow)
            # precalc for l+1 is dispatched at layer l when its pred-gate runs
            if engine == "daop" and l + 1 < l_count and l + 1 >= start:
                pre = [x for x in plans[l + 1]["executed"] if x[3]]
                c["slow_executions"] += len(pre)
                c["stale_inputs"] += len(pre)
            c["degradations"] += len(p["degraded"])
    return c
