// Decode MoE layer for one token: fused router + DAOP decision + HBM-streaming
// SwiGLU expert GEMV + combine, in ONE persistent launch with no grid barrier.
//
// Phase 0 (every CTA, redundant and bit-identical across CTAs)
//   mode 0 TRUE (l < start / fiddler): h, the E gate rows and (CTAs 0..E-1) one
//     next-layer gate row land in shared memory with ONE bulk copy at t=0;
//     x = bf16(rmsnorm(h) * gamma), p = softmax(x . Wg_l^T), selection =
//     top-k(p) (ties -> lower id, moesim/_kernels.py:63-79), then streaming.
//   mode 1 PLAN (DAOP l >= start): selection = top-k(pred_prev) + graceful
//     degradation over the layer's HBM residence (policies.py:299-336 via
//     decide.cuh) is known at t=0, so the weight stream starts immediately and
//     the router (needed only for the exported trace and the next prediction)
//     runs while the first weights are in flight.
//   CTAs 0..E-1 each compute one row of the next-layer gate from the same x
//   (PAPER.md:234); the last of them writes p_pred.
// Phase 1: unit = (pick j, ffn row i) = W1[i] + W3[i]; act[j, i] =
//   bf16(silu(W1 x) * (W3 x)).  Units are dealt to CTAs round-robin (u = cta +
//   m * G) and to the CTA's warps dynamically (shared-memory ticket), so each
//   pick's activations complete early and evenly across the grid.
// Phase 2: the CTA owns a contiguous block of output rows; its pieces
//   (pick j, row r, K-chunk c) are dealt to its warps dynamically, partial dot
//   products are reduced in shared memory by the last arriving warp in fixed
//   (j, c) order (deterministic), which writes y[q, r] and
//   h'[r] = h[r] + sum_q w_q y[q, r].
// The only grid-wide dependency is "all rows of pick j done" before a CTA
// pulls act_j into shared memory (one counter per pick, one bulk copy per CTA
// per pick) -- the weight rings never drain at the phase boundary.
//
// Each warp streams its weight pieces through its own cp.async.bulk ring
// (DS stages x DSB bytes, L2 evict_first).  Bytes per call (Mixtral-8x7B,
// 2 resident picks): 2 x 3 x 4096 x 14336 x 2 B of weights + 2 x 8 x 4096 x
// 2 B of gates = 704,774,144 B -> HBM roofline.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "decide.cuh"
#include "ep.cuh"

namespace daop {

constexpr int DK_MAX = 8;       // max top-k
constexpr int DE_MAX = 16;      // max experts (router logits live on lanes)
constexpr int DE_FAST = DE_MAX;
constexpr int kMaxChunks = 16;  // max W2 row pieces

struct DecodeArgs {
  const float* h;          // (d) fp32 residual in
  const uint16_t* gamma;   // (d) RMSNorm weight
  const uint16_t* wg;      // (E, d) gate of this layer
  const uint16_t* wg_next; // (E, d) gate of layer l+1 or null
  const float* pred_prev;  // (E) prediction carried on layer l-1 (PLAN mode)
  const uint8_t* fast_row; // (E) residence of this layer's experts
  const int32_t* slot_of;  // (E) HBM slot of expert e (valid where fast)
  const uint16_t* slab;    // expert slot slab
  int64_t slot_stride;     // elements per slot: [W1 | W3 | W2]
  int d, ffn, E, k;
  int mode;                // 0 TRUE, 1 PLAN
  int graceful;
  int weights_from_pred;   // combine weights from pred_prev (PLAN) instead of p
  float eps;
  int rows_per_cta;        // phase-2 output rows per CTA (host computed)
  uint16_t* x_out;         // (d) bf16 normalised input (stale input for layer l+1)
  float* p_true;           // (E)
  float* p_pred;           // (E) or null
  int32_t* sel;            // (k)
  float* w;                // (k)
  uint8_t* is_fast;        // (k)
  int32_t* deg;            // (2k + 1): drop[k] | sub[k] | count
  float* y;                // (k, d) per-pick expert outputs
  float* h_out;            // (d) combined residual (written when every pick is fast)
  // self-resetting workspace (zeroed once by the caller)
  unsigned* ctr;           // [0] finished CTAs, [1] pred rows, [2..2+DK_MAX) rows per pick
  float* pred_logits;      // (E)
  uint16_t* act;           // (k, ffn) bf16 SwiGLU activations
  // expert-parallel decode (ep_p2p.cu): the y rows of this GPU's picks are
  // also stored into slot [ep_epoch & 1] of every peer's decode workspace,
  // and the grid's last CTA flags them (null = single GPU)
  const uint64_t* ep_peers;
  int ep_G, ep_rank;
  unsigned ep_epoch;
  // persistent decode server (daop_server_*): the grid's last CTA publishes
  // host_seq into this pinned host word once h_out / sel are in host memory
  unsigned* host_done;
  unsigned host_seq;
  // PLAN mode launched programmatically behind the attention O-proj: the
  // predicted experts' weight stream starts before griddepcontrol.wait (the
  // plan reads only the previous MoE kernel's prediction, complete once an
  // O-proj CTA of this layer has left the SM); h is read after the wait
  int early;
  float* host_out;         // pinned host copies of h_out / sel (server mode)
  int32_t* host_sel;
  // server mode: every CTA ships its own h_out rows to host_out with one bulk
  // store as it finishes (rows_per_cta % 4 == 0: 16-byte pieces) instead of
  // the grid's last warp pulling all d rows back from HBM and pushing them
  int ship_cta;
};

__device__ unsigned long long g_decode_timeline[1024][16];
__device__ int g_decode_timeline_on;

// SM cycle counter (per-SM; phases are compared within one CTA).  %globaltimer
// was too coarse to resolve the sub-microsecond phase-0 steps.
__device__ __forceinline__ unsigned long long gtimer() { return clock64(); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Piece {   // what one ring stage holds
  int kind;      // 1 = W1/W3 piece, 2 = W2 piece, 0 = end of stream
  int j, row, c; // pick (executed index), row, piece within the unit
};
__device__ __forceinline__ uint32_t pack_piece(const Piece& p) {
  return static_cast<uint32_t>(p.kind) | (static_cast<uint32_t>(p.j) << 2) |
         (static_cast<uint32_t>(p.c) << 6) | (static_cast<uint32_t>(p.row) << 14);
}
__device__ __forceinline__ Piece unpack_piece(uint32_t v) {
  Piece p;
  p.kind = static_cast<int>(v & 3u);
  p.j = static_cast<int>((v >> 2) & 15u);
  p.c = static_cast<int>((v >> 6) & 255u);
  p.row = static_cast<int>(v >> 14);
  return p;
}

template <int DW, int DS>
struct DecodeSmem {
  uint64_t bar[DW][DS];
  uint64_t act_bar[DK_MAX];
  uint64_t in_bar;   // h + gamma
  uint64_t in_bar2;  // gate rows (+ next-layer row)
  uint32_t rec[DW][DS];
  int act_req[DK_MAX];
  int p1_next, p2_next, fin;
  int done1[DK_MAX];
  double red[DW];         // per-warp sums of squares (fp64, common.cuh rms_scale)
  float zpart[DW][DE_MAX];  // per-warp partial gate logits
  float zpp[DW];            // per-warp partial next-layer logit
  float p[DE_MAX];
  float pp[DE_MAX];
  int slot[DE_MAX];
  uint8_t fast_row[DE_MAX];
  float wsel[DK_MAX];
  int sel[DK_MAX];
  int exec_q[DK_MAX];
  uint8_t fast[DK_MAX];
  int n_exec, nd, drop[DK_MAX], sub[DK_MAX];
  int pred_last;
  const uint16_t* base[DK_MAX];  // slab slot base of each executed pick
};

struct Layout {
  // slot base per executed pick, in SHARED memory: a register array indexed by
  // the pick would be demoted to local memory, and with ~225 KB of smem the L1
  // is nearly gone, so every local access would be an L2 round trip
  const uint16_t* const* base;
  int n_exec, d, ffn, G, cta;
  int npc1, pe1, npc2, pe2;
  int n1c;         // phase-1 units of this CTA
  int r0, R, P2c;  // phase-2 rows [r0, r0+R) and pieces of this CTA
};

__device__ __forceinline__ const uint16_t* piece_src(const Layout& L, const Piece& pc, int& elems,
                                                     int& voff) {
  if (pc.kind == 1) {
    const int which = pc.c >= L.npc1;
    const int c = pc.c - which * L.npc1;
    voff = c * L.pe1;
    elems = min(L.pe1, L.d - voff);
    return L.base[pc.j] + (static_cast<int64_t>(which) * L.ffn + pc.row) * L.d + voff;
  }
  voff = pc.c * L.pe2;
  elems = min(L.pe2, L.ffn - voff);
  return L.base[pc.j] + 2ll * L.ffn * L.d + static_cast<int64_t>(pc.row) * L.ffn + voff;
}

__device__ __forceinline__ float dot_piece(const uint4* wp, const uint4* vp, int n16, int lane,
                                           float acc) {
#pragma unroll 4
  for (int c = lane; c < n16; c += 32) acc = dot8(wp[c], vp[c], acc);
  return acc;
}

// number of u in [lo, hi) with u = cta (mod G)
__device__ __forceinline__ int count_mod(int lo, int hi, int cta, int G) {
  const int f = lo + ((cta - lo) % G + G) % G;
  return hi > f ? (hi - 1 - f) / G + 1 : 0;
}

__device__ __forceinline__ int degrade_smem(const float* s, int E, int* sel, int k,
                                         const uint8_t* fast, int* drop, int* sub) {
  return degrade(s, E, sel, k, fast, drop, sub);
}

template <int DW, int DS, int DSB>
__device__ __forceinline__ void decode_body(const DecodeArgs a) {
  constexpr int NT = DW * 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const int d = a.d, E = a.E, k = a.k;
  uint8_t* ring = smem;                                                  // DW*DS*DSB
  uint16_t* act_s = reinterpret_cast<uint16_t*>(smem + DW * DS * DSB);  // k*ffn
  uint16_t* x_s = act_s + static_cast<size_t>(k) * a.ffn;               // d
  float* part = reinterpret_cast<float*>(
      reinterpret_cast<uint8_t*>(x_s) + ((static_cast<size_t>(d) * 2 + 127) / 128) * 128);
  const int npc2_max = (a.ffn * 2 + DSB - 1) / DSB;
  int* rcnt = reinterpret_cast<int*>(part + a.rows_per_cta * k * npc2_max);
  auto& s = *reinterpret_cast<DecodeSmem<DW, DS>*>(
      reinterpret_cast<uint8_t*>(rcnt) + ((a.rows_per_cta * 4 + 127) / 128) * 128);
  float* hout_s = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(&s) +
                                           (sizeof(DecodeSmem<DW, DS>) + 15) / 16 * 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tl = g_decode_timeline_on != 0 && blockIdx.x < 1024;
  const bool pred_row = a.wg_next && blockIdx.x < static_cast<unsigned>(E);
  bool wrote_out = false;  // this thread stored part of the result (host memory in server mode)

  // staging of the router inputs in the (still idle) ring area, mode 0 only
  float* h_s = reinterpret_cast<float*>(ring);
  uint16_t* gm_s = reinterpret_cast<uint16_t*>(ring + d * 4);
  uint16_t* g_s = gm_s + d;
  uint16_t* gp_s = g_s + static_cast<size_t>(E) * d;

  if (threadIdx.x == 0) {
    if (tl) {
      g_decode_timeline[blockIdx.x][0] = gtimer();
      g_decode_timeline[blockIdx.x][12] = globaltimer_ns();  // (global clock: cross-kernel spans)
    }
    for (int w = 0; w < DW; ++w)
      for (int q = 0; q < DS; ++q) mbar_init(&s.bar[w][q], 1);
    for (int q = 0; q < DK_MAX; ++q) {
      mbar_init(&s.act_bar[q], 1);
      s.act_req[q] = 0;
      s.done1[q] = 0;
    }
    mbar_init(&s.in_bar, 1);
    mbar_init(&s.in_bar2, 1);
    s.p1_next = DW;  // tickets 0..DW-1 are taken statically by the warps' first units
    s.p2_next = s.fin = 0;
    *reinterpret_cast<int*>(&s.zpart[1][0]) = 0;  // lazy-gates counter (zpart unused then)
    fence_mbar_init();
    if (a.mode == 0) {  // h + gamma (RMSNorm starts on them), then the gate rows
      // server mode: h was just written by block 0 with generic stores and
      // handed over through an acquire; it is read with generic loads below
      const bool h_bulk = a.host_seq == 0;
      mbar_arrive_expect_tx(&s.in_bar, (h_bulk ? d * 4 : 0) + d * 2);
      if (h_bulk) bulk_g2s_plain(h_s, a.h, d * 4, &s.in_bar);
      bulk_g2s_plain(gm_s, a.gamma, d * 2, &s.in_bar);
      mbar_arrive_expect_tx(&s.in_bar2, E * d * 2 + (pred_row ? d * 2 : 0));
      bulk_g2s_plain(g_s, a.wg, E * d * 2, &s.in_bar2);
      if (pred_row)
        bulk_g2s_plain(gp_s, a.wg_next + static_cast<size_t>(blockIdx.x) * d, d * 2, &s.in_bar2);
    }
  }
  if (warp == 1) {
    for (int e = lane; e < E; e += 32) {
      s.fast_row[e] = a.fast_row[e];
      s.slot[e] = a.slot_of[e];
      s.pp[e] = a.pred_prev ? a.pred_prev[e] : 0.f;
    }
  }
  for (int i = threadIdx.x; i < a.rows_per_cta; i += NT) rcnt[i] = 0;
  __syncthreads();

  Layout L;
  L.d = d;
  L.ffn = a.ffn;
  L.G = gridDim.x;
  L.cta = blockIdx.x;
  L.npc1 = (d * 2 + DSB - 1) / DSB;
  L.pe1 = (((d + L.npc1 - 1) / L.npc1) + 7) / 8 * 8;
  L.npc2 = npc2_max;
  L.pe2 = (((a.ffn + L.npc2 - 1) / L.npc2) + 7) / 8 * 8;
  L.r0 = min(d, static_cast<int>(blockIdx.x) * a.rows_per_cta);
  L.R = min(d, L.r0 + a.rows_per_cta) - L.r0;

  // ---- selection helpers (warp 0)
  // lane-parallel (lane q = pick q): residence, compaction of the resident
  // picks in pick order, weights w_q = wsrc[sel_q] / sum_q' wsrc[sel_q']
  // (summed in pick order, like the reference renormalisation)
  auto finish_selection = [&](const float* wsrc) {
    __syncwarp();
    int e = 0, slot = 0;
    bool f = false;
    if (lane < k) {
      e = s.sel[lane];
      f = s.fast_row[e] != 0;
      slot = s.slot[e];
    }
    const unsigned fm = __ballot_sync(0xffffffffu, lane < k && f);
    if (lane < k) {
      s.fast[lane] = f ? 1 : 0;
      if (f) {
        const int pos = __popc(fm & ((1u << lane) - 1u));
        s.base[pos] = a.slab + static_cast<int64_t>(slot) * a.slot_stride;
        s.exec_q[pos] = lane;
      }
    }
    if (lane == 0) s.n_exec = __popc(fm);
    if (wsrc) {
      const float v = lane < k ? wsrc[e] : 0.f;
      float den = 0.f;
      for (int q = 0; q < k; ++q) den += __shfl_sync(0xffffffffu, v, q);
      if (lane < k) s.wsel[lane] = v / den;
    }
    __syncwarp();
  };

  // ---- streaming machinery (warp-uniform state)
  uint8_t* my_ring = ring + warp * DS * DSB;
  const uint64_t pol = l2_evict_first_policy();
  int issued = 0, iss_phase = 1, iss_u = 0, iss_q = 0;
  bool have_unit = false;
  bool first_ticket = true;  // the first phase-1 ticket is the warp index (no smem atomic)
  auto next_piece = [&](Piece& pc) {
    pc.kind = 0;
    if (iss_phase == 1) {
      if (!have_unit) {
        int m = 0;
        if (lane == 0) m = first_ticket ? warp : atomicAdd(&s.p1_next, 1);
        first_ticket = false;
        m = __shfl_sync(0xffffffffu, m, 0);
        if (m < L.n1c) {
          iss_u = L.cta + m * L.G;
          iss_q = 0;
          have_unit = true;
        } else {
          iss_phase = 2;
        }
      }
      if (have_unit) {
        pc.kind = 1;
        pc.j = iss_u / L.ffn;
        pc.row = iss_u - pc.j * L.ffn;
        pc.c = iss_q;
        if (++iss_q == 2 * L.npc1) have_unit = false;
        return;
      }
    }
    if (iss_phase == 2) {
      int v = 0;
      if (lane == 0) v = atomicAdd(&s.p2_next, 1);
      v = __shfl_sync(0xffffffffu, v, 0);
      if (v >= L.P2c) {
        iss_phase = 3;
        return;
      }
      const int per_j = L.R * L.npc2;
      pc.kind = 2;
      pc.j = v / per_j;
      const int rem = v - pc.j * per_j;
      const int rr = rem / L.npc2;
      pc.c = rem - rr * L.npc2;
      pc.row = L.r0 + rr;
    }
  };
  auto issue_next = [&]() {
    Piece pc;
    next_piece(pc);
    const int stg = issued % DS;
    if (lane == 0) {
      s.rec[warp][stg] = pack_piece(pc);
      if (pc.kind) {
        int elems, voff;
        const uint16_t* src = piece_src(L, pc, elems, voff);
        mbar_arrive_expect_tx(&s.bar[warp][stg], elems * 2);
        bulk_g2s(my_ring + stg * DSB, src, elems * 2, &s.bar[warp][stg], pol);
      }
    }
    ++issued;
  };
  auto start_stream = [&]() {
    L.n_exec = s.n_exec;
    L.base = s.base;
    L.n1c = count_mod(0, L.n_exec * a.ffn, L.cta, L.G);
    L.P2c = L.n_exec * L.R * L.npc2;
    for (int q = 0; q < DS; ++q) issue_next();
  };


  // ---- lane-parallel softmax / top-k over E <= 16 experts: shuffles span only
  // the next power of two >= E; ties resolve to the lower id (topk_scan order)
  int P2 = 1;
  while (P2 < E) P2 <<= 1;
  auto lane_softmax = [&](float z) {
    float m = lane < E ? z : -INFINITY;
    for (int o = P2 >> 1; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e = lane < E ? expf(z - m) : 0.f;
    float sum = e;
    for (int o = P2 >> 1; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    return lane < E ? e / sum : 0.f;
  };
  auto lane_topk = [&](float v) {  // -> s.sel[0..k)
    bool taken = lane >= E;
    for (int j = 0; j < k; ++j) {
      float bv = taken ? -INFINITY : v;
      int bi = taken ? 0x7fffffff : lane;
      for (int o = P2 >> 1; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      bi = __shfl_sync(0xffffffffu, bi, 0);
      // NaN scores never compare: fall back to the first untaken id
      // (topk_scan's "best < 0" rule), never an out-of-range id
      if (bi >= E) bi = __ffs(__ballot_sync(0xffffffffu, !taken)) - 1;
      if (lane == 0) s.sel[j] = bi;
      if (lane == bi) taken = true;
    }
    __syncwarp();
  };

  double ss = 0.0;
  if (a.mode == 1) {
    // ---------------------------------------------------- PLAN: stream first
    if (warp == 0) {
      lane_topk(lane < E ? s.pp[lane] : 0.f);
      if (lane == 0) s.nd = a.graceful ? degrade_smem(s.pp, E, s.sel, k, s.fast_row, s.drop, s.sub) : 0;
      __syncwarp();
      finish_selection(a.weights_from_pred ? s.pp : nullptr);
    }
    __syncthreads();
    start_stream();
    if (a.early) asm volatile("griddepcontrol.wait;" ::: "memory");  // h: the O-proj's output
    for (int i = threadIdx.x; i < d / 4; i += NT)  // router inputs from global
      ss = sq_acc4(reinterpret_cast<const float4*>(a.h)[i], ss);
  } else {
    // ---------------------------------------------------- TRUE: router first
    if (a.host_seq != 0) {  // server mode: generic loads of h (each thread the elements it sums)
      for (int i = threadIdx.x; i < d / 4; i += NT) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(a.h) + i);
        reinterpret_cast<float4*>(h_s)[i] = v;
        ss = sq_acc4(v, ss);
      }
      mbar_wait(&s.in_bar, 0);  // gamma
    } else {
      mbar_wait(&s.in_bar, 0);
      for (int i = threadIdx.x; i < d / 4; i += NT)
        ss = sq_acc4(reinterpret_cast<const float4*>(h_s)[i], ss);
    }
  }
  ss = warp_sum(ss);
  if (lane == 0) s.red[warp] = ss;
  __syncthreads();
  if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][5] = gtimer();
  // ---- one fused pass: x = bf16(h * r * gamma) for this warp's slice of d,
  // and the slice's partial dot products with the E gate rows (+ this CTA's
  // next-layer gate row); partials are summed over warps in fixed order
  const bool mode0 = a.mode == 0;
  // PLAN mode with prediction weights: the selection and the weights are
  // known, so the gate logits are off the critical path -- only CTA 0 (the
  // exported p_true) and the CTAs owning a next-layer row compute them, after
  // x, from L2, while the other warps already consume the weight stream
  const bool lazy_gates = a.mode == 1 && a.weights_from_pred;
  const int n16 = d / 8;
  {
    double tot = 0.0;
    for (int w = 0; w < DW; ++w) tot += s.red[w];
    const float r = rms_scale(tot, d, a.eps);
    const float4* hsrc = reinterpret_cast<const float4*>(mode0 ? h_s : a.h);
    const uint4* gmsrc = reinterpret_cast<const uint4*>(mode0 ? gm_s : a.gamma);
    const uint16_t* gsrc = mode0 ? g_s : a.wg;
    const uint4* gpsrc = reinterpret_cast<const uint4*>(
        mode0 ? gp_s : (pred_row ? a.wg_next + static_cast<size_t>(blockIdx.x) * d : a.wg));
    const int cpw = (n16 + DW - 1) / DW;
    const int c1 = min(n16, (warp + 1) * cpw);
    // x for this warp's chunks first (h + gamma have landed; the gate rows
    // may still be in flight)
    for (int c = warp * cpw + lane; c < c1; c += 32) {
      const float4 u = hsrc[2 * c], v = hsrc[2 * c + 1];
      const uint4 gm = gmsrc[c];
      const uint32_t x0 = static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(u.x, r), bf16lo(gm.x)))) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(u.y, r), bf16hi(gm.x)))) << 16);
      const uint32_t x1 = static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(u.z, r), bf16lo(gm.y)))) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(u.w, r), bf16hi(gm.y)))) << 16);
      const uint32_t x2 = static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(v.x, r), bf16lo(gm.z)))) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(v.y, r), bf16hi(gm.z)))) << 16);
      const uint32_t x3 = static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(v.z, r), bf16lo(gm.w)))) |
                          (static_cast<uint32_t>(f32_to_bf16_bits(__fmul_rn(__fmul_rn(v.w, r), bf16hi(gm.w)))) << 16);
      reinterpret_cast<uint4*>(x_s)[c] = make_uint4(x0, x1, x2, x3);
    }
    if (mode0) mbar_wait(&s.in_bar2, 0);
    if (!lazy_gates) {
    // partial logits: 16 slots = the E <= 16 gate rows, the next-layer row in
    // slot 15 when E < 16 (else reduced separately)
    float v16[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v16[e] = 0.f;
    float accp = 0.f;
    const bool pred_in_slot = pred_row && E < 16;
    for (int c = warp * cpw + lane; c < c1; c += 32) {
      const uint4 x8 = reinterpret_cast<const uint4*>(x_s)[c];
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (e < E) v16[e] = dot8(x8, reinterpret_cast<const uint4*>(gsrc + static_cast<size_t>(e) * d)[c], v16[e]);
      if (pred_row) accp = dot8(x8, gpsrc[c], accp);
    }
    if (pred_in_slot) v16[15] = accp;
    // reduce-scatter over the warp: 8 + 4 + 2 + 1 + 1 shuffles leave the warp
    // sum of slot (lane >> 1) on lanes 2i and 2i+1
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool hi = lane & 16;
      const float send = hi ? v16[i] : v16[i + 8];
      const float keep = hi ? v16[i + 8] : v16[i];
      v16[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool hi = lane & 8;
      const float send = hi ? v16[i] : v16[i + 4];
      const float keep = hi ? v16[i + 4] : v16[i];
      v16[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool hi = lane & 4;
      const float send = hi ? v16[i] : v16[i + 2];
      const float keep = hi ? v16[i + 2] : v16[i];
      v16[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {
      const bool hi = lane & 2;
      const float send = hi ? v16[0] : v16[1];
      const float keep = hi ? v16[1] : v16[0];
      v16[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      v16[0] += __shfl_xor_sync(0xffffffffu, v16[0], 1);
    }
    const int slot16 = lane >> 1;
    if ((lane & 1) == 0) {
      if (slot16 < E) s.zpart[warp][slot16] = v16[0];
      if (pred_in_slot && slot16 == 15) s.zpp[warp] = v16[0];
    }
    if (pred_row && !pred_in_slot) {
      const float zz = warp_sum(accp);
      if (lane == 0) s.zpp[warp] = zz;
    }
    }  // !lazy_gates
  }
  __syncthreads();  // x complete in smem, partial logits visible
  if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][6] = gtimer();
  if (lazy_gates && blockIdx.x == 0 && warp < E) {
    // zpart is not used in this mode: row 0 holds the logits, [1][0] the count
    float* zfull = s.zpart[0];
    int* zdone = reinterpret_cast<int*>(&s.zpart[1][0]);
    // warp e: logit e over the full d (fixed lane-strided order + warp sum)
    const float z = warp_sum(dot_piece(reinterpret_cast<const uint4*>(a.wg + static_cast<size_t>(warp) * d),
                                       reinterpret_cast<const uint4*>(x_s), n16, lane, 0.f));
    if (lane == 0) {
      zfull[warp] = z;
      __threadfence_block();
      atomicAdd(zdone, 1);
    }
    if (warp == 0) {
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(zdone) < E) {
        }
      __syncwarp();
      __threadfence_block();
      const float p = lane_softmax(lane < E ? zfull[lane] : 0.f);
      if (lane < E) s.p[lane] = p;
      __syncwarp();
    }
  }
  // ---- every warp: logits (fixed warp order) -> softmax -> selection -> stream
  if (!lazy_gates) {
    float z = 0.f;
    if (lane < E)
      for (int w = 0; w < DW; ++w) z += s.zpart[w][lane];
    if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][7] = gtimer();
    const float p = lane_softmax(z);
    if (lane < E) s.p[lane] = p;  // identical values from every warp
    if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][9] = gtimer();
    if (mode0) {
      lane_topk(p);
      if (lane == 0) s.nd = 0;
      __syncwarp();
      if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][10] = gtimer();
      finish_selection(s.p);
      if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][11] = gtimer();
      start_stream();
    } else if (!a.weights_from_pred) {
      finish_selection(s.p);
    }
  }
  if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][8] = gtimer();
  if (pred_row && warp == DW - 1) {  // this CTA's next-layer row -> grid-wide p_pred
    float zl = 0.f;
    if (lazy_gates)
      zl = warp_sum(dot_piece(reinterpret_cast<const uint4*>(a.wg_next + static_cast<size_t>(blockIdx.x) * d),
                              reinterpret_cast<const uint4*>(x_s), n16, lane, 0.f));
    if (lane == 0) {
      float zp = zl;
      if (!lazy_gates)
        for (int w = 0; w < DW; ++w) zp += s.zpp[w];
      a.pred_logits[blockIdx.x] = zp;
      __threadfence();
      s.pred_last = atomicAdd(a.ctr + 1, 1u) == static_cast<unsigned>(E) - 1;
    }
    __syncwarp();
    if (s.pred_last) {  // the grid's last next-layer row: softmax -> p_pred
      __threadfence();
      const float pv = lane_softmax(lane < E ? __ldcg(a.pred_logits + lane) : 0.f);
      if (lane < E) a.p_pred[lane] = pv;
      if (lane == 0) a.ctr[1] = 0;
    }
  }
  if (blockIdx.x == 0) {
    if (warp == 0) {
      if (lane < E) a.p_true[lane] = s.p[lane];
      if (lane < k) {
        a.sel[lane] = s.sel[lane];
        wrote_out = true;
        a.w[lane] = s.wsel[lane];
        a.is_fast[lane] = s.fast[lane];
        a.deg[lane] = lane < s.nd ? s.drop[lane] : -1;
        a.deg[k + lane] = lane < s.nd ? s.sub[lane] : -1;
      }
      if (lane == 0) a.deg[2 * k] = s.nd;
    }
    if (a.x_out)
      for (int i = threadIdx.x; i < n16; i += NT)
        reinterpret_cast<uint4*>(a.x_out)[i] = reinterpret_cast<const uint4*>(x_s)[i];
  }
  if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][1] = gtimer();

  // ---------------------------------------------------------------- stream
  const bool all_fast = L.n_exec == k;
  const int row_target = L.n_exec * L.npc2;
  float acc0 = 0.f, acc1 = 0.f;
  int cur_j = -1, cur_cnt = 0;  // phase-1 units finished for the current pick
  auto publish = [&]() {        // CTA-aggregated per-pick completion
    if (cur_j >= 0 && cur_cnt > 0 && lane == 0) {
      __threadfence();          // this warp's act rows -> visible GPU-wide
      const int tot_j = count_mod(cur_j * a.ffn, (cur_j + 1) * a.ffn, L.cta, L.G);
      if (atomicAdd(&s.done1[cur_j], cur_cnt) + cur_cnt == tot_j) {
        // cumulativity: the other warps' act rows this warp observed through
        // done1 are ordered before the grid-wide count a consumer CTA waits on
        __threadfence();
        atomicAdd(a.ctr + 2 + cur_j, static_cast<unsigned>(tot_j));
      }
    }
    cur_cnt = 0;
  };
  bool in_p2 = false;
  for (int p = 0;; ++p) {
    const int stg = p % DS;
    __syncwarp();
    const Piece pc = unpack_piece(s.rec[warp][stg]);
    if (pc.kind == 0) break;
    int elems, voff;
    piece_src(L, pc, elems, voff);
    if (pc.kind == 2) {
      if (!in_p2) {
        in_p2 = true;
        publish();
        if (tl && threadIdx.x == 0) g_decode_timeline[blockIdx.x][2] = gtimer();
      }
      if (lane == 0 && atomicCAS(&s.act_req[pc.j], 0, 1) == 0) {
        // first use of pick j in this CTA: wait for its rows, pull act_j in
        const unsigned* cnt = a.ctr + 2 + pc.j;
        while (ld_acquire_gpu(cnt) < static_cast<unsigned>(a.ffn)) __nanosleep(64);
        if (tl && pc.j == 0) g_decode_timeline[blockIdx.x][3] = gtimer();
        asm volatile("fence.proxy.async;" ::: "memory");
        mbar_arrive_expect_tx(&s.act_bar[pc.j], a.ffn * 2);
        bulk_g2s_plain(act_s + static_cast<size_t>(pc.j) * a.ffn,
                       a.act + static_cast<size_t>(s.exec_q[pc.j]) * a.ffn, a.ffn * 2,
                       &s.act_bar[pc.j]);
      }
      mbar_wait(&s.act_bar[pc.j], 0);
    }
    mbar_wait(&s.bar[warp][stg], static_cast<uint32_t>((p / DS) & 1));
    const uint4* wp = reinterpret_cast<const uint4*>(my_ring + stg * DSB);
    if (pc.kind == 1) {
      const float v = dot_piece(wp, reinterpret_cast<const uint4*>(x_s + voff), elems / 8, lane, 0.f);
      if (pc.c < L.npc1) acc0 += v; else acc1 += v;
      __syncwarp();
      issue_next();  // refill the stage just drained
      if (pc.c == 2 * L.npc1 - 1) {  // (W1 row, W3 row) pair complete
        const float g = warp_sum(acc0), u = warp_sum(acc1);
        acc0 = acc1 = 0.f;
        if (lane == 0)
          a.act[static_cast<int64_t>(s.exec_q[pc.j]) * a.ffn + pc.row] =
              f32_to_bf16_bits(silu_f32(g) * u);
        if (pc.j != cur_j) {
          publish();
          cur_j = pc.j;
        }
        ++cur_cnt;
      }
    } else {
      const float v = warp_sum(dot_piece(
          wp, reinterpret_cast<const uint4*>(act_s + static_cast<size_t>(pc.j) * a.ffn + voff),
          elems / 8, lane, 0.f));
      __syncwarp();
      issue_next();
      if (lane == 0) {
        const int rr = pc.row - L.r0;
        float* pr = part + static_cast<size_t>(rr) * k * L.npc2;
        pr[pc.j * L.npc2 + pc.c] = v;
        __threadfence_block();
        if (atomicAdd(&rcnt[rr], 1) == row_target - 1) {  // last piece of row: reduce
          __threadfence_block();
          float o = a.h[pc.row];
          for (int jj = 0; jj < L.n_exec; ++jj) {
            float yv = 0.f;
            for (int c = 0; c < L.npc2; ++c) yv += pr[jj * L.npc2 + c];
            a.y[static_cast<int64_t>(s.exec_q[jj]) * d + pc.row] = yv;
            o = fmaf(s.wsel[s.exec_q[jj]], yv, o);
          }
          if (all_fast) {
            a.h_out[pc.row] = o;
            if (a.ship_cta) hout_s[rr] = o;
            wrote_out = true;
          }
        }
      }
    }
  }
  publish();
  // decode server: this thread's result stores (h_out rows, the selection, in
  // HBM) are visible to the grid's last warp, which ships them to the host
  if (a.host_done && wrote_out) __threadfence();
  int cta_done = 0;
  if (lane == 0) {
    if (tl) {
      atomicMax(&g_decode_timeline[blockIdx.x][4], gtimer());
      atomicMax(&g_decode_timeline[blockIdx.x][13], globaltimer_ns());  // (the CTA's last warp)
    }
    if (a.ep_peers || a.ship_cta) __threadfence_block();  // y rows / hout_s -> the CTA finisher
    cta_done = atomicAdd(&s.fin, 1) == DW - 1;      // CTA done
  }
  cta_done = __shfl_sync(0xffffffffu, cta_done, 0);
  if (cta_done && a.ship_cta && all_fast && lane == 0 && L.R > 0) {
    // decode server: this CTA's rows leave for pinned host memory now
    __threadfence_block();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // hout_s: generic -> bulk
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
        "cp.async.bulk.commit_group;\n\t"
        "cp.async.bulk.wait_group 0;" ::"l"(a.host_out + L.r0), "r"(smem_u32(hout_s)), "r"(L.R * 4)
        : "memory");
  }
  if (cta_done && a.ep_peers) {
    // expert parallelism: the finishing warp stores this CTA's block of y
    // rows (every executed pick) into slot [epoch & 1] of every peer's
    // decode workspace; one system fence before the grid-done count
    __threadfence_block();
    const int r1 = min(L.r0 + a.rows_per_cta, d);
    for (int jj = 0; jj < L.n_exec; ++jj) {
      const int q0 = s.exec_q[jj];
      const float* src = a.y + static_cast<int64_t>(q0) * d;
      for (int r = L.r0 + lane; r < r1; r += 32) {
        const float v = __ldcg(src + r);
        for (int g = 0; g < a.ep_G; ++g)
          (reinterpret_cast<float*>(a.ep_peers[g] + EP_DEC_Y) +
           (static_cast<int64_t>(a.ep_epoch & 1) * k + q0) * d)[r] = v;
      }
    }
    __threadfence_system();
    __syncwarp();
  }
  int grid_done = 0;
  if (lane == 0 && cta_done) {
    __threadfence();  // the CTA's result rows (other warps' stores + fences) before the count
    grid_done = atomicAdd(a.ctr, 1u) == gridDim.x - 1;
  }
  grid_done = __shfl_sync(0xffffffffu, grid_done, 0);
  if (grid_done) {  // the grid's last warp: reset for the next call, publish
    if (lane == 0) {
      for (int q = 0; q < DK_MAX; ++q) a.ctr[2 + q] = 0;
      a.ctr[0] = 0;
      if (a.ep_peers) {                           // every peer: this GPU's picks landed
        __threadfence_system();
        for (int q = 0; q < a.ep_G; ++q)
          st_release_sys(reinterpret_cast<unsigned*>(a.ep_peers[q] + EP_FLAGS_D) + a.ep_rank,
                         a.ep_epoch);
      }
    }
    if (a.host_done) {
      // decode server: the result (written to HBM by every CTA) leaves for
      // pinned host memory in 16-byte stores from this one warp -- a few
      // hundred large PCIe writes instead of d scattered 4-byte ones
      // (two bulk DMAs through this CTA's now idle ring: HBM -> smem -> host)
      __threadfence();
      if (lane == 0) {
        if (a.host_out && all_fast && !a.ship_cta) {
          uint64_t* bar = &s.bar[0][0];  // re-armed below for the next call's init
          mbar_init(bar, 1);
          fence_mbar_init();
          asm volatile("fence.proxy.async.global;" ::: "memory");  // h_out rows: generic -> bulk
          mbar_arrive_expect_tx(bar, d * 4);
          bulk_g2s_plain(ring, a.h_out, d * 4, bar);
          mbar_wait(bar, 0);
          asm volatile(
              "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
              "cp.async.bulk.commit_group;\n\t"
              "cp.async.bulk.wait_group 0;" ::"l"(a.host_out), "r"(smem_u32(ring)), "r"(d * 4)
              : "memory");
          asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
        }
        if (a.host_sel)
          for (int q = 0; q < k; ++q) a.host_sel[q] = __ldcg(a.sel + q);
        __threadfence_system();
        st_release_sys(a.host_done, a.host_seq);
      }
      __syncwarp();
    }
  }
}

template <int DW, int DS, int DSB>
__global__ void __launch_bounds__(DW * 32, 1) decode_layer_kernel(DecodeArgs a) {
  // a kernel launched after this one with programmatic stream serialization
  // (the next decoder layer's QKV GEMV) may be scheduled onto SMs as soon as
  // their CTAs of this grid exit; it waits (griddepcontrol.wait) for this
  // grid's completion before reading anything it produced
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // when this launch itself is programmatic (behind the attention O-proj):
  // everything below may read that kernel's output (early PLAN launches wait
  // inside decode_body, after starting their weight stream)
  if (!(a.early && a.mode == 1)) asm volatile("griddepcontrol.wait;" ::: "memory");
  decode_body<DW, DS, DSB>(a);
}

// ---------------------------------------------------------------- decode server
//
// A persistent cooperative launch that serves decode calls from the host
// without a kernel launch or a stream synchronisation per call: the host
// writes h into pinned memory and rings a doorbell word; CTA 0 sees it (PCIe
// poll), pulls h into HBM and releases the grid through a device flag; the
// grid runs the decode layer (decode_body, unchanged), writing the residual
// and the selection straight into pinned host memory; the last CTA fences
// and publishes the call's sequence number to a pinned `done` word the host
// spins on.  Idle longer than idle_ns (or doorbell = ~0u) ends the kernel.
struct ServerArgs {
  const unsigned* doorbell;  // pinned host: sequence number of the requested call, ~0u = stop
  const float* h_host;       // pinned host: the call's residual (d floats)
  unsigned* go;              // device: sequence released to the grid (~0u = stop)
  unsigned long long idle_ns;
  unsigned long long* trace;  // optional [calls][4] globaltimer: seen, released, body done, -
  int trace_cap;
};

// the doorbell is written by the CPU: acquire at system scope, so the h the
// host stored before ringing is what the following loads see
__device__ __forceinline__ unsigned ld_doorbell(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int DW, int DS, int DSB>
__global__ void __launch_bounds__(DW * 32, 1) decode_server_kernel(DecodeArgs a, ServerArgs sv) {
  // (no static shared memory here: the 8x7B layer uses all 227 KB dynamically)
  for (unsigned seq = 1;; ++seq) {
    unsigned v = 0;
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer_ns();
      if (blockIdx.x == 0) {
        while ((v = ld_doorbell(sv.doorbell)) != seq && v != ~0u) {
          if (globaltimer_ns() - t0 > sv.idle_ns) {
            v = ~0u;
            break;
          }
        }
        if (sv.trace && seq <= static_cast<unsigned>(sv.trace_cap))
          sv.trace[(seq - 1) * 4] = globaltimer_ns();
      } else {
        while ((v = ld_acquire_gpu(sv.go)) != seq && v != ~0u) {
          if (globaltimer_ns() - t0 > sv.idle_ns + 1000000000ull) {
            v = ~0u;
            break;
          }
        }
      }
    }
    if (__syncthreads_or(threadIdx.x == 0 && v == ~0u)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) st_release_gpu(sv.go, ~0u);
      return;
    }
    if (blockIdx.x == 0) {  // h: pinned host -> (one bulk DMA) smem -> HBM, release the grid
      extern __shared__ __align__(128) uint8_t smem_s[];
      uint64_t* bar = reinterpret_cast<uint64_t*>(smem_s + a.d * 4);
      if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, a.d * 4);
        bulk_g2s_plain(smem_s, sv.h_host, a.d * 4, bar);
      }
      __syncthreads();
      mbar_wait(bar, 0);
      __syncthreads();
      if (threadIdx.x == 0)  // the barrier's bytes become ring space for the body
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
      const float4* src = reinterpret_cast<const float4*>(smem_s);
      float4* dst = reinterpret_cast<float4*>(const_cast<float*>(a.h));
      for (int i = threadIdx.x; i < a.d / 4; i += DW * 32) dst[i] = src[i];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        st_release_gpu(sv.go, seq);
        if (sv.trace && seq <= static_cast<unsigned>(sv.trace_cap))
          sv.trace[(seq - 1) * 4 + 1] = globaltimer_ns();
      }
    }
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // h -> bulk copies
    __syncthreads();
    DecodeArgs b = a;
    b.host_seq = seq;
    decode_body<DW, DS, DSB>(b);
    __syncthreads();  // shared state is re-initialised by the next call
    if (sv.trace && threadIdx.x == 0 && seq <= static_cast<unsigned>(sv.trace_cap))
      atomicMax(&sv.trace[(seq - 1) * 4 + 2], globaltimer_ns());
  }
}

template <int DW, int DS, int DSB>
static int launch_decode(DecodeArgs a, int grid, cudaStream_t st, const ServerArgs* sv = nullptr) {
  a.rows_per_cta = (a.d + grid - 1) / grid;
  const int npc2 = (a.ffn * 2 + DSB - 1) / DSB;
  if (npc2 > kMaxChunks) {
    set_error("decode_layer: ffn=%d needs %d W2 pieces (max %d)", a.ffn, npc2, kMaxChunks);
    return DAOP_ERR_UNSUPPORTED;
  }
  const size_t ring = static_cast<size_t>(DW) * DS * DSB;
  const size_t stage_in = static_cast<size_t>(a.d) * 4 + static_cast<size_t>(a.E + 2) * a.d * 2;
  if (a.mode == 0 && stage_in > ring) {
    set_error("decode_layer: router inputs (%zu B) exceed the ring (%zu B)", stage_in, ring);
    return DAOP_ERR_UNSUPPORTED;
  }
  const size_t smem = ring + static_cast<size_t>(a.k) * a.ffn * 2 +
                      (static_cast<size_t>(a.d) * 2 + 127) / 128 * 128 +
                      static_cast<size_t>(a.rows_per_cta) * a.k * npc2 * 4 +
                      (static_cast<size_t>(a.rows_per_cta) * 4 + 127) / 128 * 128 +
                      (sizeof(DecodeSmem<DW, DS>) + 15) / 16 * 16 +
                      static_cast<size_t>(a.rows_per_cta) * 4 + 128;  // (+ hout_s)
  if (smem > 227 * 1024) {
    set_error("decode_layer: %zu B of shared memory exceeds 227 KB (k*ffn too large)", smem);
    return DAOP_ERR_UNSUPPORTED;
  }
  auto kern = decode_layer_kernel<DW, DS, DSB>;
  auto skern = decode_server_kernel<DW, DS, DSB>;
  DAOP_CUDA(cudaFuncSetAttribute(sv ? reinterpret_cast<const void*>(skern)
                                    : reinterpret_cast<const void*>(kern),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(DW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the per-pick waits
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (tuning: DAOP_MOE_PDL)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  // every decode launch programmatic and NOT cooperative (below): headline
  // 9,009-9,015 -> 9,155-9,159 tok/s over 3 A/B pairs (the next launch's CTAs
  // take each SM as the previous grid's CTA leaves, instead of a cooperative
  // grid dispatched once it fits as a whole); DAOP_MOE_PDL=0 turns it off
  static const int moe_pdl = [] {
    const char* v = getenv("DAOP_MOE_PDL");
    return v ? atoi(v) : 1;
  }();
  // early PLAN launches (behind the attention O-proj): without the cooperative
  // attribute -- a cooperative grid is dispatched only once the whole grid
  // fits (~5 us after the O-proj's last CTA); the grid (one CTA per SM, the
  // shared-memory footprint allows no second) is co-resident anyway once the
  // O-proj CTAs leave, which they do without waiting on this grid
  static const int early_coop = [] {
    const char* v = getenv("DAOP_EARLY_COOP");
    return v ? atoi(v) : 0;
  }();
  // programmatic launches (early PLAN layers, or DAOP_MOE_PDL=1 for every
  // decode launch) drop the cooperative attribute the same way; the kernel
  // waits for its predecessor (griddepcontrol.wait) before touching anything
  // the predecessor writes or its own self-resetting workspace
  const bool pdl = !sv && (a.early || moe_pdl);
  const bool plain = pdl && !early_coop;
  cfg.attrs = plain ? attr + 1 : attr;
  cfg.numAttrs = plain ? 1 : pdl ? 2 : 1;
  if (sv) DAOP_CUDA(cudaLaunchKernelEx(&cfg, skern, a, *sv));
  else DAOP_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return DAOP_OK;
}

}  // namespace daop

using namespace daop;

extern "C" int daop_decode_timeline(int32_t enable, uint64_t* h_out, int32_t n_cta) {
  if (h_out && n_cta > 0) {
    DAOP_CUDA(cudaMemcpyFromSymbol(h_out, g_decode_timeline,
                                   sizeof(unsigned long long) * 16 * (n_cta < 1024 ? n_cta : 1024)));
  }
  if (enable) {
    static unsigned long long zeros[1024][16];
    DAOP_CUDA(cudaMemcpyToSymbol(g_decode_timeline, zeros, sizeof(zeros)));
  }
  DAOP_CUDA(cudaMemcpyToSymbol(g_decode_timeline_on, &enable, sizeof(int)));
  return DAOP_OK;
}

extern "C" int daop_decode_workspace(int32_t d, int32_t ffn, int32_t E, int32_t k,
                                     int64_t* bytes) {
  // ctr (32 u32) | pred logits (E f32, padded) | act (k*ffn bf16)
  (void)d;
  *bytes = 128 + (static_cast<int64_t>(E) * 4 + 255) / 256 * 256 +
           (static_cast<int64_t>(k) * ffn * 2 + 255) / 256 * 256;
  return DAOP_OK;
}

static thread_local const uint64_t* t_ep_peers = nullptr;
static thread_local int t_ep_G = 0, t_ep_rank = 0;
static thread_local unsigned t_ep_epoch = 0;

extern "C" int daop_decode_layer(const float* h, const uint16_t* gamma, const uint16_t* wg,
                                 const uint16_t* wg_next, const float* pred_prev,
                                 const uint8_t* fast_row, const int32_t* slot_of,
                                 const uint16_t* slab, int64_t slot_stride, int32_t d,
                                 int32_t ffn, int32_t E, int32_t k, int32_t mode,
                                 int32_t graceful, int32_t weights_from_pred, float eps,
                                 uint16_t* x_out, float* p_true, float* p_pred, int32_t* sel,
                                 float* w, uint8_t* is_fast, int32_t* deg, float* y,
                                 float* h_out, void* workspace, int32_t variant,
                                 daop_stream_t stream) {
  if (E < 2 || E > DE_MAX || k < 1 || k > DK_MAX || k > E || d % 8 || ffn % 8) {
    set_error("decode_layer: unsupported shape (E=%d k=%d d=%d ffn=%d)", E, k, d, ffn);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (mode == 1 && !pred_prev) {
    set_error("decode_layer: PLAN mode needs the previous layer's prediction");
    return DAOP_ERR_PREDICTION_MISSING;
  }
  DecodeArgs a{};  // value-initialised: optional pointers (EP, server) stay null
  a.h = h; a.gamma = gamma; a.wg = wg; a.wg_next = wg_next; a.pred_prev = pred_prev;
  a.fast_row = fast_row; a.slot_of = slot_of; a.slab = slab; a.slot_stride = slot_stride;
  a.d = d; a.ffn = ffn; a.E = E; a.k = k; a.mode = mode; a.graceful = graceful;
  a.weights_from_pred = weights_from_pred; a.eps = eps;
  a.x_out = x_out; a.p_true = p_true; a.p_pred = wg_next ? p_pred : nullptr; a.sel = sel;
  a.w = w; a.is_fast = is_fast; a.deg = deg; a.y = y; a.h_out = h_out;
  a.ep_peers = t_ep_peers; a.ep_G = t_ep_G; a.ep_rank = t_ep_rank; a.ep_epoch = t_ep_epoch;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.ctr = reinterpret_cast<unsigned*>(ws);
  a.pred_logits = reinterpret_cast<float*>(ws + 128);
  a.act = reinterpret_cast<uint16_t*>(ws + 128 + (static_cast<int64_t>(E) * 4 + 255) / 256 * 256);
  // variant bit 8: early PLAN launch behind the attention O-proj (DecodeArgs::early)
  a.early = (variant >> 8) & 1 && mode == 1 ? 1 : 0;
  variant &= 0xff;
  int grid = sm_count();
  if (grid < E) grid = E;  // CTAs 0..E-1 own one next-layer gate row each
  cudaStream_t st = as_stream(stream);
  // default geometry: 16 warps x 1 stage x 10 KB pieces (110.6 us vs 117.2 us
  // for 8 warps x 2 stages: twice the warps computing W2 partials in phase 2)
  switch (variant) {
    case 1: return launch_decode<4, 4, 10240>(a, grid, st);
    case 9: return launch_decode<8, 2, 10240>(a, grid, st);
    case 2: return launch_decode<8, 2, 8192>(a, grid, st);
    case 3: return launch_decode<6, 3, 8192>(a, grid, st);
    case 4: return launch_decode<16, 1, 10240>(a, grid, st);
    case 5: return launch_decode<16, 2, 4608>(a, grid, st);
    case 6: return launch_decode<12, 2, 6144>(a, grid, st);
    case 7: return launch_decode<16, 1, 8192>(a, grid, st);
    case 8: return launch_decode<10, 2, 7680>(a, grid, st);
    // Mixtral-8x22B candidates (d = 6144: a W1/W3 row is 12 KB)
    case 10: return launch_decode<12, 1, 12288>(a, grid, st);
    case 11: return launch_decode<24, 1, 6144>(a, grid, st);
    case 12: return launch_decode<8, 2, 9216>(a, grid, st);
    case 13: return launch_decode<16, 1, 9216>(a, grid, st);
    default: {
      // largest ring that fits: Mixtral-8x22B (d = 6144, ffn = 16384) needs
      // 64 KB of activations in shared memory and a 144 KB router stage
      int rc = launch_decode<16, 1, 9600>(a, grid, st);
      if (rc != DAOP_ERR_UNSUPPORTED) return rc;
      rc = launch_decode<16, 1, 9216>(a, grid, st);
      if (rc != DAOP_ERR_UNSUPPORTED) return rc;
      return launch_decode<16, 1, 8192>(a, grid, st);
    }
  }
}

// Expert-parallel decode layer: daop_decode_layer whose kernel also stores
// this GPU's picks' outputs into every peer's decode workspace and flags them
// (ep_p2p.cu; the share is fused into the phase-2 reduction).
extern "C" int daop_ep_decode_layer(const uint64_t* d_peers, int32_t rank, int32_t G,
                                    uint32_t epoch, const float* h, const uint16_t* gamma,
                                    const uint16_t* wg, const uint16_t* wg_next,
                                    const uint8_t* fast_row, const int32_t* slot_of,
                                    const uint16_t* slab, int64_t slot_stride, int32_t d,
                                    int32_t ffn, int32_t E, int32_t k, float eps,
                                    uint16_t* x_out, float* p_true, float* p_pred, int32_t* sel,
                                    float* w, uint8_t* is_fast, int32_t* deg, float* y,
                                    float* h_out, void* workspace, daop_stream_t stream) {
  if (!d_peers || G < 1 || G > EP_MAX_G || rank < 0 || rank >= G || d % 4 != 0) {
    set_error("ep_decode_layer: bad peers / rank %d / world %d", rank, G);
    return DAOP_ERR_UNSUPPORTED;
  }
  t_ep_peers = d_peers;
  t_ep_G = G;
  t_ep_rank = rank;
  t_ep_epoch = epoch;
  const int rc = daop_decode_layer(h, gamma, wg, wg_next, nullptr, fast_row, slot_of, slab,
                                   slot_stride, d, ffn, E, k, 0, 0, 0, eps, x_out, p_true,
                                   p_pred, sel, w, is_fast, deg, y, h_out, workspace, 0, stream);
  t_ep_peers = nullptr;
  return rc;
}

// ---------------------------------------------------------------- decode server C ABI

static unsigned long long* g_server_trace = nullptr;  // profiling aid (daop_server_trace)
static int g_server_trace_cap = 0;

// profiling aid: per-call GPU timestamps of the next server started
// ([seq][4]: doorbell seen, h released to the grid, body done; device memory)
extern "C" int daop_server_trace(uint64_t* d_buf, int32_t cap) {
  g_server_trace = reinterpret_cast<unsigned long long*>(d_buf);
  g_server_trace_cap = cap;
  return DAOP_OK;
}

namespace {
struct DecodeServer {
  unsigned* doorbell = nullptr;  // pinned host
  unsigned* done = nullptr;      // pinned host
  float* h_host = nullptr;       // pinned host staging of the input residual
  unsigned* go = nullptr;        // device
  float* h_dev = nullptr;        // device copy of the input
  float* out_dev = nullptr;      // device residual out (shipped to the host by the last warp)
  int32_t* sel_dev = nullptr;
  unsigned seq = 0;
  int d = 0;
  cudaStream_t stream = nullptr;
};
}  // namespace

static void server_free(DecodeServer* s) {
  if (s->doorbell) cudaFreeHost(s->doorbell);
  if (s->h_host) cudaFreeHost(s->h_host);
  if (s->go) cudaFree(s->go);
  if (s->h_dev) cudaFree(s->h_dev);
  if (s->out_dev) cudaFree(s->out_dev);
  if (s->sel_dev) cudaFree(s->sel_dev);
  delete s;
}

// Start a persistent decode server for one MoE layer (mode 0, all arguments
// as daop_decode_layer; d_h_out and d_sel should be pinned host memory --
// the kernel writes the result there).  The server kernel occupies every SM
// until daop_server_stop or idle_ms without a call.
extern "C" int daop_server_start(const uint16_t* gamma, const uint16_t* wg,
                                 const uint16_t* wg_next, const uint8_t* fast_row,
                                 const int32_t* slot_of, const uint16_t* slab,
                                 int64_t slot_stride, int32_t d, int32_t ffn, int32_t E,
                                 int32_t k, float eps, uint16_t* x_out, float* p_true,
                                 float* p_pred, int32_t* sel, float* w, uint8_t* is_fast,
                                 int32_t* deg, float* y, float* h_out, void* workspace,
                                 double idle_ms, daop_stream_t stream, void** handle) {
  if (E < 2 || E > DE_MAX || k < 1 || k > DK_MAX || k > E || d % 8 || ffn % 8) {
    set_error("decode server: unsupported shape (E=%d k=%d d=%d ffn=%d)", E, k, d, ffn);
    return DAOP_ERR_UNSUPPORTED;
  }
  auto* s = new DecodeServer();
  s->d = d;
  s->stream = as_stream(stream);
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&s->doorbell), 256, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&s->h_host), d * 4,
                                          cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&s->go), 256);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&s->h_dev), d * 4);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&s->out_dev), d * 4);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&s->sel_dev), 64);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->go, 0, 256, s->stream);
  if (e != cudaSuccess) {
    server_free(s);
    return cuda_fail(e, "decode server allocation");
  }
  s->done = s->doorbell + 32;  // separate 128-byte line
  *reinterpret_cast<volatile unsigned*>(s->doorbell) = 0;
  *reinterpret_cast<volatile unsigned*>(s->done) = 0;
  DecodeArgs a{};
  a.h = s->h_dev; a.gamma = gamma; a.wg = wg; a.wg_next = wg_next; a.pred_prev = nullptr;
  a.fast_row = fast_row; a.slot_of = slot_of; a.slab = slab; a.slot_stride = slot_stride;
  a.d = d; a.ffn = ffn; a.E = E; a.k = k; a.mode = 0; a.graceful = 0;
  a.weights_from_pred = 0; a.eps = eps;
  a.x_out = x_out; a.p_true = p_true; a.p_pred = wg_next ? p_pred : nullptr;
  a.w = w; a.is_fast = is_fast; a.deg = deg; a.y = y;
  a.h_out = s->out_dev;  // every CTA writes HBM; the last warp ships it to the host
  a.sel = s->sel_dev;
  a.host_out = h_out;
  a.host_sel = sel;
  {
    static const int ship = [] {  // DAOP_SERVER_SHIP_CTA=0: the last warp ships all rows
      const char* v = getenv("DAOP_SERVER_SHIP_CTA");
      return v ? atoi(v) : 1;
    }();
    int g = sm_count();
    if (g < E) g = E;
    const int rpc = (d + g - 1) / g;
    a.ship_cta = ship && h_out && rpc % 4 == 0 &&
                 (reinterpret_cast<uintptr_t>(h_out) & 15) == 0 ? 1 : 0;
  }
  a.ep_peers = nullptr;
  a.host_done = s->done;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.ctr = reinterpret_cast<unsigned*>(ws);
  a.pred_logits = reinterpret_cast<float*>(ws + 128);
  a.act = reinterpret_cast<uint16_t*>(ws + 128 + (static_cast<int64_t>(E) * 4 + 255) / 256 * 256);
  ServerArgs sv{s->doorbell, s->h_host, s->go,
                static_cast<unsigned long long>(idle_ms * 1e6), g_server_trace,
                g_server_trace_cap};
  int grid = sm_count();
  if (grid < E) grid = E;
  int rc = launch_decode<16, 1, 9600>(a, grid, s->stream, &sv);
  if (rc == DAOP_ERR_UNSUPPORTED) rc = launch_decode<16, 1, 9216>(a, grid, s->stream, &sv);
  if (rc == DAOP_ERR_UNSUPPORTED) rc = launch_decode<16, 1, 8192>(a, grid, s->stream, &sv);
  if (rc) {
    server_free(s);
    return rc;
  }
  *handle = s;
  return DAOP_OK;
}

// One call: h (d floats, any host memory) -> the server; returns once the
// residual and the selection are in the pinned host buffers given at start.
extern "C" int daop_server_step(void* handle, const float* h_src, double timeout_ms) {
  auto* s = static_cast<DecodeServer*>(handle);
  memcpy(s->h_host, h_src, static_cast<size_t>(s->d) * 4);
  const unsigned seq = ++s->seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile unsigned*>(s->doorbell) = seq;
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (*reinterpret_cast<volatile unsigned*>(s->done) != seq) {
    if ((++spins & 1023) == 0) {
      const double ms = std::chrono::duration<double, std::milli>(
          std::chrono::steady_clock::now() - t0).count();
      if (ms > timeout_ms) {
        const cudaError_t q = cudaStreamQuery(s->stream);
        set_error("decode server: call %u not answered in %.0f ms (server %s)", seq, ms,
                  q == cudaSuccess ? "exited (idle timeout?)" : "running");
        return DAOP_ERR_CUDA;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return DAOP_OK;
}

extern "C" int daop_server_stop(void* handle) {
  auto* s = static_cast<DecodeServer*>(handle);
  *reinterpret_cast<volatile unsigned*>(s->doorbell) = ~0u;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  const cudaError_t e = cudaStreamSynchronize(s->stream);
  server_free(s);
  DAOP_CUDA(e);
  return DAOP_OK;
}
