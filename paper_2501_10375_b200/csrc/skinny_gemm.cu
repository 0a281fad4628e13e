// Grouped SwiGLU expert FFN for SMALL token counts (batched decode, b <= ~128):
// the "swap-AB" form of grouped_gemm.cu.  With a handful of tokens per expert
// the X . W^T tiles of the prefill GEMM waste the tensor pipe (M = 256/512
// rows of which a few are real) and the layer becomes compute-bound on empty
// rows (~2.7 TB/s of weights at b = 64).  Here the WEIGHTS are the M side:
//
//   up  : D1 = W1[rows] . X^T, D3 = W3[rows] . X^T   (M = 128 weight rows,
//         N = NT token columns, K = d), act[t, row] = bf16(silu(D1) * D3)
//   down: D = W2[rows] . act^T                        (K = ffn), y[t, row] fp32
//
// so a tile costs 128 x NT x K MACs and the kernel streams each expert's
// weights once per block of NT tokens -- HBM-bound like the b = 1 decode GEMV.
// One CTA per SM, persistent, warp-specialised like grouped_gemm.cu: warp 0
// TMA producer (weight box(es) 128 x 64 + token box NT x 64 per stage), warp 1
// tcgen05.mma.cta_group::1 issuer (M 128, N NT, K 16), warps 2-5 epilogue
// (thread = weight row, tcgen05.ld 32x32b.x32 over the token columns; stores
// for one token are 32 consecutive rows per warp).  Tile = (expert, token
// block, 128-row weight tile), weight tiles fastest.
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ep.cuh"
#include "tcgen05.cuh"

namespace daop {

constexpr int SK_K = 64;                      // K per stage (one 128-byte swizzle row)
constexpr int SK_W_BYTES = 128 * SK_K * 2;    // one 128-row weight box, 16 KB
constexpr int SK_MAX_E = 64;

int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box);

struct SkinnyParams {
  const int64_t* offsets;   // [E+1] token row offsets (device)
  const int32_t* slot_of;   // [E]
  int E;
  int k_blocks;             // K / 64
  int row_tiles;            // weight rows / 128 (per matrix)
  int w_half2;              // SWIGLU: row offset of W3 (= ffn)
  void* out;                // up: bf16 act (rows, ffn); down: fp32 y (rows, d)
  int64_t out_ld;
  // expert-parallel return (down only, ep_p2p.cu): row t of the output goes
  // to the address row_dst[t] (the source GPU's y_back row) and the last CTA
  // flags y[sig_rank] = sig_epoch on every peer
  const uint64_t* row_dst;
  unsigned* sig_done;
  const uint64_t* sig_peers;
  int sig_G, sig_rank;
  unsigned sig_epoch;
  // dense GEMM (daop_gemm_bf16_f32 for M <= 768): no offset / slot tables,
  // one "expert" of dense_rows token rows, weight slot 0; down only: the
  // residual added in the epilogue (may alias out); weights kept in L2
  // (evict_normal) because every token block re-reads them
  int64_t dense_rows;
  const float* resid;
  int w_keep;
};

__device__ __forceinline__ int64_t sk_off(const SkinnyParams& p, int e) {
  return p.offsets ? p.offsets[e] : (e == 0 ? 0 : p.dense_rows);
}
__device__ __forceinline__ int sk_slot(const SkinnyParams& p, int e) {
  return p.slot_of ? p.slot_of[e] : 0;
}

template <int NT>
struct SkinnySmem {
  static constexpr int STAGES = 8;  // upper bound; the kernel uses SkinnyCfg::STAGES
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int32_t prefix[SK_MAX_E + 1];
  int32_t blocks[SK_MAX_E];
  int64_t off[SK_MAX_E + 1];
};

template <bool SWIGLU, int NT>
struct SkinnyCfg {
  static constexpr int W_BYTES = SWIGLU ? 2 * SK_W_BYTES : SK_W_BYTES;
  static constexpr int X_BYTES = NT * SK_K * 2;
  static constexpr int STAGE_BYTES = W_BYTES + X_BYTES;
  // up (NT 64): 5 x 40 KB stages, one CTA per SM; down: 4 x 24 KB stages so
  // TWO CTAs share an SM -- its d / 128 row tiles per expert (256 at b = 64)
  // then fill one wave of 2 x 148 CTAs instead of leaving half a second wave
  static constexpr int CTAS_PER_SM = SWIGLU ? 1 : 2;
  static constexpr int BUDGET = SWIGLU ? 200 * 1024 : 108 * 1024;
  static constexpr int STAGES = BUDGET / STAGE_BYTES < SkinnySmem<NT>::STAGES
                                    ? BUDGET / STAGE_BYTES : SkinnySmem<NT>::STAGES;
  static constexpr int ACC_COLS = SWIGLU ? 2 * NT : NT;  // per accumulator buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 32 ? 32 : 2 * ACC_COLS <= 64 ? 64
                                   : 2 * ACC_COLS <= 128 ? 128 : 2 * ACC_COLS <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = umma_idesc_bf16_f32(128, NT);
};

template <int NT>
__device__ __forceinline__ bool skinny_tile(const SkinnySmem<NT>& s, int E, int rt, int t, int& e,
                                            int& blk, int& r) {
  if (t >= s.prefix[E]) return false;
  e = 0;
  while (s.prefix[e + 1] <= t) ++e;
  const int u = t - s.prefix[e];
  // token blocks fastest within a weight tile: an expert with more than NT
  // rows (a prompt) has its blocks of one weight tile on neighbouring CTAs at
  // the same time, so the tile crosses HBM once and the rest hit L2
  const int nb = s.blocks[e];
  r = u / nb;
  blk = u - r * nb;
  (void)rt;
  return true;
}

template <bool SWIGLU, int NT>
__global__ void __launch_bounds__(192, SkinnyCfg<SWIGLU, NT>::CTAS_PER_SM)
    skinny_gemm_kernel(const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmX, SkinnyParams p) {
  pdl_prologue();  // (launched with launch_pdl)
  using C = SkinnyCfg<SWIGLU, NT>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  SkinnySmem<NT>& s = *reinterpret_cast<SkinnySmem<NT>*>(tiles + C::STAGES * C::STAGE_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = p.E, rt = p.row_tiles;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 4);
    }
    fence_mbar_init();
    int acc = 0;
    s.prefix[0] = 0;
    for (int e = 0; e <= E; ++e) s.off[e] = sk_off(p, e);
    for (int e = 0; e < E; ++e) {
      const int64_t me = sk_slot(p, e) >= 0 ? s.off[e + 1] - s.off[e] : 0;
      s.blocks[e] = static_cast<int>((me + NT - 1) / NT);
      acc += s.blocks[e] * rt;
      s.prefix[e + 1] = acc;
    }
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = s.tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      const uint64_t pol_once = l2_evict_first_policy();   // weights read by one token block
      const uint64_t pol_reuse = l2_evict_normal_policy();  // ... by several (neighbour CTAs)
      const uint64_t pol_x = l2_evict_last_policy();   // tokens: re-read by every row tile
      int stage = 0;
      uint32_t phase = 0;
      int e, blk, r;
      for (int t = blockIdx.x; skinny_tile(s, E, rt, t, e, blk, r); t += gridDim.x) {
        const int slot = sk_slot(p, e);
        const int xrow = static_cast<int>(s.off[e]) + blk * NT;
        const uint64_t pol_w = (p.w_keep || s.blocks[e] > 1) ? pol_reuse : pol_once;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          uint8_t* st = tiles + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&s.full[stage], C::STAGE_BYTES);
          tma_load_3d(st, &tmW, &s.full[stage], kb * SK_K, r * 128, slot, pol_w);
          if constexpr (SWIGLU)
            tma_load_3d(st + SK_W_BYTES, &tmW, &s.full[stage], kb * SK_K, r * 128 + p.w_half2,
                        slot, pol_w);
          tma_load_2d(st + C::W_BYTES, &tmX, &s.full[stage], kb * SK_K, xrow, pol_x);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      int e, blk, r;
      for (int t = blockIdx.x; skinny_tile(s, E, rt, t, e, blk, r); t += gridDim.x) {
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * C::ACC_COLS;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&s.full[stage], phase);
          tc_fence_after();
          uint8_t* st = tiles + stage * C::STAGE_BYTES;
          const uint64_t wdesc = umma_desc_sw128(smem_u32(st));
          const uint64_t xdesc = umma_desc_sw128(smem_u32(st + C::W_BYTES));
#pragma unroll
          for (int k = 0; k < SK_K / 16; ++k) {
            umma_bf16(d0, wdesc + 2 * k, xdesc + 2 * k, C::IDESC, (kb | k) != 0);
            if constexpr (SWIGLU) {
              const uint64_t w3desc = umma_desc_sw128(smem_u32(st + SK_W_BYTES));
              umma_bf16(d0 + NT, w3desc + 2 * k, xdesc + 2 * k, C::IDESC, (kb | k) != 0);
            }
          }
          umma_commit(&s.empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&s.tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {  // epilogue: thread = weight row of the tile, columns = tokens
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int e, blk, r;
    for (int t = blockIdx.x; skinny_tile(s, E, rt, t, e, blk, r); t += gridDim.x) {
      mbar_wait(&s.tfull[acc], acc_phase);
      tc_fence_after();
      const int row = r * 128 + q * 32 + lane;
      const int64_t t0 = s.off[e] + static_cast<int64_t>(blk) * NT;
      const int64_t rem = s.off[e + 1] - t0;
      const int nvalid = rem < NT ? static_cast<int>(rem) : NT;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < NT; c += 32) {
        uint32_t g[32];
        tmem_ld32(tb + c, g);
        if constexpr (SWIGLU) {
          uint32_t u[32];
          tmem_ld32(tb + NT + c, u);
          tmem_ld_wait();
          const int nj = nvalid - c < 32 ? nvalid - c : 32;
          uint16_t* o = static_cast<uint16_t*>(p.out) + (t0 + c) * p.out_ld + row;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < nj)
              *o = f32_to_bf16_bits(
                  __fdividef(__uint_as_float(g[j]), 1.0f + __expf(-__uint_as_float(g[j]))) *
                  __uint_as_float(u[j]));  // the prefill GEMM's SwiGLU (silu_fast)
            o += p.out_ld;
          }
        } else {
          tmem_ld_wait();
          const int nj = nvalid - c < 32 ? nvalid - c : 32;
          if (p.row_dst) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nj) reinterpret_cast<float*>(p.row_dst[t0 + c + j])[row] = __uint_as_float(g[j]);
          } else {
            // one running pointer per stream (precomputed per-token addresses
            // cost 2 x 32 registers and spilled for NT > 64)
            const int64_t off = (t0 + c) * p.out_ld + row;
            float* o = static_cast<float*>(p.out) + off;
            const float* rr = p.resid ? p.resid + off : nullptr;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (j < nj) *o = rr ? __uint_as_float(g[j]) + *rr : __uint_as_float(g[j]);
              o += p.out_ld;
              if (rr) rr += p.out_ld;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  if (p.sig_done) __threadfence_system();  // this thread's (remote) output rows
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
  if (p.sig_done && threadIdx.x == 0 && atomicAdd(p.sig_done, 1u) == gridDim.x - 1) {
    *p.sig_done = 0;
    __threadfence_system();
    for (int q = 0; q < p.sig_G; ++q)
      st_release_sys(reinterpret_cast<unsigned*>(p.sig_peers[q] + EP_FLAGS_Y) + p.sig_rank,
                     p.sig_epoch);
  }
}

template <bool SWIGLU, int NT>
static int launch_skinny(const CUtensorMap& tw, const CUtensorMap& tx, const SkinnyParams& p,
                         int64_t rows_total, cudaStream_t st) {
  using C = SkinnyCfg<SWIGLU, NT>;
  const size_t smem = 1024 + C::STAGES * C::STAGE_BYTES + sizeof(SkinnySmem<NT>);
  auto kern = skinny_gemm_kernel<SWIGLU, NT>;
  DAOP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const int64_t max_tiles = (rows_total / NT + p.E) * static_cast<int64_t>(p.row_tiles);
  int grid = sm_count() * C::CTAS_PER_SM;
  if (max_tiles < grid) grid = static_cast<int>(max_tiles < 1 ? 1 : max_tiles);
  static const bool skinny_pdl = [] {  // tuning: DAOP_PDL_SKINNY=0 launches it plainly
    const char* v = getenv("DAOP_PDL_SKINNY");
    return !(v && v[0] == '0');
  }();
  // decode-sized batches launch plainly: with PDL the batched-decode step
  // (b = 64, 128 rows) took 0.454-0.455 vs 0.447 ms; prompt-sized ones gain
  // (256-token prefill 0.636-0.642 -> 0.633-0.634 ms per layer)
  if (skinny_pdl && rows_total > 256) {
    DAOP_CUDA(launch_pdl(kern, dim3(grid), dim3(192), smem, st, tw, tx, p));
  } else {
    kern<<<grid, 192, smem, st>>>(tw, tx, p);  // (its griddepcontrol.wait is a no-op)
  }
  DAOP_CHECK_LAUNCH(SWIGLU ? "skinny_gemm_up" : "skinny_gemm_down");
  return DAOP_OK;
}

// token block NT = the MMA's N: any multiple of 16 works for M = 128; these
// cover decode batches (32), prompts of ~100-400 tokens per layer (48..128:
// the caller sizes NT to the expected rows per expert so one block holds an
// expert's tokens without streaming mostly-empty token rows)
template <bool SWIGLU>
static int skinny_dispatch(const CUtensorMap& tw, const CUtensorMap& tx, const SkinnyParams& p,
                           int64_t rows, int32_t nt, cudaStream_t st) {
  switch (nt) {
    case 32: return launch_skinny<SWIGLU, 32>(tw, tx, p, rows, st);
    case 48: return launch_skinny<SWIGLU, 48>(tw, tx, p, rows, st);
    case 80: return launch_skinny<SWIGLU, 80>(tw, tx, p, rows, st);
    case 96: return launch_skinny<SWIGLU, 96>(tw, tx, p, rows, st);
    case 128: return launch_skinny<SWIGLU, 128>(tw, tx, p, rows, st);
    default: return launch_skinny<SWIGLU, 64>(tw, tx, p, rows, st);
  }
}

}  // namespace daop

using namespace daop;

static int check_skinny(int64_t rows, int32_t d, int32_t ffn, int32_t E, int32_t nt) {
  if (E < 1 || E > SK_MAX_E || d % 128 != 0 || ffn % 128 != 0 || d % 64 != 0 ||
      (nt != 32 && nt != 48 && nt != 64 && nt != 80 && nt != 96 && nt != 128) || rows < 0 ||
      rows >= (1ll << 31)) {
    set_error("skinny expert GEMM: unsupported shape (rows=%lld d=%d ffn=%d E=%d nt=%d)",
              static_cast<long long>(rows), d, ffn, E, nt);
    return DAOP_ERR_UNSUPPORTED;
  }
  return DAOP_OK;
}

extern "C" int daop_expert_gemm_up_skinny(const uint16_t* x_perm, int64_t rows, int32_t d,
                                          int32_t ffn, const uint16_t* slab, int64_t n_slots,
                                          int64_t slot_stride_elems, const int64_t* d_offsets,
                                          const int32_t* d_slot_of, int32_t E, uint16_t* act,
                                          int32_t nt, daop_stream_t stream) {
  int rc = check_skinny(rows, d, ffn, E, nt);
  if (rc) return rc;
  if (rows == 0) return DAOP_OK;
  CUtensorMap tw, tx;
  const uint64_t wdims[3] = {static_cast<uint64_t>(d), static_cast<uint64_t>(2 * ffn),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t wstr[2] = {static_cast<uint64_t>(d) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t wbox[3] = {SK_K, 128, 1};
  if ((rc = make_tmap_bf16(&tw, slab, 3, wdims, wstr, wbox))) return rc;
  const uint64_t xdims[2] = {static_cast<uint64_t>(d), static_cast<uint64_t>(rows)};
  const uint64_t xstr[1] = {static_cast<uint64_t>(d) * 2};
  const uint32_t xbox[2] = {SK_K, static_cast<uint32_t>(nt)};
  if ((rc = make_tmap_bf16(&tx, x_perm, 2, xdims, xstr, xbox))) return rc;
  SkinnyParams p{d_offsets, d_slot_of, E, d / SK_K, ffn / 128, ffn, act, ffn};
  return skinny_dispatch<true>(tw, tx, p, rows, nt, as_stream(stream));
}

extern "C" int daop_expert_gemm_down_skinny(const uint16_t* act, int64_t rows, int32_t d,
                                            int32_t ffn, const uint16_t* slab, int64_t n_slots,
                                            int64_t slot_stride_elems, const int64_t* d_offsets,
                                            const int32_t* d_slot_of, int32_t E, float* y,
                                            int32_t nt, daop_stream_t stream) {
  int rc = check_skinny(rows, d, ffn, E, nt);
  if (rc) return rc;
  if (rows == 0) return DAOP_OK;
  CUtensorMap tw, tx;
  const uint64_t wdims[3] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(d),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t wstr[2] = {static_cast<uint64_t>(ffn) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t wbox[3] = {SK_K, 128, 1};
  const uint16_t* w2 = slab + static_cast<int64_t>(2) * ffn * d;
  if ((rc = make_tmap_bf16(&tw, w2, 3, wdims, wstr, wbox))) return rc;
  const uint64_t xdims[2] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(rows)};
  const uint64_t xstr[1] = {static_cast<uint64_t>(ffn) * 2};
  const uint32_t xbox[2] = {SK_K, static_cast<uint32_t>(nt)};
  if ((rc = make_tmap_bf16(&tx, act, 2, xdims, xstr, xbox))) return rc;
  SkinnyParams p{d_offsets, d_slot_of, E, ffn / SK_K, d / 128, 0, y, d};
  return skinny_dispatch<false>(tw, tx, p, rows, nt, as_stream(stream));
}

// Expert-parallel down GEMM for small receive buffers (batched decode over
// several GPUs): the skinny kernel with the return table and the peer flags
// of daop_ep_expert_gemm_down.
extern "C" int daop_ep_expert_gemm_down_skinny(const uint16_t* act, int64_t rows_cap, int32_t d,
                                               int32_t ffn, const uint16_t* slab, int64_t n_slots,
                                               int64_t slot_stride_elems,
                                               const int32_t* d_slot_of, int32_t E,
                                               const uint64_t* d_peers, void* d_ws, int32_t rank,
                                               int32_t G, uint32_t epoch, int32_t nt,
                                               daop_stream_t stream) {
  int rc = check_skinny(rows_cap, d, ffn, E, nt);
  if (rc) return rc;
  if (G < 1 || G > EP_MAX_G || rank < 0 || rank >= G || rows_cap < 1) {
    set_error("ep skinny gemm: bad rank/world (%d/%d) or capacity", rank, G);
    return DAOP_ERR_UNSUPPORTED;
  }
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  CUtensorMap tw, tx;
  const uint64_t wdims[3] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(d),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t wstr[2] = {static_cast<uint64_t>(ffn) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t wbox[3] = {SK_K, 128, 1};
  const uint16_t* w2 = slab + static_cast<int64_t>(2) * ffn * d;
  if ((rc = make_tmap_bf16(&tw, w2, 3, wdims, wstr, wbox))) return rc;
  const uint64_t xdims[2] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(rows_cap)};
  const uint64_t xstr[1] = {static_cast<uint64_t>(ffn) * 2};
  const uint32_t xbox[2] = {SK_K, static_cast<uint32_t>(nt)};
  if ((rc = make_tmap_bf16(&tx, act, 2, xdims, xstr, xbox))) return rc;
  SkinnyParams p{reinterpret_cast<const int64_t*>(ws + EP_LOCAL_OFF), d_slot_of, E, ffn / SK_K,
                 d / 128, 0, nullptr, d, reinterpret_cast<const uint64_t*>(ws + EP_ROWMAP),
                 reinterpret_cast<unsigned*>(ws + EP_DONE_GEMM), d_peers, G, rank, epoch};
  return skinny_dispatch<false>(tw, tx, p, rows_cap, nt, as_stream(stream));
}

// the dense projection entry's small-M path (grouped_gemm.cu daop_gemm_bf16_f32)
int skinny_dense_gemm(const uint16_t* a, int64_t M, int32_t K, const uint16_t* w, int32_t N,
                      const float* resid, float* out, cudaStream_t st) {
  int rc;
  CUtensorMap tw, tx;
  const uint64_t wdims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), 1};
  const uint64_t wstr[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * N * 2};
  const uint32_t wbox[3] = {SK_K, 128, 1};
  if ((rc = make_tmap_bf16(&tw, w, 3, wdims, wstr, wbox))) return rc;
  // token block (tuning override: DAOP_DENSE_NT environment variable)
  static const int nt_env = [] {
    const char* v = getenv("DAOP_DENSE_NT");
    return v ? atoi(v) : 0;
  }();
  // default: 64-token blocks unless they leave SMs without a weight tile
  // (256-token prompt: O-proj 128 tiles -> 32-token blocks, 56 vs 71 us;
  // QKV 192 tiles -> 64, 43 vs 60 us)
  const int64_t tiles64 = (N / 128) * ((M + 63) / 64);
  const int nt = nt_env == 32 || nt_env == 64 || nt_env == 128
                     ? nt_env
                     : (M <= 32 || tiles64 < sm_count() ? 32 : 64);
  const uint64_t xdims[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(M)};
  const uint64_t xstr[1] = {static_cast<uint64_t>(K) * 2};
  const uint32_t xbox[2] = {SK_K, static_cast<uint32_t>(nt)};
  if ((rc = make_tmap_bf16(&tx, a, 2, xdims, xstr, xbox))) return rc;
  SkinnyParams p{nullptr, nullptr, 1, K / SK_K, N / 128, 0, out, N};
  p.dense_rows = M;
  p.resid = resid;
  p.w_keep = M > nt;
  return skinny_dispatch<false>(tw, tx, p, M, nt, st);
}
