// Grouped SwiGLU expert FFN for prefill on the 5th-gen tensor cores.
//
// Two persistent, warp-specialised tcgen05 GEMMs over the expert-sorted token
// rows produced by the permutation (offsets[e] .. offsets[e+1] belong to
// expert e; the weights of expert e live in HBM slot slot_of[e] of the slab):
//
//   up   : act[r, :] = bf16( silu(x_r . W1_e^T) * (x_r . W3_e^T) )   K = d
//          one 128x256 tile = 128 W1 rows + the matching 128 W3 rows, so the
//          SwiGLU is applied in the epilogue straight out of TMEM.
//   down : y[r, :]   = act_r . W2_e^T  (fp32)                          K = ffn
//
// Roles per CTA (one CTA per SM, 192 threads):
//   warp 0     TMA producer: A box 64x128 + two B boxes 64x128 per stage
//              (cp.async.bulk.tensor, SWIZZLE_128B), 4-stage mbarrier ring
//   warp 1     MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16
//              M=128 N=256 K=16 (x4 per stage) into a TMEM accumulator,
//              tcgen05.commit frees the smem stage / publishes the accumulator
//   warps 2-5  epilogue: tcgen05.ld 32x32b -> registers -> SwiGLU / fp32 store;
//              two TMEM accumulators (2 x 256 columns) double-buffer MMA vs
//              epilogue.
// Tiles are (expert, m-tile, n-tile), rasterised in groups of G m-tiles so
// the weight tile is shared in L2 by the CTAs working on the same group.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ep.cuh"
#include "tcgen05.cuh"

namespace daop {

constexpr int GB_M = 128, GB_N = 256, GB_K = 64, G_STAGES = 4;
constexpr int G_A_BYTES = GB_M * GB_K * 2;               // 16 KB
constexpr int G_B_BYTES = GB_N * GB_K * 2;               // 32 KB
constexpr int G_STAGE_BYTES = G_A_BYTES + G_B_BYTES;      // 48 KB
constexpr int G_THREADS = 192;
constexpr int G_MAX_EXPERTS = 64;
constexpr uint32_t G_IDESC = umma_idesc_bf16_f32(GB_M, GB_N);

// SwiGLU of the GEMM epilogues: hardware ex2 / fast divide (a few ulp in fp32,
// far below the bf16 rounding of act; the decode GEMV keeps silu_f32)
__device__ __forceinline__ float silu_fast(float a) { return __fdividef(a, 1.0f + __expf(-a)); }

struct GemmParams {
  const int64_t* offsets;  // [E+1] expert row offsets (device)
  const int32_t* slot_of;  // [E] HBM slot of each expert (device)
  int E;
  int k_blocks;    // K / 64
  int n_tiles;     // output tiles per expert
  int group_m;     // rasterisation group
  int b_tile_rows; // B row advance per n-tile (up: 128, down: 256)
  int b_half2;     // B row offset of the second 128-row box (up: ffn, down: 128)
  void* out;       // up: bf16 act (rows, out_ld); down: fp32 y (rows, out_ld)
  int64_t out_ld;
  int out_cols_per_tile;  // up: 128, down: 256
  int policy;             // L2 hint set (tuning): 0 A last/B normal, 1 both normal, 2 both last, 3 A normal/B last,
                          // 4 A first/B last, 5 A first/B normal, 6 A last/B first
  int raster;             // pair kernel tile order: 0 m-groups, 1 n-groups (see map_tile_pair)
  // L2 demotion at last use (pair kernel): operand lines loaded with
  // evict_last are switched back to evict_normal by the epilogue once no tile
  // of this launch reads them again, so the persisting set-aside is free for
  // the next expert's tiles instead of holding stale ones
  int demote;              // bit 0: A rows (raster 0), bit 1: B rows (raster 1)
  const uint16_t* a_ptr;   // A base (rows x a_ld bf16)
  int64_t a_ld;
  const uint16_t* b_ptr;   // B base of slot 0 (rows x b_ld bf16)
  int64_t b_ld;
  int64_t b_slot_stride;   // elements
  // expert-parallel return (down GEMM only, ep_p2p.cu): row r of the output
  // is stored at the address row_dst[r] (the source rank's y_back row, over
  // NVLink) instead of out + r * out_ld, and the CTA that finishes last
  // flags y[sig_rank] = sig_epoch on every peer workspace
  const uint64_t* row_dst;
  unsigned* sig_done;
  const uint64_t* sig_peers;
  int sig_G, sig_rank;
  unsigned sig_epoch;
  // fused combine (down GEMM, single GPU): after storing its y slice of
  // (row, n-tile), a thread counts it on the token's counter; the token's
  // last pick to land computes out = h + sum_j w_j y_j over that n-tile in
  // fixed j order (the combine kernel's arithmetic) -- no separate pass
  // A rows gathered by TMA (up GEMM, single GPU): sorted row r reads row
  // a_perm[r] / a_k of the token matrix (the permutation never materialises
  // x_perm); null = dense A rows
  const int32_t* a_perm;
  int a_k;
  int a_src_rows;
  const int32_t* comb_perm;  // sorted row -> t * k + j
  const int32_t* comb_inv;   // t * k + j -> sorted row
  const float* comb_h;       // (T, d) residual in
  const float* comb_w;       // (T, k) weights
  float* comb_out;           // (T, d)
  unsigned* comb_cnt;        // (T, n_tiles) zeroed once, self-resetting
  int comb_k;
  // dense GEMM (daop_gemm_bf16_f32: one "expert" of dense_rows rows, weight
  // slot 0, no device offset / slot tables) and an optional fp32 residual
  // added in the down epilogue: out = resid + A . B^T (resid may alias out)
  int64_t dense_rows;
  const float* resid;
  // split-K (dense GEMM, 256-row pair tile only): n_tiles counts ksplit x the
  // real n-tiles (tile n_eff -> k-slice n_eff / n_real, n-tile n_eff % n_real);
  // slice ks covers k-blocks [ks K / ksplit, (ks + 1) K / ksplit) and stores
  // its fp32 partial at out + ks * part_stride (resid is added by the
  // fixed-order reduction, dense_splitk_reduce_kernel)
  int ksplit;
  int64_t part_stride;
  // epilogue stores as streaming (st.global.cs: evict-first in L2) so the
  // 1.9 GB act / 1.1 GB y output streams do not push the re-read A / B
  // operand tiles out of L2 (tuning bit, daop_set_gemm_mode bit 14)
  int store_cs;
  // diagnostic bits (daop_set_gemm_mode bits 20..22; results are WRONG with
  // any set): 1 epilogue skips TMEM -> global, 2 producer skips the TMA loads
  // (MMAs on stale smem), 4 producer reloads the tile's own first 4 k-blocks
  // (L2-hot, spread over the L2 slices like the real operands).
  // They split a GEMM's time into MMA / operand feed / epilogue.
  int exp;
  // per-die tile schedule (pair kernel, B200's two dies; null = one die):
  // die_tab[smid] is the die of each SM; die_ctr (3 words, zeroed before the
  // launch) counts the clusters of each die and the arrivals.  Every cluster
  // takes a rank on its die; each expert's m-tiles are split between the dies
  // in proportion to their cluster counts, and a die's clusters stride only
  // over its own tiles -- so the A rows (and the act / y output) a die
  // re-reads stay in that die's L2 instead of crossing the die-to-die fabric.
  const int8_t* die_tab;
  unsigned* die_ctr;
  // which dimension the dies split: 0 the m-tiles (raster 0 keeps A groups
  // resident: each die holds its share of A), 1 the n-tiles (raster 1 keeps
  // weight groups resident: each die holds its share of B and streams A)
  int die_split_n;
  int no_stage;  // tuning: epilogue stores straight from the TMEM row layout (mode bit 19)
  int no_tmem_pipe;  // tuning: SwiGLU epilogue without overlapped TMEM reads (mode bit 23)
};

__device__ __forceinline__ int64_t off_at(const GemmParams& p, int e) {
  return p.offsets ? p.offsets[e] : (e == 0 ? 0 : p.dense_rows);
}
__device__ __forceinline__ int slot_at(const GemmParams& p, int e) {
  return p.slot_of ? p.slot_of[e] : 0;
}

// 32 accumulator columns -> fp32 row slice (+ the residual when given)
__device__ __forceinline__ void store_f32x32(float* out, const float* res, const uint32_t (&v)[32],
                                             bool cs) {
  float4* o = reinterpret_cast<float4*>(out);
  const float4* r = reinterpret_cast<const float4*>(res);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float4 a = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                           __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
    if (res) {
      const float4 b = r[i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    if (cs) __stcs(o + i, a);
    else o[i] = a;
  }
}

// the fused combine of one (row, n-tile): called by the row's thread after
// its y slice is stored and the accumulator released
__device__ __forceinline__ void fused_combine(const GemmParams& p, int64_t grow, int n,
                                              int parts) {
  __threadfence();  // this thread's y slice -> visible to the token's last pick
  const int k = p.comb_k;
  const int src = p.comb_perm[grow];
  const int64_t t = src / k;
  const int nt = p.n_tiles;
  // every pick's (row, n-tile) slice is stored in `parts` column pieces
  const unsigned old = atomicAdd(p.comb_cnt + t * nt + n, 1u);
  if (old != static_cast<unsigned>(k * parts - 1)) return;
  p.comb_cnt[t * nt + n] = 0;  // self-resetting for the next layer
  __threadfence();
  const int64_t d = p.out_ld;
  const float* y = static_cast<const float*>(p.out);
  const float4* hr = reinterpret_cast<const float4*>(p.comb_h + t * d + n * GB_N);
  float4* o = reinterpret_cast<float4*>(p.comb_out + t * d + n * GB_N);
  float wj[8];
  const float4* yr[8];
  for (int j = 0; j < k && j < 8; ++j) {
    wj[j] = p.comb_w[t * k + j];
    yr[j] = reinterpret_cast<const float4*>(y + static_cast<int64_t>(p.comb_inv[t * k + j]) * d +
                                            n * GB_N);
  }
#pragma unroll 4
  for (int c = 0; c < GB_N / 4; ++c) {
    float4 acc = __ldcg(hr + c);
    for (int j = 0; j < k && j < 8; ++j) {
      const float4 v = __ldcg(yr[j] + c);
      acc.x = fmaf(wj[j], v.x, acc.x);
      acc.y = fmaf(wj[j], v.y, acc.y);
      acc.z = fmaf(wj[j], v.z, acc.z);
      acc.w = fmaf(wj[j], v.w, acc.w);
    }
    o[c] = acc;
  }
}

// end-of-kernel EP signal: every thread fences its (remote) output stores,
// the last CTA to arrive publishes the flags
__device__ __forceinline__ void ep_gemm_signal_fence(const GemmParams& p) {
  if (p.sig_done) __threadfence_system();
}

__device__ __forceinline__ void ep_gemm_signal(const GemmParams& p) {
  if (p.sig_done && threadIdx.x == 0) {
    if (atomicAdd(p.sig_done, 1u) == gridDim.x - 1) {
      *p.sig_done = 0;
      __threadfence_system();
      for (int s = 0; s < p.sig_G; ++s)
        st_release_sys(reinterpret_cast<unsigned*>(p.sig_peers[s] + EP_FLAGS_Y) + p.sig_rank,
                       p.sig_epoch);
    }
  }
}

__device__ __forceinline__ void l2_demote_range(const void* p, int64_t bytes) {
  const char* c = static_cast<const char*>(p);
  for (int64_t o = 0; o < bytes; o += 128)
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(c + o) : "memory");
}

struct GemmSmem {
  uint64_t full[G_STAGES];
  uint64_t empty[G_STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int32_t prefix[G_MAX_EXPERTS + 1];  // tile prefix over experts
  int32_t mt[G_MAX_EXPERTS];           // m-tiles per expert
  int64_t off[G_MAX_EXPERTS + 1];
};

__device__ __forceinline__ bool map_tile(const GemmSmem& s, int E, int nt, int G, int t, int& e,
                                         int& m, int& n) {
  if (t >= s.prefix[E]) return false;
  e = 0;
  while (s.prefix[e + 1] <= t) ++e;
  const int u = t - s.prefix[e];
  const int grp = u / (G * nt);
  const int r = u - grp * G * nt;
  const int gm = min(G, s.mt[e] - grp * G);
  m = grp * G + r % gm;
  n = r / gm;
  return true;
}

template <bool SWIGLU>
__global__ void __launch_bounds__(G_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // SWIZZLE_128B needs 1024-byte aligned tiles
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  GemmSmem& s = *reinterpret_cast<GemmSmem*>(tiles + G_STAGES * G_STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = p.E;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < G_STAGES; ++i) {
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
    for (int e = 0; e <= E; ++e) s.off[e] = off_at(p, e);
    for (int e = 0; e < E; ++e) {
      // experts without an HBM slot (slow tier) get no tiles: their rows are
      // computed by the host tier and written into the output by the caller
      const int64_t me = slot_at(p, e) >= 0 ? s.off[e + 1] - s.off[e] : 0;
      s.mt[e] = static_cast<int>((me + GB_M - 1) / GB_M);
      acc += s.mt[e] * p.n_tiles;
      s.prefix[e + 1] = acc;
    }
  }
  if (warp == 2) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = s.tmem_base;
  const int nt = p.n_tiles, G = p.group_m;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      // weights are read by every concurrent CTA of the wave (they run the
      // m-tiles of one n-tile side by side): evict_first would evict a tile
      // after its first reader and re-fetch it from DRAM for every m-tile
      const uint64_t pol_a = l2_evict_last_policy();    // activations: re-read across n-tiles
      const uint64_t pol_b = l2_evict_normal_policy();
      int stage = 0;
      uint32_t phase = 0;
      int e, m, n;
      for (int t = blockIdx.x; map_tile(s, E, nt, G, t, e, m, n); t += gridDim.x) {
        const int row0 = static_cast<int>(s.off[e] + static_cast<int64_t>(m) * GB_M);
        const int slot = slot_at(p, e);
        const int brow = n * p.b_tile_rows;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          uint8_t* st = tiles + stage * G_STAGE_BYTES;
          mbar_arrive_expect_tx(&s.full[stage], G_STAGE_BYTES);
          tma_load_2d(st, &tmA, &s.full[stage], kb * GB_K, row0, pol_a);
          tma_load_3d(st + G_A_BYTES, &tmB, &s.full[stage], kb * GB_K, brow, slot, pol_b);
          tma_load_3d(st + G_A_BYTES + G_B_BYTES / 2, &tmB, &s.full[stage], kb * GB_K,
                      brow + p.b_half2, slot, pol_b);
          if (++stage == G_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      int e, m, n;
      for (int t = blockIdx.x; map_tile(s, E, nt, G, t, e, m, n); t += gridDim.x) {
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * GB_N;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&s.full[stage], phase);
          tc_fence_after();
          uint8_t* st = tiles + stage * G_STAGE_BYTES;
          const uint64_t adesc = umma_desc_sw128(smem_u32(st));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(st + G_A_BYTES));
#pragma unroll
          for (int k = 0; k < GB_K / 16; ++k)  // +32 bytes along K per UMMA_K=16
            umma_bf16(tmem_d, adesc + 2 * k, bdesc + 2 * k, G_IDESC, (kb | k) != 0);
          umma_commit(&s.empty[stage]);
          if (++stage == G_STAGES) {
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
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    int e, m, n;
    for (int t = blockIdx.x; map_tile(s, E, nt, G, t, e, m, n); t += gridDim.x) {
      mbar_wait(&s.tfull[acc], acc_phase);
      tc_fence_after();
      const int row_in_tile = q * 32 + lane;
      const int64_t me = s.off[e + 1] - s.off[e];
      const bool valid = static_cast<int64_t>(m) * GB_M + row_in_tile < me;
      const int64_t grow = s.off[e] + static_cast<int64_t>(m) * GB_M + row_in_tile;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * GB_N;
      if constexpr (SWIGLU) {
        uint16_t* out = static_cast<uint16_t*>(p.out) + grow * p.out_ld + n * 128;
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tb + c, g);
          tmem_ld32(tb + 128 + c, u);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = __uint_as_float(g[2 * i]), a1 = __uint_as_float(g[2 * i + 1]);
            const float b0 = __uint_as_float(u[2 * i]), b1 = __uint_as_float(u[2 * i + 1]);
            const float h0 = silu_fast(a0) * b0, h1 = silu_fast(a1) * b1;
            packed[i] = static_cast<uint32_t>(f32_to_bf16_bits(h0)) |
                        (static_cast<uint32_t>(f32_to_bf16_bits(h1)) << 16);
          }
          if (valid) {
            uint4* o = reinterpret_cast<uint4*>(out + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
            {
              const uint4 pk = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                                          packed[4 * i + 3]);
              if (p.store_cs) __stcs(o + i, pk);
              else o[i] = pk;
            }
          }
        }
      } else {
        float* out = p.row_dst ? (valid ? reinterpret_cast<float*>(p.row_dst[grow]) + n * GB_N
                                        : nullptr)
                               : static_cast<float*>(p.out) + grow * p.out_ld + n * GB_N;
        const float* resid = p.resid;  // (no split-K on the single-CTA kernel)
#pragma unroll 1
        for (int c = 0; c < GB_N; c += 32) {
          uint32_t v[32];
          tmem_ld32(tb + c, v);
          tmem_ld_wait();
          if (valid)
            store_f32x32(out + c, resid ? resid + grow * p.out_ld + n * GB_N + c : nullptr, v,
                         p.store_cs);
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
  ep_gemm_signal_fence(p);
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
  ep_gemm_signal(p);
}

// ---------------------------------------------------------------- host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return DAOP_ERR_CUDA;
  }
  cuuint64_t gd[3], gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gd, gs,
                   bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return DAOP_ERR_CUDA;
  }
  return DAOP_OK;
}

// ---------------------------------------------------------------- CTA-pair variant
//
// Same tiles, scheduled per CTA pair (cluster of 2 on one TPC) with
// tcgen05.mma.cta_group::2: the pair computes a 256 x 256 tile, each CTA
// loading its own 128 A rows and ONE of the two 128-row B boxes (up GEMM:
// the W1 box on the leader, the W3 box on the follower) -- so a stage is 32 KB
// per CTA instead of 48 KB (6 stages fit) and every B byte is fetched once per
// pair instead of once per CTA.  The leader issues the MMAs; both CTAs' TMA
// completions land on the leader's full barrier (2-SM TMA, peer bit cleared);
// commits are multicast to both CTAs; both CTAs' epilogues release the
// accumulator by remote-arriving on the leader's TMEM-empty barrier.
constexpr int P_M = 256;                                  // pair tile rows
constexpr int P_STAGES = 6;
constexpr int P_A_BYTES = 128 * GB_K * 2;                 // 16 KB per CTA
constexpr int P_B_BYTES = 128 * GB_K * 2;                 // 16 KB per CTA
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;      // 32 KB
constexpr uint32_t P_IDESC = umma_idesc_bf16_f32(P_M, GB_N);
// TWO_M variant: 512-row pair tile = two M=256 MMAs per k-step sharing the
// B box (each CTA holds 256 A rows: two 128-row boxes), so every B byte
// brought into shared memory feeds twice the MMA work and the operand
// traffic per FLOP drops by a quarter (the tile shape cuBLAS picks here);
// the two accumulators fill all 512 TMEM columns (no double buffering).
constexpr int P2_M = 512;
constexpr int P2_STAGES = 4;
constexpr int P2_STAGE_BYTES = 2 * P_A_BYTES + P_B_BYTES; // 48 KB

template <bool TWO_M, int EW = 8>
struct PairCfg {
  static constexpr int M = TWO_M ? P2_M : P_M;
  static constexpr int STAGES = TWO_M ? P2_STAGES : P_STAGES;
  static constexpr int STAGE_BYTES = TWO_M ? P2_STAGE_BYTES : P_STAGE_BYTES;
  static constexpr int A_BYTES = TWO_M ? 2 * P_A_BYTES : P_A_BYTES;
  static constexpr int NACC = TWO_M ? 1 : 2;  // TMEM accumulator buffers
  // TWO_M: EW = 8 or 16 epilogue warps (2 or 4 per TMEM lane quarter; each
  // drains one accumulator half, or a quarter of the columns) -- the MMAs of
  // the next tile wait for the single accumulator, so a faster drain is
  // tensor-pipe time
  static constexpr int EPI_WARPS = TWO_M ? EW : 4;
  static constexpr int GROUPS_PER_HALF = TWO_M ? EW / 8 : 1;  // warps per (quarter, half)
  static constexpr int THREADS = (2 + EPI_WARPS) * 32;
  // epilogue stores staged through a 2 KB shared buffer per warp (32 rows x
  // 64 B) so each store instruction writes 8 rows x 64 contiguous bytes
  // instead of 32 rows x 16 B (TMEM gives a thread one row); the 16-warp
  // variant has no shared memory left for it
  static constexpr bool STAGE_EPI = EPI_WARPS <= 8;
  static constexpr int STAGE_EPI_BYTES = STAGE_EPI ? EPI_WARPS * 2048 : 0;
};


struct PairSmem {
  uint64_t full[P_STAGES];
  uint64_t empty[P_STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int32_t prefix[G_MAX_EXPERTS + 1];
  int32_t mt[G_MAX_EXPERTS];   // m-tiles of expert e this CTA's schedule covers
  int32_t mlo[G_MAX_EXPERTS];  // first of them (per-die schedule; else 0)
  int32_t ntd[G_MAX_EXPERTS];  // n-tiles of expert e this CTA's schedule covers
  int32_t nlo[G_MAX_EXPERTS];  // first of them
  int64_t off[G_MAX_EXPERTS + 1];
  int32_t tcl, ncl;            // this cluster's first tile and the tile stride
  int32_t dinfo[4];            // per-die schedule: die, rank, clusters on die 0 / 1
};

// raster 0: groups of G m-tiles, m fastest (the wave shares one weight tile
//           across G m-tiles; the group's activation rows are re-read per n)
// raster 1: groups of G n-tiles, n fastest (the group's G weight tiles stay
//           L2-resident while every activation m-tile streams through once)
__device__ __forceinline__ bool map_tile_pair(const PairSmem& s, int E, int nt, int G,
                                              int raster, int t, int& e, int& m, int& n) {
  if (t >= s.prefix[E]) return false;
  e = 0;
  while (s.prefix[e + 1] <= t) ++e;
  const int u = t - s.prefix[e];
  nt = s.ntd[e];  // (this CTA's schedule: the die's n-tiles of expert e)
  if (raster == 0) {
    const int grp = u / (G * nt);
    const int r = u - grp * G * nt;
    const int gm = min(G, s.mt[e] - grp * G);
    m = s.mlo[e] + grp * G + r % gm;
    n = s.nlo[e] + r / gm;
  } else {
    const int mt = s.mt[e];
    const int grp = u / (G * mt);
    const int r = u - grp * G * mt;
    const int gn = min(G, nt - grp * G);
    n = s.nlo[e] + grp * G + r % gn;
    m = s.mlo[e] + r / gn;
  }
  return true;
}

// Warp-staged epilogue stores.  After tcgen05.ld.32x32b a lane holds one
// row; written straight out, every store instruction touches 32 rows x 16 B.
// Instead each lane parks 64 B of its row in the warp's 2 KB buffer (16-byte
// chunks XOR-swizzled by the row: conflict-free both ways) and the warp
// writes them back as 4 rounds of 8 rows x 64 contiguous bytes.
__device__ __forceinline__ uint32_t stg_off(int row, int chunk) {
  return static_cast<uint32_t>(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4));
}
__device__ __forceinline__ void stg_put(uint8_t* stg, int lane, const uint4 (&v)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) *reinterpret_cast<uint4*>(stg + stg_off(lane, j)) = v[j];
}
// round r: lane -> (row r * 8 + lane / 4, chunk lane % 4)
__device__ __forceinline__ uint4 stg_get(const uint8_t* stg, int r, int lane) {
  return *reinterpret_cast<const uint4*>(stg + stg_off(r * 8 + (lane >> 2), lane & 3));
}

// split-K decode of a tile's n index (GemmParams::ksplit)
__device__ __forceinline__ void split_tile(const GemmParams& p, int n_eff, int& n, int& ks, int& kb0,
                                           int& kb1) {
  if (p.ksplit <= 1) {
    n = n_eff;
    ks = 0;
    kb0 = 0;
    kb1 = p.k_blocks;
    return;
  }
  const int nr = p.n_tiles / p.ksplit;
  ks = n_eff / nr;
  n = n_eff - ks * nr;
  kb0 = ks * p.k_blocks / p.ksplit;
  kb1 = (ks + 1) * p.k_blocks / p.ksplit;
}

// QUAD (TWO_M only; tuning, off): a 4-CTA cluster = two CTA pairs on the same
// 512-row m-tile and neighbouring n-tiles (pair q takes n = 2 j + q).  Each A
// box is loaded once and multicast to the matching CTA of both pairs, so a CTA
// requests 16 KB of A + 16 KB of B per stage instead of 32 + 16 (L2 reads
// -33 %).  A stage is refilled only after BOTH pairs' MMAs released it.
// Measured: no gain -- only 33 four-CTA clusters fit the GPCs (132 SMs), and
// with L2-hot operands the per-SM feed is as slow as without multicast (the
// limit is the SM's ingress, ~36 B/clk, not L2 output).
// profiling aid (daop_gemm_timeline): global-timer stamps of each CTA of the
// pair kernel's last launch -- [entry, setup done (TMEM + cluster sync), last
// MMA commit (leader), last epilogue warp done, last accumulator-ready wait
// returned in an epilogue warp, fp32 path: last first-chunk TMEM load done]
constexpr int GT_CTAS = 512;
__device__ unsigned long long g_pair_tl[GT_CTAS][6];
__device__ int g_pair_tl_on;
__device__ __forceinline__ void pair_tl(int k) {
  if (g_pair_tl_on && blockIdx.x < GT_CTAS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&g_pair_tl[blockIdx.x][k], t);
  }
}

template <bool SWIGLU, bool TWO_M = false, int EW = 8, bool QUAD = false>
__global__ void __cluster_dims__(QUAD ? 4 : 2, 1, 1) __launch_bounds__(PairCfg<TWO_M, EW>::THREADS, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  pdl_prologue();  // (launched with launch_pdl)
  if (threadIdx.x == 0) pair_tl(0);
  static_assert(!QUAD || TWO_M, "QUAD multicast needs the 512-row pair tile");
  using C = PairCfg<TWO_M, EW>;
  constexpr int CL = QUAD ? 4 : 2;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* tiles = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
  PairSmem& s = *reinterpret_cast<PairSmem*>(tiles + C::STAGES * C::STAGE_BYTES);
  uint8_t* stage_epi = tiles + C::STAGES * C::STAGE_BYTES + (sizeof(PairSmem) + 127) / 128 * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;            // rank within the CTA pair
  const int pairq = static_cast<int>(crank >> 1);  // QUAD: which pair of the cluster
  const uint32_t lead_cta = crank & ~1u;      // this pair's leader CTA
  const bool leader = rank == 0;
  const int E = p.E;
  const int cluster = blockIdx.x / CL, nclusters = gridDim.x / CL;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&s.full[i], 2);   // leader: own expect_tx arrive + follower's remote arrive
      mbar_init(&s.empty[i], QUAD ? 2 : 1);  // multicast commit (QUAD: from both pairs)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.tfull[i], 1);   // multicast commit
      mbar_init(&s.tempty[i], 2 * C::EPI_WARPS);  // epilogue warps x 2 CTAs (leader's copy)
    }
    fence_mbar_init();
  }
  const bool per_die = !QUAD && p.die_tab != nullptr;
  if (per_die) {
    if (threadIdx.x == 0 && leader) {  // rank on this die; wait until every cluster has one
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      const int die = sm < 1024 && p.die_tab[sm] ? 1 : 0;  // (table: 1024 entries)
      const unsigned r = atomicAdd(p.die_ctr + die, 1u);
      __threadfence();
      atomicAdd(p.die_ctr + 2, 1u);
      while (ld_acquire_gpu(p.die_ctr + 2) < static_cast<unsigned>(nclusters)) {
      }
      s.dinfo[0] = die;
      s.dinfo[1] = static_cast<int>(r);
      s.dinfo[2] = static_cast<int>(ld_acquire_gpu(p.die_ctr));
      s.dinfo[3] = static_cast<int>(ld_acquire_gpu(p.die_ctr + 1));
    }
    cluster_sync_all();
    if (threadIdx.x == 0 && !leader) {  // the leader's rank (distributed shared memory)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t v;
        asm volatile(
            "{\n\t.reg .u32 ra;\n\t"
            "mapa.shared::cluster.u32 ra, %1, %2;\n\t"
            "ld.shared::cluster.u32 %0, [ra];\n\t}"
            : "=r"(v)
            : "r"(smem_u32(&s.dinfo[i])), "r"(lead_cta)
            : "memory");
        s.dinfo[i] = static_cast<int>(v);
      }
    }
  }
  if (threadIdx.x == 0) {
    int acc = 0;
    s.prefix[0] = 0;
    for (int e = 0; e <= E; ++e) s.off[e] = off_at(p, e);
    // per-die: expert e's m-tiles (or n-tiles, die_split_n) [0, split_e) go
    // to die 0, the rest to die 1, split_e from the running total so the
    // remainders spread over experts
    const int64_t n0 = per_die ? s.dinfo[2] : 1, nall = per_die ? s.dinfo[2] + s.dinfo[3] : 1;
    const int die = per_die ? s.dinfo[0] : 0;
    const bool by_n = per_die && p.die_split_n;
    const int nte = QUAD ? p.n_tiles / 2 : p.n_tiles;
    int64_t cum = 0;
    for (int e = 0; e < E; ++e) {
      const int64_t me = slot_at(p, e) >= 0 ? s.off[e + 1] - s.off[e] : 0;
      const int mte = static_cast<int>((me + C::M - 1) / C::M);
      const int units = by_n ? (mte > 0 ? nte : 0) : mte;
      const int a = static_cast<int>((cum * n0 + nall / 2) / nall);
      cum += units;
      const int b = static_cast<int>((cum * n0 + nall / 2) / nall);
      const int split = per_die ? b - a : units;  // die 0's share of this expert
      const int lo = die == 0 ? 0 : split, cnt = die == 0 ? split : units - split;
      s.mlo[e] = by_n ? 0 : lo;
      s.mt[e] = by_n ? (cnt > 0 ? mte : 0) : cnt;
      s.nlo[e] = by_n ? lo : 0;
      s.ntd[e] = by_n ? cnt : nte;
      acc += s.mt[e] * s.ntd[e];
      s.prefix[e + 1] = acc;
    }
    s.tcl = per_die ? s.dinfo[1] : cluster;
    s.ncl = per_die ? (die == 0 ? s.dinfo[2] : s.dinfo[3]) : nclusters;
  }
  if (warp == 2) tmem_alloc_pair<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x == 0) pair_tl(1);
  const uint32_t tmem_base = s.tmem_base;
  const int nt = QUAD ? p.n_tiles / 2 : p.n_tiles, G = p.group_m;

  if (warp == 0) {
    if (p.a_perm || lane == 0) {  // TMA producer (both CTAs; all lanes when gathering A)
      uint64_t pol_a = l2_evict_last_policy();
      uint64_t pol_b = l2_evict_normal_policy();  // shared by the wave's m-tiles
      if (p.policy == 1) pol_a = l2_evict_normal_policy();
      if (p.policy == 2) pol_b = l2_evict_last_policy();
      if (p.policy == 3) {
        pol_a = l2_evict_normal_policy();
        pol_b = l2_evict_last_policy();
      }
      if (p.policy == 4) {
        pol_a = l2_evict_first_policy();
        pol_b = l2_evict_last_policy();
      }
      if (p.policy == 5) {
        pol_a = l2_evict_first_policy();
        pol_b = l2_evict_normal_policy();
      }
      if (p.policy == 6) pol_b = l2_evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      int e, m, n;
      for (int t = s.tcl; map_tile_pair(s, E, nt, G, p.raster, t, e, m, n); t += s.ncl) {
        if (QUAD) n = 2 * n + pairq;
        int ks, kb0, kb1;
        split_tile(p, n, n, ks, kb0, kb1);
        const int row0 = static_cast<int>(s.off[e] + static_cast<int64_t>(m) * C::M) + rank * 128;
        const int slot = slot_at(p, e);
        const int brow = n * p.b_tile_rows + (leader ? 0 : p.b_half2);
        // gathered A: lane L fetches rows 4L .. 4L+3 of each 128-row box; the
        // token indices stay in registers for the whole tile (rows past the
        // matrix repeat a valid row; the epilogue never stores them)
        int gi[2][4];
        if (p.a_perm) {
          const int last = s.off[E] > 0 ? static_cast<int>(s.off[E]) - 1 : 0;
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              const int r = min(row0 + b * 256 + 4 * lane + q2, last);
              gi[b][q2] = p.a_perm[r] / p.a_k;
            }
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          if (lane == 0) mbar_wait(&s.empty[stage], phase ^ 1);
          if (p.a_perm) __syncwarp();  // (dense A: lane 0 runs this loop alone)
          uint8_t* st = tiles + stage * C::STAGE_BYTES;
          if (p.exp & 2) {
            if (lane == 0) {
              if (leader) mbar_arrive(&s.full[stage]);
              else mbar_arrive_cluster(&s.full[stage], lead_cta);
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(&s.full[stage], 2 * C::STAGE_BYTES);
            else mbar_arrive_cluster(&s.full[stage], lead_cta);
          }
          if (p.a_perm) {
            __syncwarp();  // the expect_tx precedes every lane's gather
            tma_gather4_pair(st + lane * 4 * GB_K * 2, &tmA, &s.full[stage], kb * GB_K,
                             gi[0][0], gi[0][1], gi[0][2], gi[0][3], pol_a);
            if constexpr (TWO_M)
              tma_gather4_pair(st + P_A_BYTES + lane * 4 * GB_K * 2, &tmA, &s.full[stage],
                               kb * GB_K, gi[1][0], gi[1][1], gi[1][2], gi[1][3], pol_a);
          } else if (lane == 0) {
            const int kx = (p.exp & 4) ? (kb & 3) * GB_K : kb * GB_K;  // diagnostic: L2-hot operands
            const int ra = row0;
            if constexpr (QUAD) {  // box `pairq` for this CTA and its twin in the other pair
              tma_load_2d_pair_mc(st + pairq * P_A_BYTES, &tmA, &s.full[stage], kx,
                                  ra + pairq * 256, static_cast<uint16_t>(0x5u << rank), pol_a);
            } else {
              tma_load_2d_pair(st, &tmA, &s.full[stage], kx, ra, pol_a);
              if constexpr (TWO_M)  // second M=256 half: tile rows 256 + rank * 128
                tma_load_2d_pair(st + P_A_BYTES, &tmA, &s.full[stage], kx, ra + 256, pol_a);
            }
          }
          if (lane == 0)
            tma_load_3d_pair(st + C::A_BYTES, &tmB, &s.full[stage], (p.exp & 4) ? (kb & 3) * GB_K : kb * GB_K,
                             brow, slot, pol_b);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {  // MMA issuer (leader only)
      int stage = 0, acc = 0, iters = 0;
      uint32_t phase = 0, acc_phase = 0;
      int e, m, n;
      for (int t = s.tcl; map_tile_pair(s, E, nt, G, p.raster, t, e, m, n); t += s.ncl) {
        if (QUAD) n = 2 * n + pairq;
        int ks, kb0, kb1;
        split_tile(p, n, n, ks, kb0, kb1);
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * GB_N;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&s.full[stage], phase);
          tc_fence_after();
          uint8_t* st = tiles + stage * C::STAGE_BYTES;
          const uint64_t adesc = umma_desc_sw128(smem_u32(st));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(st + C::A_BYTES));
#pragma unroll
          for (int k = 0; k < GB_K / 16; ++k) {
            umma_bf16_pair(tmem_d, adesc + 2 * k, bdesc + 2 * k, P_IDESC, ((kb - kb0) | k) != 0);
            if constexpr (TWO_M) {  // same B, second A half -> TMEM columns 256..511
              const uint64_t adesc1 = umma_desc_sw128(smem_u32(st + P_A_BYTES));
              umma_bf16_pair(tmem_d + GB_N, adesc1 + 2 * k, bdesc + 2 * k, P_IDESC,
                             ((kb - kb0) | k) != 0);
            }
          }
          umma_commit_pair(&s.empty[stage], QUAD ? 0xF : 0x3);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&s.tfull[acc], static_cast<uint16_t>(0x3u << (2 * pairq)));
        ++iters;
        if (++acc == C::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      pair_tl(2);
      // drain: wait until both epilogues released the last accumulator(s)
      for (int i = 0; i < C::NACC && i < iters; ++i) {
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        if (++acc == C::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int e, m, n;
    for (int t = s.tcl; map_tile_pair(s, E, nt, G, p.raster, t, e, m, n); t += s.ncl) {
      if (QUAD) n = 2 * n + pairq;
      int ks, kb0, kb1;
      split_tile(p, n, n, ks, kb0, kb1);
      mbar_wait(&s.tfull[acc], acc_phase);
      if (lane == 0) pair_tl(4);
      tc_fence_after();
      const int64_t me = s.off[e + 1] - s.off[e];
      const int grp = (warp - 2) >> 2;  // 0 .. EPI_WARPS / 4 - 1
      const int half = TWO_M ? grp / C::GROUPS_PER_HALF : 0;  // this warp's accumulator half
      const int sub = TWO_M ? grp % C::GROUPS_PER_HALF : 0;   // its share of the half's columns
      {
      const int row_in_tile = half * 256 + rank * 128 + q * 32 + lane;
      const bool valid = static_cast<int64_t>(m) * C::M + row_in_tile < me && !(p.exp & 1);
      const int64_t grow = s.off[e] + static_cast<int64_t>(m) * C::M + row_in_tile;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * GB_N +
                          half * GB_N;
      // staged stores: rows row0 .. row0 + 31 of the tile (this warp's lane
      // quarter); lane L writes row row0 + r * 8 + L / 4, bytes (L % 4) * 16
      const int64_t row0g = s.off[e] + static_cast<int64_t>(m) * C::M + half * 256 + rank * 128 + q * 32;
      const int64_t rows_left = me - (static_cast<int64_t>(m) * C::M + half * 256 + rank * 128 + q * 32);
      uint8_t* stg = stage_epi + (warp - 2) * 2048;
      // (SwiGLU never has row_dst; the fp32 path stages EP row returns too)
      const bool staged = C::STAGE_EPI && !p.no_stage && p.comb_cnt == nullptr &&
                          (!SWIGLU || p.row_dst == nullptr);
      if constexpr (SWIGLU) {
        if (staged) {
          uint16_t* outb = static_cast<uint16_t*>(p.out) + n * 128;
          // 32 SwiGLU outputs of this lane's row -> staging -> coalesced rows
          auto emit = [&](int c, const uint32_t (&g)[32], const uint32_t (&u)[32]) {
            uint4 pk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint32_t w[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int x = 8 * i + 2 * j;
                const float h0 = silu_fast(__uint_as_float(g[x])) * __uint_as_float(u[x]);
                const float h1 = silu_fast(__uint_as_float(g[x + 1])) * __uint_as_float(u[x + 1]);
                w[j] = static_cast<uint32_t>(f32_to_bf16_bits(h0)) |
                       (static_cast<uint32_t>(f32_to_bf16_bits(h1)) << 16);
              }
              pk[i] = make_uint4(w[0], w[1], w[2], w[3]);
            }
            __syncwarp();  // the previous chunk's reads of the buffer are done
            stg_put(stg, lane, pk);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = r * 8 + (lane >> 2);
              if (row < rows_left) {
                uint4* o = reinterpret_cast<uint4*>(outb + (row0g + row) * p.out_ld + c) + (lane & 3);
                const uint4 v = stg_get(stg, r, lane);
                if (p.store_cs) __stcs(o, v);
                else *o = v;
              }
            }
          };
          if (!(p.exp & 1) && !p.no_tmem_pipe) {
            // software-pipelined TMEM reads: the next 32 columns' tcgen05.ld
            // are in flight while this chunk's SwiGLU and stores run
            uint32_t ga[32], ua[32], gb[32], ub[32];
            tmem_ld32(tb, ga);
            tmem_ld32(tb + 128, ua);
            tmem_ld_wait();
            reg_fence(ga);
            reg_fence(ua);
            tmem_ld32(tb + 32, gb);
            tmem_ld32(tb + 160, ub);
            emit(0, ga, ua);
            tmem_ld_wait();
            reg_fence(gb);
            reg_fence(ub);
            tmem_ld32(tb + 64, ga);
            tmem_ld32(tb + 192, ua);
            emit(32, gb, ub);
            tmem_ld_wait();
            reg_fence(ga);
            reg_fence(ua);
            tmem_ld32(tb + 96, gb);
            tmem_ld32(tb + 224, ub);
            emit(64, ga, ua);
            tmem_ld_wait();
            reg_fence(gb);
            reg_fence(ub);
            emit(96, gb, ub);
          } else {
#pragma unroll 1
            for (int c = 0; c < 128 && !(p.exp & 1); c += 32) {
              uint32_t g[32], u[32];
              tmem_ld32(tb + c, g);
              tmem_ld32(tb + 128 + c, u);
              tmem_ld_wait();
              emit(c, g, u);
            }
          }
        } else {
        uint16_t* out = static_cast<uint16_t*>(p.out) + grow * p.out_ld + n * 128;
#pragma unroll 1
        for (int c = sub * (128 / C::GROUPS_PER_HALF);
             c < (sub + 1) * (128 / C::GROUPS_PER_HALF) && !(p.exp & 1); c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tb + c, g);
          tmem_ld32(tb + 128 + c, u);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float h0 = silu_fast(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
            const float h1 = silu_fast(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
            packed[i] = static_cast<uint32_t>(f32_to_bf16_bits(h0)) |
                        (static_cast<uint32_t>(f32_to_bf16_bits(h1)) << 16);
          }
          if (valid) {
            uint4* o = reinterpret_cast<uint4*>(out + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
            {
              const uint4 pk = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                                          packed[4 * i + 3]);
              if (p.store_cs) __stcs(o + i, pk);
              else o[i] = pk;
            }
          }
        }
        }
      } else if (staged) {
        // fp32 y (+ the residual): 32 accumulator columns = two 64-byte halves
        float* outf = static_cast<float*>(p.out) + ks * p.part_stride + n * GB_N;
        const float* resid = p.ksplit > 1 ? nullptr : p.resid;
#pragma unroll 1
        for (int c = sub * (GB_N / C::GROUPS_PER_HALF);
             c < (sub + 1) * (GB_N / C::GROUPS_PER_HALF) && !(p.exp & 1); c += 32) {
          uint32_t v[32];
          if (p.exp & 16) {  // diagnostic: staging + stores only
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = static_cast<uint32_t>(c + i + lane);
          } else {
            tmem_ld32(tb + c, v);
            tmem_ld_wait();
          }
          if (lane == 0 && c == sub * (GB_N / C::GROUPS_PER_HALF)) pair_tl(5);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint4 pk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              pk[i] = make_uint4(v[16 * hh + 4 * i], v[16 * hh + 4 * i + 1], v[16 * hh + 4 * i + 2],
                                 v[16 * hh + 4 * i + 3]);
            __syncwarp();
            stg_put(stg, lane, pk);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = r * 8 + (lane >> 2);
              if (row < rows_left) {
                const int64_t off = (row0g + row) * p.out_ld + c + 16 * hh + 4 * (lane & 3);
                const uint4 u4 = stg_get(stg, r, lane);
                float4 a = make_float4(__uint_as_float(u4.x), __uint_as_float(u4.y),
                                       __uint_as_float(u4.z), __uint_as_float(u4.w));
                if (resid) {
                  const float4 b = *reinterpret_cast<const float4*>(resid + n * GB_N + off);
                  a.x += b.x;
                  a.y += b.y;
                  a.z += b.z;
                  a.w += b.w;
                }
                // EP return: the row's slot on its source rank (peer memory)
                float4* o = p.row_dst
                                ? reinterpret_cast<float4*>(reinterpret_cast<float*>(p.row_dst[row0g + row]) +
                                                            n * GB_N + c + 16 * hh + 4 * (lane & 3))
                                : reinterpret_cast<float4*>(outf + off);
                if (p.exp & 8) continue;  // diagnostic: TMEM loads + staging only
                if (p.store_cs) __stcs(o, a);
                else *o = a;
              }
            }
          }
        }
      } else {
        float* out = p.row_dst ? (valid ? reinterpret_cast<float*>(p.row_dst[grow]) + n * GB_N
                                        : nullptr)
                               : static_cast<float*>(p.out) + ks * p.part_stride +
                                     grow * p.out_ld + n * GB_N;
        const float* resid = p.ksplit > 1 ? nullptr : p.resid;
#pragma unroll 1
        for (int c = sub * (GB_N / C::GROUPS_PER_HALF);
             c < (sub + 1) * (GB_N / C::GROUPS_PER_HALF) && !(p.exp & 1); c += 32) {
          uint32_t v[32];
          tmem_ld32(tb + c, v);
          tmem_ld_wait();
          if (valid)
            store_f32x32(out + c, resid ? resid + grow * p.out_ld + n * GB_N + c : nullptr, v,
                         p.store_cs);
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&s.tempty[acc], lead_cta);
      if constexpr (!SWIGLU) {
        if (p.comb_cnt) {  // accumulator released: the combine runs off the MMA's path
          const int row_in_tile = half * 256 + rank * 128 + q * 32 + lane;
          if (static_cast<int64_t>(m) * C::M + row_in_tile < me)
            fused_combine(p, s.off[e] + static_cast<int64_t>(m) * C::M + row_in_tile, n,
                          C::GROUPS_PER_HALF);
        }
      }
      if (p.demote && !TWO_M) {
        const int row_in_tile = rank * 128 + q * 32 + lane;
        const bool valid = static_cast<int64_t>(m) * C::M + row_in_tile < me;
        const int64_t grow = s.off[e] + static_cast<int64_t>(m) * C::M + row_in_tile;
        if ((p.demote & 1) && p.raster == 0 && n == s.nlo[e] + s.ntd[e] - 1 && valid)  // A m-tile done
          l2_demote_range(p.a_ptr + grow * p.a_ld, p.a_ld * 2);
        if ((p.demote & 2) && p.raster == 1 && m == s.mlo[e] + s.mt[e] - 1) {  // B n-tile done
          const int brow = n * p.b_tile_rows + (rank == 0 ? 0 : p.b_half2) + q * 32 + lane;
          l2_demote_range(p.b_ptr + static_cast<int64_t>(slot_at(p, e)) * p.b_slot_stride +
                              static_cast<int64_t>(brow) * p.b_ld,
                          p.b_ld * 2);
        }
      }
      if (++acc == C::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) pair_tl(3);
  }
  tc_fence_before();
  ep_gemm_signal_fence(p);
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
  ep_gemm_signal(p);
}

static int g_gemm_mode = 0;    // 0: CTA pair (default), 1: single CTA
static int g_gemm_policy = -1;  // L2 hint set override (tuning); -1 = per-GEMM default
static int g_gemm_demote = 0;   // bit 0: demote A (up), bit 1: demote B (down)

static size_t gemm_smem_bytes() { return 1024 + G_STAGES * G_STAGE_BYTES + sizeof(GemmSmem); }
// bit 0: up GEMM, bit 1: down GEMM use the 512-row pair tile.  Default: both
// (down: sustained 5.6-6.0 vs 6.2-6.7 ms on 8 x 4096 tokens, DRAM 13 vs 28 GB;
// up, with 8 epilogue warps and the fast SwiGLU: 11.8 vs 12.0 ms; whole layer
// 19.2 vs 19.6 ms -- profiles/r01/gemm_two_m.txt)
static int g_gemm_two_m = 3;
static int g_gemm_store_cs = 0;  // epilogue streaming stores (tuning)
static int g_gemm_dense_skinny = 1;  // tuning: small-M dense GEMMs on the skinny kernel
static int g_gemm_epi16 = 0;  // tuning: 16 epilogue warps for the 512-row pair tile
// persisting L2 set-aside for the evict_last operand loads: OFF by default.
// With it on (mode bit 11), the GEMMs' persisting lines stay in L2 after the
// GEMM and the HBM-bound kernels that follow slow down ~2x (router 160 -> 299
// us, permutation 157 -> 331, combine 328 -> 568 at configs[3]); the GEMMs do
// not gain from it (scripts/persist_ab.py: layer 17.70 -> 17.16 ms off)
static int g_gemm_persist_off = 1;
static int g_gemm_splitk = 1;
static int g_gemm_nostage = 0;  // tuning: unstaged epilogue stores (mode bit 19)
static int g_gemm_no_tmem_pipe = 0;  // tuning: SwiGLU epilogue TMEM reads not overlapped (bit 23)
static int g_gemm_exp = 0;  // EXPERIMENT bits (GemmParams::exp)
static int g_gemm_quad = 0;  // tuning: 4-CTA multicast clusters for the 512-row pair tile (mode bit 18)  // tuning: split-K for prompt-sized dense projections (_ws entry)

// per-die tile schedule (GemmParams::die_tab): the device table of each SM's
// die and a ring of per-launch counters.  g_die_mode: -1 auto (the measured
// map, daop_die_map, when it finds two dies), 0 off, 1 the table set by
// daop_set_gemm_die_table.
static int g_die_mode = -1;
static std::mutex g_die_mu;
static std::vector<int8_t> g_die_host;  // custom table (mode 1)
struct DieState {
  int8_t* tab = nullptr;
  unsigned* ctr = nullptr;
  int slot = 0;
  int mode = -2;  // g_die_mode the table was built for
  bool on = false;
};
static DieState g_die_state[64];
constexpr int DIE_SLOTS = 64;

// (table, zeroed counters) for a launch on `st`, or nullptrs when off
static int die_schedule(cudaStream_t st, const int8_t** tab, unsigned** ctr) {
  *tab = nullptr;
  *ctr = nullptr;
  static const bool env_off = [] {
    const char* v = getenv("DAOP_GEMM_DIE");  // "0": plain schedule (A/B runs)
    return v && v[0] == '0';
  }();
  if (g_die_mode == 0 || (env_off && g_die_mode < 0)) return DAOP_OK;
  int dev = 0;
  DAOP_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return DAOP_OK;
  std::lock_guard<std::mutex> lk(g_die_mu);
  DieState& d = g_die_state[dev];
  if (d.mode != g_die_mode) {
    // the probe synchronises the device: never inside a stream capture (this
    // launch runs the plain schedule; the next one outside a capture probes)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      (void)cudaGetLastError();
      return DAOP_OK;
    }
    const int n = sm_count();
    std::vector<int8_t> h(static_cast<size_t>(n), 0);
    bool two = false;
    if (g_die_mode == 1) {
      for (int i = 0; i < n && i < static_cast<int>(g_die_host.size()); ++i) h[i] = g_die_host[i] ? 1 : 0;
      two = true;
    } else {
      std::vector<int32_t> m(static_cast<size_t>(n));
      int32_t nd = 1;
      if (daop_die_map(m.data(), n, &nd) == DAOP_OK && nd == 2) {
        for (int i = 0; i < n; ++i) h[i] = static_cast<int8_t>(m[i]);
        two = true;
      }
    }
    if (!d.tab) DAOP_CUDA(cudaMalloc(&d.tab, 1024));
    if (!d.ctr) DAOP_CUDA(cudaMalloc(&d.ctr, DIE_SLOTS * 4 * sizeof(unsigned)));
    DAOP_CUDA(cudaMemcpy(d.tab, h.data(), h.size(), cudaMemcpyHostToDevice));
    d.on = two;
    d.mode = g_die_mode;
  }
  if (!d.on) return DAOP_OK;
  unsigned* c = d.ctr + 4 * d.slot;
  d.slot = (d.slot + 1) % DIE_SLOTS;  // concurrent launches on other streams get other slots
  DAOP_CUDA(cudaMemsetAsync(c, 0, 4 * sizeof(unsigned), st));
  *tab = d.tab;
  *ctr = c;
  return DAOP_OK;
}

// co-resident clusters of a pair-kernel instantiation (the per-die schedule
// waits for every cluster of the launch)
static int max_active_clusters(const void* kern, int cl, int threads, size_t smem, int want) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * want);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cl;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    return want;
  }
  return n < want ? n : want;
}

template <bool TWO_M, int EW = 8>
static size_t pair_smem_bytes() {
  using C = PairCfg<TWO_M, EW>;
  return 1024 + C::STAGES * C::STAGE_BYTES + (sizeof(PairSmem) + 127) / 128 * 128 +
         C::STAGE_EPI_BYTES;
}

template <bool SWIGLU, bool TWO_M, int EW, bool QUAD = false>
static int launch_pair_ew(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                          int64_t rows_total, cudaStream_t st) {
  using C = PairCfg<TWO_M, EW>;
  constexpr int CL = QUAD ? 4 : 2;
  const size_t smem = pair_smem_bytes<TWO_M, EW>();
  auto kern = grouped_gemm_pair_kernel<SWIGLU, TWO_M, EW, QUAD>;
  DAOP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const int64_t max_tiles =
      (rows_total / C::M + p.E) * static_cast<int64_t>(QUAD ? p.n_tiles / 2 : p.n_tiles);
  int clusters = sm_count() / CL;
  if (QUAD) {
    // 4-CTA clusters must fit inside a GPC: launch only the co-resident ones
    // (a persistent grid with a second wave of clusters doubles the tail)
    static int max_active = 0;
    if (!max_active) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL * clusters);
      cfg.blockDim = dim3(C::THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = CL;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        n = clusters;
      }
      max_active = n;
      if (getenv("DAOP_GEMM_VERBOSE")) fprintf(stderr, "quad gemm: %d co-resident 4-CTA clusters\n", n);
    }
    if (max_active < clusters) clusters = max_active;
  }
  if (max_tiles < clusters) clusters = static_cast<int>(max_tiles < 1 ? 1 : max_tiles);
  GemmParams pp = p;
  // per-die schedule for the big grouped GEMMs only: with few m-tiles (prompt-
  // sized dense projections, split-K) a die would get no tiles
  if (!QUAD && p.ksplit <= 1 && rows_total / C::M >= 16) {
    int rc = die_schedule(st, &pp.die_tab, &pp.die_ctr);
    if (rc) return rc;
    if (pp.die_tab) {
      static int co[2] = {0, 0};  // per SWIGLU instantiation family (same smem / threads)
      int& c = co[TWO_M ? 1 : 0];
      if (!c) c = max_active_clusters(reinterpret_cast<const void*>(kern), CL, C::THREADS, smem,
                                      sm_count() / CL);
      if (c < clusters) clusters = c;
    }
  }
  pp.store_cs = g_gemm_store_cs;
  pp.exp = g_gemm_exp;
  pp.no_stage = g_gemm_nostage;
  pp.no_tmem_pipe = g_gemm_no_tmem_pipe;
  if (p.group_m < 0) {  // negative group = n-grouped raster of |group| weight tiles
    pp.raster = 1;
    pp.group_m = QUAD ? (-p.group_m > 1 ? -p.group_m / 2 : 1) : -p.group_m;  // (QUAD: n-pairs)
  } else {              // group counted in 128-row units -> pair tiles of C::M rows
    pp.raster = 0;
    pp.group_m = p.group_m > C::M / 128 ? p.group_m / (C::M / 128) : 1;
  }
  pp.die_split_n = pp.raster == 1;
  DAOP_CUDA(launch_pdl(kern, dim3(CL * clusters), dim3(C::THREADS), smem, st, ta, tb, pp));
  DAOP_CHECK_LAUNCH(SWIGLU ? "grouped_gemm_pair_up" : "grouped_gemm_pair_down");
  return DAOP_OK;
}

template <bool SWIGLU, bool TWO_M>
static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                       int64_t rows_total, cudaStream_t st) {
  if constexpr (TWO_M) {
    // 4-CTA clusters with A multicast across two pairs (plain prefill GEMMs)
    const bool quad = g_gemm_quad && p.n_tiles % 2 == 0 && !p.a_perm && !p.row_dst &&
                      !p.comb_cnt && p.ksplit <= 1;
    if (quad) {
      if (g_gemm_epi16) return launch_pair_ew<SWIGLU, TWO_M, 16, true>(ta, tb, p, rows_total, st);
      return launch_pair_ew<SWIGLU, TWO_M, 8, true>(ta, tb, p, rows_total, st);
    }
    if (g_gemm_epi16) return launch_pair_ew<SWIGLU, TWO_M, 16>(ta, tb, p, rows_total, st);
  }
  return launch_pair_ew<SWIGLU, TWO_M, 8>(ta, tb, p, rows_total, st);
}

// Default rasterisation groups.  Up GEMM (m-grouped): the group's A rows
// (group x 128 rows x d x 2 B) are re-read by every n-tile of the group and
// must stay in the die's L2 (the per-die schedule splits each expert's
// m-tiles between the dies first).  Down GEMM (n-grouped): 16 W2 tiles.
// DAOP_GEMM_GROUPS="up,down" overrides both (tuning).
static int default_group_up(int d) {
  static const int env = [] {
    const char* v = getenv("DAOP_GEMM_GROUPS");
    return v ? atoi(v) : 0;
  }();
  if (env) return env;
  // with the per-die schedule a die's group of an expert's A rows should stay
  // near 32 MB: 8x7B (d 4096) keeps the whole per-die range (4096 rows, 32 MB);
  // 8x22B (d 6144) groups 2048 rows (25 MB per die group): up 18.6 -> 17.9 ms,
  // DRAM reads 37-42 -> 23-28 GB (profiles/r02/die/ncu_ep_groups.txt)
  return d > 5120 ? 16 : 64;
}
static int default_group_down(int ffn) {
  static const int env = [] {
    const char* v = getenv("DAOP_GEMM_GROUPS");
    const char* c = v ? strchr(v, ',') : nullptr;
    return c ? atoi(c + 1) : 0;
  }();
  if (env) return env;
  return (g_gemm_two_m & 2) ? -16 : -8;  // (8x22B: -16 9.10-9.15 vs -8 9.24 ms, per-die schedule)
}

static void apply_persisting_l2() {
  {
    // L2::evict_last (the A operand, re-read by every n-tile of its group) is
    // only honoured inside the persisting L2 set-aside, which defaults to 0
    // (tuning bit: g_gemm_persist_off leaves / resets it to 0)
    static int applied[64];
    static bool init = false;
    if (!init) {
      for (int i = 0; i < 64; ++i) applied[i] = -1;
      init = true;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64) {
      int want = 0;
      if (!g_gemm_persist_off)
        cudaDeviceGetAttribute(&want, cudaDevAttrMaxPersistingL2CacheSize, dev);
      if (applied[dev] != want) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        cudaGetLastError();
        applied[dev] = want;
      }
    }
  }
}

template <bool SWIGLU>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                       int64_t rows_total, cudaStream_t st) {
  apply_persisting_l2();
  if (g_gemm_demote & 4) cudaCtxResetPersistingL2Cache();  // tuning: start from a clean set-aside
  if (g_gemm_mode == 0) {
    const bool two = (g_gemm_two_m >> (SWIGLU ? 0 : 1)) & 1;
    return two ? launch_pair<SWIGLU, true>(ta, tb, p, rows_total, st)
               : launch_pair<SWIGLU, false>(ta, tb, p, rows_total, st);
  }
  const size_t smem = gemm_smem_bytes();
  DAOP_CUDA(cudaFuncSetAttribute(grouped_gemm_kernel<SWIGLU>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const int64_t max_tiles = (rows_total / GB_M + p.E) * static_cast<int64_t>(p.n_tiles);
  int grid = sm_count();
  if (max_tiles < grid) grid = static_cast<int>(max_tiles < 1 ? 1 : max_tiles);
  GemmParams q = p;
  if (q.group_m <= 0) q.group_m = 16;  // the single-CTA kernel only has m-grouped rasters
  grouped_gemm_kernel<SWIGLU><<<grid, G_THREADS, smem, st>>>(ta, tb, q);
  DAOP_CHECK_LAUNCH(SWIGLU ? "grouped_gemm_up" : "grouped_gemm_down");
  return DAOP_OK;
}

}  // namespace daop

using namespace daop;

static int check_ffn_shape(int64_t rows, int32_t d, int32_t ffn, int32_t E) {
  if (E < 1 || E > G_MAX_EXPERTS || d % 256 != 0 || ffn % 128 != 0 || d < 64 || ffn < 64 ||
      rows >= (1ll << 31)) {
    set_error("expert GEMM: unsupported shape (rows=%lld d=%d ffn=%d E=%d): needs d %% 256 == 0, "
              "ffn %% 128 == 0, E <= %d",
              static_cast<long long>(rows), d, ffn, E, G_MAX_EXPERTS);
    return DAOP_ERR_UNSUPPORTED;
  }
  return DAOP_OK;
}

// device-wide GEMM setup (the persisting-L2 limit) outside any stream
// capture: a CUDA graph that captures the GEMMs calls this first
extern "C" int daop_gemm_prepare() {
  apply_persisting_l2();
  return DAOP_OK;
}

// per-die tile schedule of the CTA-pair GEMMs: n == 0 off, n < 0 the measured
// SM -> die map (daop_die_map), n > 0 the given table (die of SM i = tab[i])
extern "C" int daop_set_gemm_die_table(const int32_t* tab, int32_t n) {
  if (n > 1024) {
    set_error("gemm die table: %d entries (max 1024)", n);
    return DAOP_ERR_CONFIG;
  }
  if (n == 0) {
    g_die_mode = 0;
  } else if (n < 0) {
    g_die_mode = -1;
  } else {
    g_die_host.assign(tab, tab + n);
    g_die_mode = 1;
    for (auto& d : g_die_state) d.mode = -2;  // rebuild the device table
  }
  return DAOP_OK;
}

extern "C" int daop_set_gemm_mode(int32_t mode) {
  // low nibble: kernel (0 CTA pair, 1 single CTA); bits 4..6: L2 hint set (tuning)
  if ((mode & 15) > 1 || ((mode >> 4) & 15) > 6) {
    set_error("gemm mode must be kernel (0 pair / 1 single) | policy << 4");
    return DAOP_ERR_CONFIG;
  }
  g_gemm_mode = mode & 15;
  g_gemm_policy = ((mode >> 4) & 15) ? ((mode >> 4) & 15) : -1;
  g_gemm_demote = (mode >> 8) & 7;
  g_gemm_persist_off = !((mode >> 11) & 1);  // bit 11: persisting set-aside ON (tuning)
  g_gemm_two_m = ((mode >> 12) & 3) ^ 3;  // mode bits flip the default (tuning)
  g_gemm_store_cs = (mode >> 14) & 1;
  g_gemm_dense_skinny = !((mode >> 15) & 1);
  g_gemm_epi16 = (mode >> 16) & 1;
  g_gemm_splitk = !((mode >> 17) & 1);
  // exp bit 3: no fp32 y stores, bit 4: no fp32 TMEM loads (diagnostics)
  g_gemm_exp = ((mode >> 20) & 7) | (((mode >> 24) & 3) << 3);
  g_gemm_quad = (mode >> 18) & 1;
  g_gemm_nostage = (mode >> 19) & 1;
  g_gemm_no_tmem_pipe = (mode >> 23) & 1;
  return DAOP_OK;
}

extern "C" int daop_expert_gemm_up(const uint16_t* x_perm, int64_t rows, int32_t d, int32_t ffn,
                                   const uint16_t* slab, int64_t n_slots,
                                   int64_t slot_stride_elems, const int64_t* d_offsets,
                                   const int32_t* d_slot_of, int32_t E, uint16_t* act,
                                   int32_t group_m, daop_stream_t stream) {
  int rc = check_ffn_shape(rows, d, ffn, E);
  if (rc) return rc;
  if (rows == 0) return DAOP_OK;
  CUtensorMap ta, tb;
  const uint64_t adims[2] = {static_cast<uint64_t>(d), static_cast<uint64_t>(rows)};
  const uint64_t astr[1] = {static_cast<uint64_t>(d) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, x_perm, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(d), static_cast<uint64_t>(2 * ffn),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t bstr[2] = {static_cast<uint64_t>(d) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  if ((rc = make_tmap_bf16(&tb, slab, 3, bdims, bstr, bbox))) return rc;
  GemmParams p{d_offsets, d_slot_of, E, d / GB_K, ffn / 128, group_m > 0 ? group_m : default_group_up(d),
               128, ffn, act, ffn, 128, g_gemm_policy >= 0 ? g_gemm_policy : 0, 0,
               g_gemm_demote & 1, x_perm, d, slab, d, slot_stride_elems};
  return launch_gemm<true>(ta, tb, p, rows, as_stream(stream));
}

// Up GEMM reading its A rows straight from the token matrix x (T_src, d)
// through TMA row gathers (sorted row r = token perm[r] / k): the
// permutation's gather pass and x_perm disappear from the prefill.
extern "C" int daop_expert_gemm_up_gather(const uint16_t* x, int64_t src_rows,
                                          const int32_t* d_perm, int32_t k, int64_t rows,
                                          int32_t d, int32_t ffn, const uint16_t* slab,
                                          int64_t n_slots, int64_t slot_stride_elems,
                                          const int64_t* d_offsets, const int32_t* d_slot_of,
                                          int32_t E, uint16_t* act, int32_t group_m,
                                          daop_stream_t stream) {
  int rc = check_ffn_shape(rows, d, ffn, E);
  if (rc) return rc;
  if (g_gemm_mode != 0 || k < 1 || src_rows < 1) {
    set_error("gathered up GEMM: needs the CTA-pair kernel (mode %d), k >= 1, rows >= 1",
              g_gemm_mode);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (rows == 0) return DAOP_OK;
  CUtensorMap ta, tb;
  const uint64_t adims[2] = {static_cast<uint64_t>(d), static_cast<uint64_t>(src_rows)};
  const uint64_t astr[1] = {static_cast<uint64_t>(d) * 2};
  const uint32_t abox[2] = {GB_K, 1};  // gather4: 4 rows of one 64-element box each
  if ((rc = make_tmap_bf16(&ta, x, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(d), static_cast<uint64_t>(2 * ffn),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t bstr[2] = {static_cast<uint64_t>(d) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  if ((rc = make_tmap_bf16(&tb, slab, 3, bdims, bstr, bbox))) return rc;
  GemmParams p{d_offsets, d_slot_of, E, d / GB_K, ffn / 128, group_m > 0 ? group_m : default_group_up(d),
               128, ffn, act, ffn, 128, g_gemm_policy >= 0 ? g_gemm_policy : 0, 0,
               g_gemm_demote & 1, x, d, slab, d, slot_stride_elems};
  p.a_perm = d_perm;
  p.a_k = k;
  p.a_src_rows = static_cast<int>(src_rows);
  return launch_gemm<true>(ta, tb, p, rows, as_stream(stream));
}

extern "C" int daop_expert_gemm_down(const uint16_t* act, int64_t rows, int32_t d, int32_t ffn,
                                     const uint16_t* slab, int64_t n_slots,
                                     int64_t slot_stride_elems, const int64_t* d_offsets,
                                     const int32_t* d_slot_of, int32_t E, float* y,
                                     int32_t group_m, daop_stream_t stream) {
  int rc = check_ffn_shape(rows, d, ffn, E);
  if (rc) return rc;
  if (rows == 0) return DAOP_OK;
  CUtensorMap ta, tb;
  const uint64_t adims[2] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(rows)};
  const uint64_t astr[1] = {static_cast<uint64_t>(ffn) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, act, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(d),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t bstr[2] = {static_cast<uint64_t>(ffn) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  const uint16_t* w2 = slab + static_cast<int64_t>(2) * ffn * d;
  if ((rc = make_tmap_bf16(&tb, w2, 3, bdims, bstr, bbox))) return rc;
  // default: n-grouped raster, 16 weight n-tiles per group with the 512-row
  // tile (8 with the 256-row one); profiles/r01/gemm_two_m.txt, gemm_sweep.txt
  const int grp = group_m != 0 ? group_m : default_group_down(ffn);
  GemmParams p{d_offsets, d_slot_of, E, ffn / GB_K, d / GB_N, grp,
               GB_N, 128, y, d, GB_N, g_gemm_policy >= 0 ? g_gemm_policy : 2, 0,
               g_gemm_demote & 2, act, ffn, w2, ffn, slot_stride_elems};
  return launch_gemm<false>(ta, tb, p, rows, as_stream(stream));
}

int skinny_dense_gemm(const uint16_t* a, int64_t M, int32_t K, const uint16_t* w, int32_t N,
                      const float* resid, float* out, cudaStream_t st);

// Dense projection on the same tcgen05 pipeline (the prompt attention's QKV
// and O projections, attention.py): out (M, N) fp32 = A (M, K) bf16 . W^T,
// W (N, K) bf16 row-major, optionally + resid (M, N) fp32 (may alias out).
// One "expert" of M rows without device tables; N % 256 == 0, K % 64 == 0.
extern "C" int daop_gemm_bf16_f32(const uint16_t* a, int64_t M, int32_t K, const uint16_t* w,
                                  int32_t N, const float* resid, float* out,
                                  daop_stream_t stream) {
  if (M < 0 || M >= (1ll << 31) || K < 64 || K % GB_K != 0 || N < GB_N || N % GB_N != 0) {
    set_error("dense GEMM: unsupported shape (M=%lld K=%d N=%d): needs K %% 64 == 0, "
              "N %% 256 == 0", static_cast<long long>(M), K, N);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (M == 0) return DAOP_OK;
  // prompt-sized M: the swap-AB skinny kernel (weights as the MMA M side), so
  // the weight tiles spread over every SM instead of N / 256 CTA pairs
  if (M <= 768 && g_gemm_dense_skinny)
    return skinny_dense_gemm(a, M, K, w, N, resid, out, as_stream(stream));
  CUtensorMap ta, tb;
  int rc;
  const uint64_t adims[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(M)};
  const uint64_t astr[1] = {static_cast<uint64_t>(K) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, a, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), 1};
  const uint64_t bstr[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * N * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  if ((rc = make_tmap_bf16(&tb, w, 3, bdims, bstr, bbox))) return rc;
  const int grp = (g_gemm_two_m & 2) ? -16 : -8;
  GemmParams p{nullptr, nullptr, 1, K / GB_K, N / GB_N, grp, GB_N, 128, out, N,
               GB_N, g_gemm_policy >= 0 ? g_gemm_policy : 2, 0, 0, a, K, w, K,
               static_cast<int64_t>(K) * N};
  p.dense_rows = M;
  p.resid = resid;
  return launch_gemm<false>(ta, tb, p, M, as_stream(stream));
}

// fixed-order reduction of the split-K partials: out = [resid +] p_0 + p_1 + ...
__global__ void __launch_bounds__(256) dense_splitk_reduce_kernel(const float4* parts, int ksplit,
                                                                  int64_t stride4,
                                                                  const float4* resid,
                                                                  float4* out, int64_t n4) {
  pdl_prologue();  // (launched with launch_pdl)
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = resid ? resid[i] : parts[i];
    for (int ks = resid ? 0 : 1; ks < ksplit; ++ks) {
      const float4 b = parts[ks * stride4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    out[i] = a;
  }
}

// Prompt-sized dense projections (M <= 256 rows: one 256-row CTA-pair tile
// of N / 256 n-tiles, fewer than the SM pairs): split K over the idle pairs,
// fp32 partials into the caller's workspace, then one fixed-order reduction
// pass (+ the residual).  Otherwise daop_gemm_bf16_f32.
extern "C" int daop_gemm_bf16_f32_ws(const uint16_t* a, int64_t M, int32_t K, const uint16_t* w,
                                     int32_t N, const float* resid, float* out, float* ws,
                                     int64_t ws_bytes, daop_stream_t stream) {
  if (M < 0 || M >= (1ll << 31) || K < 64 || K % GB_K != 0 || N < GB_N || N % GB_N != 0) {
    set_error("dense GEMM: unsupported shape (M=%lld K=%d N=%d): needs K %% 64 == 0, "
              "N %% 256 == 0", static_cast<long long>(M), K, N);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (M == 0) return DAOP_OK;
  const int n_real = N / GB_N, kb = K / GB_K;
  int ksplit = M <= P_M ? (sm_count() / 2) / n_real : 1;
  if (ksplit > 8) ksplit = 8;
  if (ksplit > kb / 4) ksplit = kb / 4;
  if (ksplit < 2 || g_gemm_mode != 0 || !g_gemm_splitk || !ws ||
      ws_bytes < static_cast<int64_t>(ksplit) * M * N * 4)
    return daop_gemm_bf16_f32(a, M, K, w, N, resid, out, stream);
  CUtensorMap ta, tb;
  int rc;
  const uint64_t adims[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(M)};
  const uint64_t astr[1] = {static_cast<uint64_t>(K) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, a, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), 1};
  const uint64_t bstr[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * N * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  if ((rc = make_tmap_bf16(&tb, w, 3, bdims, bstr, bbox))) return rc;
  GemmParams p{nullptr, nullptr, 1, kb, n_real * ksplit, -16, GB_N, 128, ws, N,
               GB_N, g_gemm_policy >= 0 ? g_gemm_policy : 2, 0, 0, a, K, w, K,
               static_cast<int64_t>(K) * N};
  p.dense_rows = M;
  p.ksplit = ksplit;
  p.part_stride = M * static_cast<int64_t>(N);
  apply_persisting_l2();
  cudaStream_t st = as_stream(stream);
  if ((rc = launch_pair<false, false>(ta, tb, p, M, st))) return rc;
  const int64_t n4 = M * static_cast<int64_t>(N) / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
  DAOP_CUDA(launch_pdl(dense_splitk_reduce_kernel, dim3(static_cast<int>(blocks)), dim3(256), 0, st, 
      reinterpret_cast<const float4*>(ws), ksplit, p.part_stride / 4,
      reinterpret_cast<const float4*>(resid), reinterpret_cast<float4*>(out), n4));
  DAOP_CHECK_LAUNCH("dense_splitk_reduce");
  return DAOP_OK;
}

// Down GEMM with the combine fused into its epilogue (single GPU prefill;
// measured 0.7 ms per 8 x 4096-token layer SLOWER than GEMM + bulk combine
// kernel -- the last picks' combine loads delay the single-accumulator
// epilogue -- so MoEBlockEngine.prefill keeps the separate pass by default):
// y (rows, d) fp32 is still written (the first picks of a token park their
// slice there); out (T, d) = h + sum_j w_j y_j is written by each token's last
// pick per n-tile.  cnt: (T, d / 256) u32, zeroed once, self-resetting.
extern "C" int daop_expert_gemm_down_combine(const uint16_t* act, int64_t rows, int32_t d,
                                             int32_t ffn, const uint16_t* slab, int64_t n_slots,
                                             int64_t slot_stride_elems, const int64_t* d_offsets,
                                             const int32_t* d_slot_of, int32_t E, float* y,
                                             const int32_t* d_perm, const int32_t* d_inv,
                                             const float* d_h, const float* d_w, int32_t k,
                                             float* d_out, uint32_t* d_cnt, int32_t group_m,
                                             daop_stream_t stream) {
  int rc = check_ffn_shape(rows, d, ffn, E);
  if (rc) return rc;
  if (k < 1 || k > 8 || g_gemm_mode != 0 || d % GB_N != 0) {
    set_error("fused combine: needs the CTA-pair kernel, k in 1..8 and d %% 256 == 0 "
              "(k=%d, mode=%d)", k, g_gemm_mode);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (rows == 0) return DAOP_OK;
  CUtensorMap ta, tb;
  const uint64_t adims[2] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(rows)};
  const uint64_t astr[1] = {static_cast<uint64_t>(ffn) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, act, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(d),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t bstr[2] = {static_cast<uint64_t>(ffn) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  const uint16_t* w2 = slab + static_cast<int64_t>(2) * ffn * d;
  if ((rc = make_tmap_bf16(&tb, w2, 3, bdims, bstr, bbox))) return rc;
  const int grp = group_m != 0 ? group_m : default_group_down(ffn);
  GemmParams p{d_offsets, d_slot_of, E, ffn / GB_K, d / GB_N, grp,
               GB_N, 128, y, d, GB_N, g_gemm_policy >= 0 ? g_gemm_policy : 2, 0,
               g_gemm_demote & 2, act, ffn, w2, ffn, slot_stride_elems};
  p.comb_perm = d_perm;
  p.comb_inv = d_inv;
  p.comb_h = d_h;
  p.comb_w = d_w;
  p.comb_out = d_out;
  p.comb_cnt = reinterpret_cast<unsigned*>(d_cnt);
  p.comb_k = k;
  return launch_gemm<false>(ta, tb, p, rows, as_stream(stream));
}

// Expert-parallel down GEMM (ep_p2p.cu): rows of the expert-major receive
// buffer (capacity rows_cap; the real extents come from the device offsets
// the receive kernel wrote into the workspace), outputs stored through the
// workspace's return table straight into the source ranks' y_back, then
// y[rank] flagged on every peer.
extern "C" int daop_ep_expert_gemm_down(const uint16_t* act, int64_t rows_cap, int32_t d,
                                        int32_t ffn, const uint16_t* slab, int64_t n_slots,
                                        int64_t slot_stride_elems, const int32_t* d_slot_of,
                                        int32_t E, const uint64_t* d_peers, void* d_ws,
                                        int32_t rank, int32_t G, uint32_t epoch, int32_t group_m,
                                        daop_stream_t stream) {
  int rc = check_ffn_shape(rows_cap, d, ffn, E);
  if (rc) return rc;
  if (G < 1 || G > EP_MAX_G || rank < 0 || rank >= G || rows_cap < 1) {
    set_error("ep gemm: bad rank/world (%d/%d) or capacity %lld", rank, G,
              static_cast<long long>(rows_cap));
    return DAOP_ERR_UNSUPPORTED;
  }
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  CUtensorMap ta, tb;
  const uint64_t adims[2] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(rows_cap)};
  const uint64_t astr[1] = {static_cast<uint64_t>(ffn) * 2};
  const uint32_t abox[2] = {GB_K, GB_M};
  if ((rc = make_tmap_bf16(&ta, act, 2, adims, astr, abox))) return rc;
  const uint64_t bdims[3] = {static_cast<uint64_t>(ffn), static_cast<uint64_t>(d),
                             static_cast<uint64_t>(n_slots)};
  const uint64_t bstr[2] = {static_cast<uint64_t>(ffn) * 2,
                            static_cast<uint64_t>(slot_stride_elems) * 2};
  const uint32_t bbox[3] = {GB_K, 128, 1};
  const uint16_t* w2 = slab + static_cast<int64_t>(2) * ffn * d;
  if ((rc = make_tmap_bf16(&tb, w2, 3, bdims, bstr, bbox))) return rc;
  GemmParams p{reinterpret_cast<const int64_t*>(ws + EP_LOCAL_OFF), d_slot_of, E, ffn / GB_K,
               d / GB_N, group_m != 0 ? group_m : default_group_down(ffn), GB_N, 128,
               nullptr, d, GB_N,
               g_gemm_policy >= 0 ? g_gemm_policy : 2, 0, g_gemm_demote & 2, act, ffn, w2, ffn,
               slot_stride_elems, reinterpret_cast<const uint64_t*>(ws + EP_ROWMAP),
               reinterpret_cast<unsigned*>(ws + EP_DONE_GEMM), d_peers, G, rank, epoch};
  return launch_gemm<false>(ta, tb, p, rows_cap, as_stream(stream));
}

extern "C" int daop_gemm_timeline(int32_t enable, uint64_t* h_out) {
  if (h_out) DAOP_CUDA(cudaMemcpyFromSymbol(h_out, g_pair_tl, sizeof(g_pair_tl)));
  if (enable) {
    static unsigned long long zeros[GT_CTAS][6];
    DAOP_CUDA(cudaMemcpyToSymbol(g_pair_tl, zeros, sizeof(zeros)));
  }
  DAOP_CUDA(cudaMemcpyToSymbol(g_pair_tl_on, &enable, sizeof(int)));
  return DAOP_OK;
}
