/* daop_b200.h -- C ABI of the B200-native DAOP MoE-block hot path.
 *
 * One shared library (libdaop_b200.so, built from paper_2501_10375_b200/csrc)
 * exporting plain C entry points: raw pointers, sizes and a cudaStream_t
 * passed as an opaque handle.  No C++ or torch types cross this boundary.
 *
 * Conventions
 *   - every function returns 0 (DAOP_OK) or a negative DAOP_ERR_* code and
 *     then sets a thread-local message readable with daop_last_error();
 *     the Python layer maps codes onto the reference's MoesimError classes
 *     (moesim/errors.py:8-45).
 *   - "d_" pointers are device memory, "h_" pointers host memory; functions
 *     without a stream argument are host-only and synchronous.
 *   - device functions are asynchronous and stream ordered; callers own all
 *     buffers.  The library owns nothing except what *_create returns.
 *
 * Each entry point names the reference interface it replaces (file:line in
 * /root/reference/pkg/src/moesim).
 */
#ifndef DAOP_B200_H
#define DAOP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* daop_stream_t; /* cudaStream_t */

#define DAOP_OK 0
#define DAOP_ERR_SHAPE (-1)              /* ShapeMismatchError      errors.py:16 */
#define DAOP_ERR_NORMALIZATION (-2)      /* NormalizationError      errors.py:20 */
#define DAOP_ERR_BUDGET (-3)             /* BudgetError             errors.py:40 */
#define DAOP_ERR_PREDICTION_MISSING (-4) /* PredictionMissingError  errors.py:32 */
#define DAOP_ERR_CONFIG (-5)             /* ConfigError             errors.py:44 */
#define DAOP_ERR_EMPTY_PHASE (-6)        /* EmptyPhaseError         errors.py:24 */
#define DAOP_ERR_CUDA (-100)             /* CUDA runtime failure (no reference analogue) */
#define DAOP_ERR_UNSUPPORTED (-101)      /* shape outside the kernel envelope */

#define DAOP_ENGINE_ONDEMAND 0 /* policies.py:32 ENGINES index */
#define DAOP_ENGINE_PREFETCH 1
#define DAOP_ENGINE_FIDDLER 2
#define DAOP_ENGINE_DAOP 3

/* ------------------------------------------------------------------ library */
const char* daop_last_error(void);
int daop_version(void);
/* sm count and compute capability of the current device (fails without GPU) */
int daop_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* one synchronous step of a captured CUDA graph (cudaGraphExec_t): copy
 * `bytes` from h_src into the graph's pinned staging buffer, launch, wait.
 * The end-to-end decode call (no reference analogue: the reference prices a
 * decode step, simulator.py:289-391). */
int daop_graph_step(void* graph_exec, daop_stream_t stream, const void* h_src, void* h_staging,
                    int64_t bytes);
/* completion wait of daop_graph_step: 0 = cudaStreamSynchronize (default), 1 = busy-poll */
int daop_graph_step_mode(int32_t spin);

/* ---------------------------------------------- operator table (_kernels.py)
 * Device replacements of the reference's module-level operator table,
 * resolved at call time by metrics.py:59,70 and policies.py:180,302,318. */

/* replaces _kernels.topk_rows (_kernels.py:32-40,63-79,104-105):
 * (n, e) scores -> (n, k) int64 ids, highest first, ties to the lower index */
int daop_topk_rows_f64(const double* d_scores, int64_t n, int32_t e, int32_t k, int64_t* d_out,
                       daop_stream_t stream);
int daop_topk_rows_f32(const float* d_scores, int64_t n, int32_t e, int32_t k, int64_t* d_out,
                       daop_stream_t stream);
/* replaces _kernels.activation_counts (_kernels.py:52-58,94-102):
 * (t, l, k) int64 ids -> d_counts (l, e) int64 += counts (caller zeroes) */
int daop_activation_counts(const int64_t* d_topk, int64_t t, int32_t l, int32_t k, int32_t e,
                           int64_t* d_counts, daop_stream_t stream);
/* replaces _kernels.pair_overlap (_kernels.py:43-49,81-92) */
int daop_pair_overlap(const int64_t* d_a, const int64_t* d_b, int64_t n, int32_t ka, int32_t kb,
                      int64_t* d_out, daop_stream_t stream);

/* --------------------------------------- host decisions (placement/policies)
 * Pure host functions, bit-exact restatements of the reference. */

/* replaces placement.slot_budget_for_ecr (placement.py:123-125) */
int daop_slot_budget(double ecr, int32_t num_layers, int32_t num_experts, int64_t* h_budget);
/* replaces placement.init_from_calibration (placement.py:128-185):
 * h_calib (L, E) float64 -> h_on_fast (L, E) uint8 membership, h_budget */
int daop_placement_init(const double* h_calib, int32_t num_layers, int32_t num_experts, double ecr,
                        uint8_t* h_on_fast, int64_t* h_budget);
/* replaces placement.allocate_for_sequence (placement.py:188-237), threshold
 * given as the exact rational thr_num/thr_den = Fraction(str(float(s))).
 * h_events: capacity L*(E/2) rows of (layer, in, out, hot, cold). */
int daop_allocate(const uint8_t* h_on_fast, const int64_t* h_counts, int32_t num_layers,
                  int32_t num_experts, int64_t thr_num, int64_t thr_den, uint8_t* h_on_fast_out,
                  int64_t* h_events, int32_t* h_n_events);
/* replaces policies.degrade_selection (policies.py:264-296): h_sel_io (k) is
 * edited in place; h_drop/h_sub (capacity k) receive the degradation pairs */
int daop_degrade_f64(const double* h_scores, int32_t num_experts, int32_t* h_sel_io, int32_t k,
                     const uint8_t* h_fast, int32_t* h_drop, int32_t* h_sub, int32_t* h_n_deg);
/* replaces {Fiddler,Daop}Planner.plan_token (policies.py:248-261,299-336)
 * for one token: h_true (L,E), h_pred (L,E) with h_pred_mask (L), h_on_fast
 * (L,E).  Outputs h_sel (L,k), h_is_fast (L,k), h_drop/h_sub (L,k), h_n_deg (L). */
int daop_plan_token_f64(const double* h_true, const double* h_pred, const uint8_t* h_pred_mask,
                        const uint8_t* h_on_fast, int32_t num_layers, int32_t num_experts,
                        int32_t k, int32_t start_layer, int32_t engine, int32_t graceful,
                        int32_t* h_sel, uint8_t* h_is_fast, int32_t* h_drop, int32_t* h_sub,
                        int32_t* h_n_deg);

/* replaces one layer of {OnDemand,Prefetch}Planner.plan_token
 * (policies.py:103-245): per-layer LRU caches seeded from the placement.
 * The caller owns the cache state: h_last_use (L,E) int64 recency (-1 = not
 * cached; seed members with 0), h_capacity (L) = seeded set sizes, *h_step
 * the global step (ticked once per call).  Call for l = 0..L-1 per token.
 * h_true_row (E): layer l's true scores; h_pred_row (E) or NULL: the
 * prediction carried on layer l (prefetch engine, l+1 >= start).
 * Outputs: h_sel (k) = top-k (all executed on the fast tier); demand
 * migrations h_mig (k) sorted, with the expert each one evicted in
 * h_mig_evict (-1: a free slot); prefetches for layer l+1 h_pf / h_pf_evict.
 * DAOP_ERR_PREDICTION_MISSING after this layer's demand updates (as the
 * reference). */
int daop_lru_plan_layer(int32_t layer, int32_t num_layers, int32_t num_experts, int32_t k,
                        int32_t engine, int32_t start_layer, const double* h_true_row,
                        const double* h_pred_row, int64_t* h_last_use, const int32_t* h_capacity,
                        int64_t* h_step, int32_t* h_sel, int32_t* h_mig, int32_t* h_mig_evict,
                        int32_t* h_n_mig, int32_t* h_pf, int32_t* h_pf_evict, int32_t* h_n_pf);

/* ------------------------------------------------ device decision kernel
 * The same plan as daop_plan_token_f64, on the router's exported float32
 * probabilities, for n tokens at one layer, entirely on device (the decode
 * loop never syncs to the host for a decision).  d_pred_prev may be NULL
 * when the layer is below start (or engine is fiddler). */
int daop_plan_layer_f32(const float* d_true, const float* d_pred_prev, const uint8_t* d_fast_row,
                        int64_t n, int32_t layer, int32_t num_experts, int32_t k,
                        int32_t start_layer, int32_t engine, int32_t graceful, int32_t* d_sel,
                        uint8_t* d_is_fast, int32_t* d_drop, int32_t* d_sub, int32_t* d_n_deg,
                        daop_stream_t stream);

/* ------------------------------------------------ random-init tensors
 * Counter-based generator shared bit-for-bit with oracle/rng.py. */
int daop_fill_uniform_bf16(uint16_t* d_dst, int64_t n, uint64_t seed, uint64_t tag, float scale,
                           int64_t index_offset, daop_stream_t stream);
int daop_fill_uniform_f32(float* d_dst, int64_t n, uint64_t seed, uint64_t tag, float scale,
                          int64_t index_offset, daop_stream_t stream);
/* RMSNorm weight bf16(1 + 0.25 u) of one layer */
int daop_fill_norm_bf16(uint16_t* d_dst, int64_t d, uint64_t seed, int32_t layer,
                        daop_stream_t stream);
/* host-side fill (for the pinned slow-tier pool), multi-threaded */
int daop_fill_uniform_bf16_host(uint16_t* h_dst, int64_t n, uint64_t seed, uint64_t tag,
                                float scale, int64_t index_offset, int32_t threads);

/* ------------------------------------------------ fused router (prefill)
 * Realises SURVEY a1+a2+a3+a9 in one pass per token: x = bf16(rmsnorm(h) *
 * gamma) (written to d_x when non-NULL), p = softmax(x.Wg^T), p_pred =
 * softmax(x.Wg_next^T) (when d_wg_next != NULL), top-k of p with ties to the
 * lower id (_kernels.py:63-79), renormalised weights, and the per-sequence
 * activation counter d_hist[(t / tokens_per_seq) * hist_seq_stride + e] += 1
 * (metrics.expert_counts, metrics.py:64-71) when d_hist != NULL. */
/* tuning: bit 0 = 1 (default) single-pass tensor-core router where d = 256 *
 * {4, 8, 12, 16} (h slice held in registers), 0 = the two-pass variant (the
 * two are bit-identical, tests); bits 4..7 = 1 + the single-pass kernel's L2
 * prefetch distance in grid-strides (0 = keep). */
int daop_set_router_mode(int32_t mode);
/* tuning: gather / combine kernel variants (0 = default bulk-DMA kernels for
 * large T, 1 = warp-per-token register kernels), bulk gather CTAs per SM and
 * combine ring stages (<= 0 keeps the current value). */
int daop_set_stream_mode(int32_t gather, int32_t combine, int32_t gather_ctas_per_sm,
                         int32_t combine_stages);
int daop_router(const float* d_h, const uint16_t* d_gamma, const uint16_t* d_wg,
                const uint16_t* d_wg_next, int64_t t, int32_t d, int32_t num_experts, int32_t k,
                float eps, uint16_t* d_x, float* d_p_true, float* d_p_pred, int32_t* d_topk_idx,
                float* d_topk_w, int32_t* d_hist, int64_t tokens_per_seq,
                int64_t hist_seq_stride, daop_stream_t stream);

/* ------------------------------------------------ permutation + combine
 * Stable token->expert permutation (histogram + exclusive scan): rows (t, j)
 * sorted by (expert, t, j); d_offsets (E+1) int64, d_perm[p] = t*k + j,
 * d_inv[t*k + j] = p, d_x_perm[p] = d_x[t] (skipped when NULL).  No reference
 * analogue; builder-defined contract in DESIGN.md. */
int daop_permute_workspace(int64_t t, int32_t k, int32_t num_experts, int64_t* h_bytes);
int daop_permute(const int32_t* d_topk_idx, int64_t t, int32_t k, int32_t num_experts,
                 const uint16_t* d_x, int32_t d, int64_t* d_offsets, int32_t* d_perm,
                 int32_t* d_inv, uint16_t* d_x_perm, void* d_workspace, int64_t ws_bytes,
                 daop_stream_t stream);
/* d_out[t] = d_h[t] + sum_{j<k} d_w[t,j] * d_y[d_inv[t,j]]   (fixed j order) */
int daop_combine(const float* d_h, const float* d_y_sorted, const int32_t* d_inv,
                 const float* d_w, int64_t t, int32_t k, int32_t d, float* d_out,
                 daop_stream_t stream);

/* decode-side combine when some picks ran on the slow (host) tier:
 * d_out[i] = d_h[i] + sum_{q<k} d_w[q] * d_y[q*d + i]   (fixed q order) */
int daop_combine_dense(const float* d_h, const float* d_y, const float* d_w, int32_t k,
                       int32_t d, float* d_out, daop_stream_t stream);

/* ------------------------------------------------ DAOP slow tier (host CPU)
 * SwiGLU expert on the host for experts resident in pinned host memory
 * (moesim "slow device"): h_x (n, d) bf16 -> h_y (n, d) fp32
 * with act = bf16(silu(x.W1^T) * (x.W3^T)), y = act.W2^T, fp32 accumulation
 * (AVX-512 BF16 when available).  h_act_scratch (n*ffn bf16) may be NULL. */
int daop_host_expert_ffn(const uint16_t* h_x, int64_t n, const uint16_t* h_w1,
                         const uint16_t* h_w3, const uint16_t* h_w2, int32_t d, int32_t ffn,
                         float* h_y, uint16_t* h_act_scratch, int32_t threads);
/* The slow expert restricted to ffn rows [r0, r1) (decode-sized n < 16):
 * y (n, d) fp32 = W2[:, r0:r1] . bf16(silu(x W1[r0:r1]^T) * (x W3[r0:r1]^T)).
 * The host's share of a slow expert split with the GPU (DaopEngine: the GPU
 * computes rows [0, r0) from a copy pulled from the pinned pool over PCIe;
 * both read the host's DRAM).  Replaces part of the CPU expert execution the
 * reference prices as t_slow (simulator.py:196-234). */
int daop_host_expert_ffn_rows(const uint16_t* x, int64_t n, const uint16_t* w1, const uint16_t* w3,
                              const uint16_t* w2, int32_t d, int32_t ffn, int32_t r0, int32_t r1,
                              float* y, int32_t threads);
/* The GPU's share of that split: rows [0, rows) of W1 / W3 and columns [0, rows)
 * of W2 from the expert's pinned host copy (h_w1/h_w3/h_w2, ffn columns / rows)
 * into d_stage laid out as an expert with ffn = rows: [W1 | W3 | W2 (d x rows)]
 * (three async copies on `stream`, W2 as one 2-D copy). */
int daop_slow_split_pull(const uint16_t* h_w1, const uint16_t* h_w3, const uint16_t* h_w2,
                         int32_t d, int32_t ffn, int32_t rows, uint16_t* d_stage,
                         daop_stream_t stream);
/* Pinned host memory for the expert pool (the slow tier and the migration
 * source): mmap + transparent huge pages, parallel first touch on `threads`
 * cores (<= 0: all), cudaHostRegister (*h_registered = 1; 0 when the host has
 * no CUDA device, e.g. a build machine).  Free with daop_host_pool_free. */
int daop_host_pool_alloc(int64_t bytes, int32_t threads, void** h_out, int32_t* h_registered);
int daop_host_pool_free(void* h_ptr, int64_t bytes, int32_t registered);
int daop_host_caps(int32_t* avx512_bf16, int32_t* hw_threads);

/* Host-tier scheduling: rows per work chunk of the up / down GEMV phases
 * (0 = one contiguous share per worker).  Tuning knob; no reference
 * counterpart (the reference only prices t_expert_slow, simulator.py:49). */
int daop_host_set_grain(int64_t up_rows, int64_t down_rows);
/* profiling aid: stream-read `bytes` of host memory on the slow tier's thread
 * pool (the bandwidth ceiling of its GEMV); *checksum defeats elision */
int daop_host_stream_read(const void* h_buf, int64_t bytes, int32_t threads, double* checksum);

/* ------------------------------------------------ grouped expert GEMMs (prefill)
 * tcgen05/TMEM/TMA grouped GEMMs over expert-sorted rows.  Expert e owns rows
 * [d_offsets[e], d_offsets[e+1]) and its weights live in slab slot
 * d_slot_of[e]; a slot is [W1 (ffn,d) | W3 (ffn,d) | W2 (d,ffn)] bf16.
 *   up:   d_act (rows, ffn) bf16 = silu(x W1^T) * (x W3^T)
 *   down: d_y   (rows, d)   f32  = act W2^T
 * group_m <= 0 picks the default rasterisation group. */
/* tuning switch: 0 = tcgen05.mma.cta_group::2 CTA-pair kernel (default),
 * 1 = single-CTA kernel */
int daop_set_gemm_mode(int32_t mode);
/* device-wide GEMM setup (persisting-L2 limit); call before capturing GEMMs
 * into a CUDA graph (the launch path does it lazily otherwise). */
int daop_gemm_prepare(void);
int daop_expert_gemm_up(const uint16_t* d_x_perm, int64_t rows, int32_t d, int32_t ffn,
                        const uint16_t* d_slab, int64_t n_slots, int64_t slot_stride_elems,
                        const int64_t* d_offsets, const int32_t* d_slot_of, int32_t num_experts,
                        uint16_t* d_act, int32_t group_m, daop_stream_t stream);
/* the same two GEMMs for SMALL token counts (batched decode): weights are the
 * M side (128-row tiles), the expert's tokens the N side (nt = 32, 64 or 128 per
 * block), so each expert's weights stream once per block of nt tokens. */
int daop_expert_gemm_up_skinny(const uint16_t* d_x_perm, int64_t rows, int32_t d, int32_t ffn,
                               const uint16_t* d_slab, int64_t n_slots, int64_t slot_stride_elems,
                               const int64_t* d_offsets, const int32_t* d_slot_of,
                               int32_t num_experts, uint16_t* d_act, int32_t nt,
                               daop_stream_t stream);
int daop_expert_gemm_down_skinny(const uint16_t* d_act, int64_t rows, int32_t d, int32_t ffn,
                                 const uint16_t* d_slab, int64_t n_slots,
                                 int64_t slot_stride_elems, const int64_t* d_offsets,
                                 const int32_t* d_slot_of, int32_t num_experts, float* d_y,
                                 int32_t nt, daop_stream_t stream);
/* up GEMM with its A rows gathered by TMA straight from the token matrix
 * d_x (src_rows, d): sorted row r reads token d_perm[r] / k (no x_perm). */
int daop_expert_gemm_up_gather(const uint16_t* d_x, int64_t src_rows, const int32_t* d_perm,
                               int32_t k, int64_t rows, int32_t d, int32_t ffn,
                               const uint16_t* d_slab, int64_t n_slots, int64_t slot_stride_elems,
                               const int64_t* d_offsets, const int32_t* d_slot_of,
                               int32_t num_experts, uint16_t* d_act, int32_t group_m,
                               daop_stream_t stream);
int daop_expert_gemm_down(const uint16_t* d_act, int64_t rows, int32_t d, int32_t ffn,
                          const uint16_t* d_slab, int64_t n_slots, int64_t slot_stride_elems,
                          const int64_t* d_offsets, const int32_t* d_slot_of,
                          int32_t num_experts, float* d_y, int32_t group_m,
                          daop_stream_t stream);
/* down GEMM with the combine fused into its epilogue: each token's last pick
 * to land (per 256-column tile) writes d_out = d_h + sum_j w_j y_j in fixed j
 * order (daop_combine's arithmetic); d_perm / d_inv from daop_permute,
 * d_cnt (T, d / 256) u32 zeroed once and self-resetting.  Needs the CTA-pair
 * kernel (gemm mode 0). */
int daop_expert_gemm_down_combine(const uint16_t* d_act, int64_t rows, int32_t d, int32_t ffn,
                                  const uint16_t* d_slab, int64_t n_slots,
                                  int64_t slot_stride_elems, const int64_t* d_offsets,
                                  const int32_t* d_slot_of, int32_t num_experts, float* d_y,
                                  const int32_t* d_perm, const int32_t* d_inv, const float* d_h,
                                  const float* d_w, int32_t k, float* d_out, uint32_t* d_cnt,
                                  int32_t group_m, daop_stream_t stream);

/* ------------------------------------------------ expert parallelism over peer memory
 * Replaces the NCCL all-to-all dispatch / combine that SURVEY.md §8b
 * proposes as "daop_ep_dispatch / daop_ep_combine" -- the reference has no
 * devices; its only exchange is the priced expert-activation
 * transfer, moesim/simulator.py:196-234.  One symmetric workspace per rank
 * (daop_ep_ws_layout bytes, zeroed, shared with the peers by CUDA IPC);
 * d_peers[G] = the G workspace bases as seen from this GPU.  Per layer, on
 * one stream, no host sync: publish -> dispatch -> recv -> up GEMM ->
 * daop_ep_expert_gemm_down -> wait_back -> daop_combine.  `epoch` increases
 * by one per layer call and is identical on every rank. */
int daop_ep_ws_layout(int32_t world, int32_t num_experts, int32_t d, int64_t cap_recv_rows,
                      int64_t cap_send_rows, int64_t* h_total_bytes, int64_t* h_recv_off,
                      int64_t* h_yback_off, int64_t* h_local_offsets_off);
/* per-expert row counts of this rank's permutation -> every peer */
int daop_ep_publish(const uint64_t* d_peers, int32_t rank, int32_t world, int32_t num_experts,
                    const int64_t* d_offsets, uint32_t epoch, daop_stream_t stream);
/* permutation gather fused with the all-to-all: x rows (token order) are
 * stored straight into the owners' expert-major receive buffers */
int daop_ep_dispatch(const uint64_t* d_peers, int32_t rank, int32_t world, int32_t num_experts,
                     int32_t k, int32_t d, const uint16_t* d_x, const int32_t* d_perm,
                     int64_t rows_cap, int64_t recv_off, uint32_t epoch, daop_stream_t stream);
/* waits for every source's rows; writes the local expert offsets and the
 * per-row return addresses into the workspace */
int daop_ep_recv(const uint64_t* d_peers, int32_t rank, int32_t world, int32_t num_experts,
                 int32_t d, int64_t yback_off, uint32_t epoch, daop_stream_t stream);
/* down GEMM fused with the return all-to-all (outputs stored into the
 * source ranks' y_back, tile by tile) */
int daop_ep_expert_gemm_down(const uint16_t* d_act, int64_t rows_cap, int32_t d, int32_t ffn,
                             const uint16_t* d_slab, int64_t n_slots, int64_t slot_stride_elems,
                             const int32_t* d_slot_of, int32_t num_experts,
                             const uint64_t* d_peers, void* d_ws, int32_t rank, int32_t world,
                             uint32_t epoch, int32_t group_m, daop_stream_t stream);
/* the skinny (batched-decode) form of the fused-return down GEMM */
int daop_ep_expert_gemm_down_skinny(const uint16_t* d_act, int64_t rows_cap, int32_t d,
                                    int32_t ffn, const uint16_t* d_slab, int64_t n_slots,
                                    int64_t slot_stride_elems, const int32_t* d_slot_of,
                                    int32_t num_experts, const uint64_t* d_peers, void* d_ws,
                                    int32_t rank, int32_t world, uint32_t epoch, int32_t nt,
                                    daop_stream_t stream);
int daop_ep_wait_back(void* d_ws, int32_t world, uint32_t epoch, daop_stream_t stream);
/* decode b = 1 over G GPUs: the residual is replicated, every rank runs
 * daop_decode_layer (mode 0) with its own experts as the resident set, then
 * daop_ep_decode_share stores its picks' outputs (d_y rows where d_is_fast)
 * into every peer's decode workspace (daop_ep_decode_ws_bytes, zeroed) slot
 * [epoch & 1]; after daop_ep_decode_wait, daop_combine_dense on that slot
 * gives every rank the same next residual. */
int daop_ep_decode_ws_bytes(int32_t k, int32_t d, int64_t* h_bytes);
int daop_ep_decode_share(const uint64_t* d_peers, int32_t rank, int32_t world, int32_t k,
                         int32_t d, const float* d_y, const uint8_t* d_is_fast, uint32_t epoch,
                         daop_stream_t stream);
int daop_ep_decode_wait(void* d_ws, int32_t world, uint32_t epoch, daop_stream_t stream);
/* the fused form: daop_decode_layer (mode 0) whose phase-2 reduction also
 * stores the local picks' outputs into every peer's slot and whose last CTA
 * flags them; then daop_ep_decode_finish = wait + fixed-order combine */
int daop_ep_decode_layer(const uint64_t* d_peers, int32_t rank, int32_t world, uint32_t epoch,
                         const float* d_h, const uint16_t* d_gamma, const uint16_t* d_wg,
                         const uint16_t* d_wg_next, const uint8_t* d_fast_row,
                         const int32_t* d_slot_of, const uint16_t* d_slab,
                         int64_t slot_stride_elems, int32_t d, int32_t ffn, int32_t num_experts,
                         int32_t k, float eps, uint16_t* d_x_out, float* d_p_true,
                         float* d_p_pred, int32_t* d_sel, float* d_w, uint8_t* d_is_fast,
                         int32_t* d_deg, float* d_y, float* d_h_out, void* d_workspace,
                         daop_stream_t stream);
int daop_ep_decode_finish(void* d_ws, int32_t world, int32_t k, int32_t d, const float* d_h,
                          const float* d_w, float* d_out, uint32_t epoch, daop_stream_t stream);
/* 1 if any wait of this workspace timed out (synchronous read) */
int daop_ep_status(const void* d_ws, int32_t* h_err);
/* CUDA IPC of a workspace: 64-byte handle + offset inside its allocation */
int daop_ep_ipc_handle(const void* d_ptr, void* h_handle64, int64_t* h_offset);
int daop_ep_ipc_open(const void* h_handle64, int64_t offset, void** h_base, void** h_ptr);
int daop_ep_ipc_close(void* h_base);

/* ------------------------------------------------ decode layer (b = 1)
 * One persistent cooperative launch: RMSNorm + gate + next-layer gate, the
 * selection (mode 0: true top-k -- Fiddler / l < start; mode 1: DAOP plan
 * from d_pred_prev with graceful degradation, policies.py:299-336), then the
 * HBM-streaming SwiGLU GEMV of every HBM-resident pick and the combine
 * d_h_out = d_h + sum_q w_q y_q (written only when every pick is resident;
 * otherwise d_y holds the resident picks' outputs for an external combine
 * with the slow tier).  d_deg: drop[k] | sub[k] | count.
 * d_workspace: daop_decode_workspace() bytes, zeroed once, self-resetting. */
/* profiling aid: enable (1) / read back the per-CTA phase timeline of the
 * last decode_layer launches (SM clock64 cycles: [0] start, [1] phase 0 done,
 * [2] phase 1 done, [3] act ready, [4] end, [5] rms, [6] x+gates, [8]
 * selection+first issue); enabling also clears it. */
int daop_decode_timeline(int32_t enable, uint64_t* h_out, int32_t n_cta);
int daop_decode_workspace(int32_t d, int32_t ffn, int32_t num_experts, int32_t k,
                          int64_t* h_bytes);
int daop_decode_layer(const float* d_h, const uint16_t* d_gamma, const uint16_t* d_wg,
                      const uint16_t* d_wg_next, const float* d_pred_prev,
                      const uint8_t* d_fast_row, const int32_t* d_slot_of,
                      const uint16_t* d_slab, int64_t slot_stride_elems, int32_t d, int32_t ffn,
                      int32_t num_experts, int32_t k, int32_t mode, int32_t graceful,
                      int32_t weights_from_pred, float eps, uint16_t* d_x_out, float* d_p_true,
                      float* d_p_pred, int32_t* d_sel, float* d_w, uint8_t* d_is_fast,
                      int32_t* d_deg, float* d_y, float* d_h_out, void* d_workspace,
                      int32_t variant, daop_stream_t stream);
/* variant: ring geometry (warps x stages x stage bytes); 0 = default
 * (16 x 1 x 10 KB), 1..9 = tuning alternatives.  num_experts <= 16. */

/* ------------------------------------------------ non-MoE block: attention (decode, b = 1)
 * The caller of the MoE block (priced by
 * the reference as t_nonmoe, simulator.py:291): RMSNorm -> QKV GEMV -> RoPE
 * (theta) -> append to the layer's KV cache (n_kv, max_seq, 128) bf16 at
 * `pos` -> GQA flash-decoding over positions 0..pos -> O-proj GEMV ->
 * d_h_out = d_h + o Wo^T.  head_dim 128; Wqkv (q + 2 kv, d), Wo (d, q) bf16.
 * d_workspace: daop_attn_workspace() bytes. */
int daop_attn_workspace(int32_t n_heads, int32_t n_kv, int32_t max_seq, int64_t* h_bytes);
int daop_attn_decode(const float* d_h, const uint16_t* d_gamma, const uint16_t* d_wqkv,
                     const uint16_t* d_wo, uint16_t* d_k_cache, uint16_t* d_v_cache, int32_t d,
                     int32_t n_heads, int32_t n_kv, int32_t max_seq, int32_t pos, float eps,
                     float theta, uint16_t* d_xa_out, float* d_h_out, void* d_workspace,
                     daop_stream_t stream);

/* L2 prefetch of up to two byte ranges on `stream` (fire and forget): the
 * decode loop issues the next layer's Wqkv / Wo before this layer's MoE
 * decode kernel, whose expert stream is L2::evict_first. */
int daop_l2_prefetch(const void* d_p0, int64_t n0, const void* d_p1, int64_t n1,
                     daop_stream_t stream);

/* Prefill of T prompt tokens through the same attention block, positions
 * pos0 .. pos0 + T - 1 (the calls DaopEngine.prefill makes per layer; the
 * reference prices this as the prefill t_nonmoe, simulator.py:438-441):
 *   daop_attn_norm_rows: d_xa (T, d) bf16 = rmsnorm(d_h (T, d) fp32) * gamma
 *   daop_gemm_bf16_f32:  qkv = xa . Wqkv^T  (T, q + 2 kv) fp32   (tcgen05)
 *   daop_attn_prefill:   k (RoPE), v of every token -> the cache, then causal
 *                        flash attention on the tensor cores -> d_o (T, q) bf16
 *   daop_gemm_bf16_f32:  h' = h + o . Wo^T  (residual in the epilogue) */
/* Dense projection on the grouped-GEMM tcgen05 pipeline: d_out (M, N) fp32 =
 * d_a (M, K) bf16 . d_w^T (d_w (N, K) bf16 row-major) [+ d_resid (M, N) fp32,
 * may alias d_out, NULL for none].  K % 64 == 0, N % 256 == 0. */
int daop_gemm_bf16_f32(const uint16_t* d_a, int64_t M, int32_t K, const uint16_t* d_w, int32_t N,
                       const float* d_resid, float* d_out, daop_stream_t stream);
/* Same product with a caller-owned fp32 workspace d_ws (ws_bytes): prompt-sized
 * M (<= 256 rows, whose N / 256 CTA-pair tiles leave most SMs idle) splits K
 * over the idle SM pairs into ksplit fp32 partials in d_ws (ksplit x M x N x 4
 * bytes, ksplit <= 8) and sums them in fixed order [+ d_resid] into d_out.
 * Without room in d_ws, or for larger M, it is daop_gemm_bf16_f32. */
int daop_gemm_bf16_f32_ws(const uint16_t* d_a, int64_t M, int32_t K, const uint16_t* d_w,
                          int32_t N, const float* d_resid, float* d_out, float* d_ws,
                          int64_t ws_bytes, daop_stream_t stream);
int daop_attn_norm_rows(const float* d_h, int64_t T, const uint16_t* d_gamma, int32_t d, float eps,
                        uint16_t* d_xa, daop_stream_t stream);
int daop_attn_prefill(const float* d_qkv, int64_t T, int32_t pos0, uint16_t* d_k_cache,
                      uint16_t* d_v_cache, int32_t n_heads, int32_t n_kv, int32_t max_seq,
                      float theta, uint16_t* d_o, daop_stream_t stream);

/* ------------------------------------------------ persistent decode server (b = 1)
 * The end-to-end decode call without a launch or a stream synchronisation
 * per call: daop_server_start launches ONE persistent cooperative kernel for
 * a layer (mode 0; arguments as daop_decode_layer, d_h_out / d_sel normally
 * pinned host memory); each daop_server_step copies h into pinned memory,
 * rings a doorbell the kernel polls, and spins until the kernel has written
 * the residual and the selection to the host.  The kernel holds every SM
 * until daop_server_stop, or exits by itself after idle_ms without a call.
 * (The reference's decode step is priced, not executed: simulator.py:289-391.) */
int daop_server_start(const uint16_t* d_gamma, const uint16_t* d_wg, const uint16_t* d_wg_next,
                      const uint8_t* d_fast_row, const int32_t* d_slot_of,
                      const uint16_t* d_slab, int64_t slot_stride_elems, int32_t d, int32_t ffn,
                      int32_t num_experts, int32_t k, float eps, uint16_t* d_x_out,
                      float* d_p_true, float* d_p_pred, int32_t* sel, float* d_w,
                      uint8_t* d_is_fast, int32_t* d_deg, float* d_y, float* h_out,
                      void* d_workspace, double idle_ms, daop_stream_t stream, void** handle);
int daop_server_step(void* handle, const float* h_in, double timeout_ms);
int daop_server_stop(void* handle);
/* profiling aid: per-call GPU timestamps of servers started afterwards
 * (d_buf [cap][4] u64 zeroed: doorbell seen, input released, body done) */
int daop_server_trace(uint64_t* d_buf, int32_t cap);
/* decode attention: attention core + O projection as two launches (0, the
 * default) or ONE cooperative launch whose Wo stream overlaps the attention
 * core (1; 2: the stream waits for the split tasks' K / V) -- measured slower */
int daop_set_attn_fused(int32_t fused);
/* profiling aid: per-CTA global-timer stamps of the decode attention kernels'
 * last launches (h_out: [qkv, core, oproj][256 CTAs][start, end] ns); enable
 * zeroes them */
int daop_attn_timeline(int32_t enable, uint64_t* h_out);
/* profiling aid: per-CTA global-timer stamps of the CTA-pair GEMM kernel's
 * launches since enabling (h_out: [512 CTAs][entry, setup done, last MMA
 * commit, last epilogue warp done, last accumulator ready in an epilogue
 * warp, fp32 epilogue: first TMEM chunk loaded] ns, max over launches);
 * enable zeroes them */
int daop_gemm_timeline(int32_t enable, uint64_t* h_out);

/* ------------------------------------------------ die topology (B200: two dies)
 * SM -> die map of the current device, measured once and cached (csrc/
 * topology.cu: one CTA per SM times loads of sampled L2 lines; lines homed on
 * the SM's own die answer faster).  die_of_sm[smid] for smid < n_sm; *n_die =
 * 2 when the SMs split into two clean halves, else 1 (all zeros).  Used by the
 * prefill GEMMs' per-die tile schedule (no reference counterpart). */
int daop_die_map(int32_t* die_of_sm, int32_t n_sm, int32_t* n_die);
/* Per-die tile schedule of the CTA-pair prefill GEMMs (each die strides over
 * its own share of every expert's m-tiles): n == 0 off, n < 0 the measured map
 * (daop_die_map), n > 0 an explicit table (die of SM i = tab[i] != 0). */
int daop_set_gemm_die_table(const int32_t* tab, int32_t n);
/* profiling aid (under ncu, lts__t_sectors_srcunit_ltcfabric): SM `ref` reads
 * the buffer, then SM `test` reads it (test == ref: one SM reads twice) */
int daop_die_pair_probe(const void* d_buf, int64_t bytes, int32_t ref, int32_t test,
                        uint32_t* d_flag, daop_stream_t stream);
/* profiling aid: the raw measurement (lat: grid x nlines clocks, smid: grid) */
int daop_die_probe(const uint32_t* d_buf, int32_t nlines, int32_t stride_words, int32_t grid,
                   uint32_t* d_lat, int32_t* d_smid, daop_stream_t stream);

/* ------------------------------------------------ trace files (moesim JSONL)
 * Formats one phase's token records of a RoutingTrace exactly as
 * moesim/trace.py:328-362 save_trace does ("%.17g" scores, "null" where the
 * mask is 0, one '\n'-terminated line per token).  true/pred (T, L, E) f64,
 * mask (T, L) u8, phase 0 = prefill / 1 = decode.  out == NULL: size query
 * into *written. */
int daop_trace_format_phase(const double* h_true, const double* h_pred, const uint8_t* h_mask,
                            int64_t T, int32_t L, int32_t E, int32_t phase, char* h_out,
                            int64_t cap, int64_t* written);

#ifdef __cplusplus
}
#endif
#endif /* DAOP_B200_H */
