// DAOP decision primitives, shared by the host C++ entry points and the
// device decision code inside the decode kernel (one source, two targets, so
// the bits cannot drift).  Each routine restates the reference line by line:
//
//   topk_scan     <- moesim/_kernels.py:63-79   (k passes of a strict '>' scan:
//                                               highest first, ties -> lower id)
//   degrade       <- moesim/policies.py:264-296 (graceful degradation)
//   plan_layer    <- moesim/policies.py:248-261 (fiddler) and :299-336 (daop)
//
// Scores are compared, never combined arithmetically, so the template works
// bit-exactly for the reference's float64 and the router's exported float32
// (float32 -> float64 widening is exact and order preserving).
#pragma once
#include <stdint.h>

namespace daop {

template <class S>
__host__ __device__ inline void topk_scan(const S* s, int e, int k, int* out) {
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int c = 0; c < e; ++c) {
      bool taken = false;
      for (int q = 0; q < j; ++q) taken |= (out[q] == c);
      if (taken) continue;
      if (best < 0 || s[c] > s[best]) best = c;
    }
    out[j] = best;
  }
}

// policies.py:278-296.  sel[0..k) is edited in place; returns the number of
// degradations and records (dropped, substitute) pairs.
template <class S>
__host__ __device__ inline int degrade(const S* s, int e, int* sel, int k, const uint8_t* fast,
                                       int* drop_out, int* sub_out) {
  int nd = 0;
  while (true) {
    int n_slow = 0;
    for (int q = 0; q < k; ++q) n_slow += fast[sel[q]] ? 0 : 1;
    if (n_slow < 2) break;  // :281-283
    int sub = -1;           // max over alternatives by (score, -idx)  :284-289
    for (int c = 0; c < e; ++c) {
      if (!fast[c]) continue;
      bool in_sel = false;
      for (int q = 0; q < k; ++q) in_sel |= (sel[q] == c);
      if (in_sel) continue;
      if (sub < 0 || s[c] > s[sub]) sub = c;
    }
    if (sub < 0) break;
    int drop = -1, drop_pos = -1;  // min over slow picks by (score, idx)  :287
    for (int q = 0; q < k; ++q) {
      int c = sel[q];
      if (fast[c]) continue;
      if (drop < 0 || s[c] < s[drop] || (s[c] == s[drop] && c < drop)) {
        drop = c;
        drop_pos = q;
      }
    }
    sel[drop_pos] = sub;  // :290 selection[selection.index(drop)] = sub
    drop_out[nd] = drop;
    sub_out[nd] = sub;
    ++nd;
  }
  return nd;
}

// One layer of a decode token plan.  Returns the number of degradations, or
// -1 when the required prediction (carried on layer l-1) is missing.
// is_fast[q] = residence of sel[q]; for daop at l >= start a slow pick is
// (slow, stale, precalc) and a fast pick (fast, current) -- policies.py:325-330;
// below start (and for fiddler) every pick uses the current input.
template <class S>
__host__ __device__ inline int plan_layer(int l, const S* true_row, const S* pred_prev_row,
                                          bool pred_present, const uint8_t* fast_row, int e, int k,
                                          int start, bool daop_engine, bool graceful, int* sel,
                                          uint8_t* is_fast, int* drop, int* sub) {
  int nd = 0;
  if (!daop_engine || l < start) {
    topk_scan(true_row, e, k, sel);
  } else {
    if (!pred_present) return -1;
    topk_scan(pred_prev_row, e, k, sel);
    if (graceful) nd = degrade(pred_prev_row, e, sel, k, fast_row, drop, sub);
  }
  for (int q = 0; q < k; ++q) is_fast[q] = fast_row[sel[q]] ? 1 : 0;
  return nd;
}

}  // namespace daop
