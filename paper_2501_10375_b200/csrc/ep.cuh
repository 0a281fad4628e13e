// Symmetric expert-parallel workspace layout (ep_p2p.cu, grouped_gemm.cu).
// One workspace per rank, identical layout on every GPU; byte offsets:
#pragma once
#include <cstdint>

namespace daop {

constexpr int EP_MAX_G = 8;
constexpr int EP_MAX_E = 64;
constexpr int64_t EP_FLAGS_COUNTS = 0;     // u32 [EP_MAX_G]
constexpr int64_t EP_FLAGS_X = 64;         // u32 [EP_MAX_G]
constexpr int64_t EP_FLAGS_Y = 128;        // u32 [EP_MAX_G]
constexpr int64_t EP_ERR = 192;            // u32
constexpr int64_t EP_DONE_DISPATCH = 196;  // u32
constexpr int64_t EP_DONE_GEMM = 200;      // u32
constexpr int64_t EP_DONE_SHARE = 204;     // u32 (decode workspace)
constexpr int64_t EP_FLAGS_D = 256;        // u32 [EP_MAX_G] (decode workspace)
constexpr int64_t EP_DEC_Y = 1024;         // f32 [2][k][d] gathered pick outputs (decode workspace)
constexpr int64_t EP_COUNTS = 1024;        // i64 [2][EP_MAX_G][EP_MAX_E]
constexpr int64_t EP_LOCAL_OFF = EP_COUNTS + 2 * EP_MAX_G * EP_MAX_E * 8;  // i64 [EP_MAX_E+1]
constexpr int64_t EP_ROWMAP = 16384;       // u64 [cap_recv]
constexpr unsigned long long EP_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;

// system-scope flag accesses (the flags are written by peer GPUs over NVLink)
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


}  // namespace daop
