// Shared device helpers for the B200 event-camera kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace evs {

constexpr int kWarp = 32;
constexpr int kChunk = 32;  // reference CHUNK_WIDTH (parallel.py:32)

// Decoupled-lookback status word: [flag:2 | epoch:22 | value:40].
// flag 0 = not ready, 1 = aggregate only, 2 = inclusive prefix.
// Epoch tags make stale words from earlier launches read as "not ready",
// so the status arrays never need clearing between launches.
constexpr uint64_t kFlagAgg = 1, kFlagInc = 2;
constexpr int kEpochBits = 22;
constexpr uint32_t kEpochMask = (1u << kEpochBits) - 1;
constexpr uint64_t kValueMask = (1ull << 40) - 1;

__device__ __forceinline__ uint64_t pack_status(uint64_t flag, uint32_t epoch, uint64_t v) {
  return (flag << 62) | ((uint64_t)(epoch & kEpochMask) << 40) | (v & kValueMask);
}
// returns flag (0 if epoch mismatch) and value
__device__ __forceinline__ uint32_t status_flag(uint64_t w, uint32_t epoch) {
  if ((uint32_t)((w >> 40) & kEpochMask) != (epoch & kEpochMask)) return 0;
  return (uint32_t)(w >> 62);
}
__device__ __forceinline__ uint64_t status_value(uint64_t w) { return w & kValueMask; }

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_relaxed_i64(const int64_t* p) {
  return (int64_t)ld_relaxed(reinterpret_cast<const uint64_t*>(p));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one value per thread (NT threads).
// smem must hold NT/32 + 1 elements.  Returns exclusive prefix; *total = sum.
template <int NT, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NW ? smem[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < NW) smem[lane] = wi - w;
    if (lane == NW - 1) smem[NW] = wi;
  }
  __syncthreads();
  T r = smem[warp] + inc - v;
  *total = smem[NW];
  __syncthreads();
  return r;
}

// Block-wide exclusive scan with a single barrier: every thread sums the warp
// totals itself.  `buf` (NT/32 elements) must not be rewritten before every
// thread has returned (callers alternate buffers or have a barrier between).
template <int NT, typename T>
__device__ __forceinline__ T block_excl_scan_1s(T v, T* buf, T* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) buf[warp] = inc;
  __syncthreads();
  T pre = T(0), tot = T(0);
  if constexpr (NW == 8 && sizeof(T) == 4) {  // the 8 warp totals in two 16-byte loads (buf 16-byte aligned)
    const uint4 q0 = reinterpret_cast<const uint4*>(buf)[0], q1 = reinterpret_cast<const uint4*>(buf)[1];
    const T x[8] = {(T)q0.x, (T)q0.y, (T)q0.z, (T)q0.w, (T)q1.x, (T)q1.y, (T)q1.z, (T)q1.w};
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      pre += w < warp ? x[w] : T(0);
      tot += x[w];
    }
  } else {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const T x = buf[w];
      pre += w < warp ? x : T(0);
      tot += x;
    }
  }
  *total = tot;
  return pre + inc - v;
}

// Warp-cooperative decoupled lookback (called by a full warp).  `status`
// points at the tile-status array of one chain; tile `t` has already
// published its aggregate.  Returns the exclusive prefix for tile t.
//
// Wide windows: each round reads kLookWin*32 predecessors at once (lane l,
// slot m -> tile base - l - 32m), so a whole wave of tiles that publish their
// aggregates together resolves in one or two L2 round trips instead of
// walking back 32 tiles per round trip.
constexpr int kLookWin = 8;
__device__ __forceinline__ uint64_t warp_lookback(const uint64_t* status, int64_t t, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = t - 1;
  while (base >= 0) {
    uint32_t flag[kLookWin];
    uint64_t val[kLookWin];
    for (;;) {
      uint64_t w[kLookWin];
#pragma unroll
      for (int m = 0; m < kLookWin; ++m) {
        const int64_t idx = base - lane - 32 * m;
        w[m] = idx >= 0 ? ld_relaxed(status + idx) : 0ull;
      }
      // first (nearest) window slot that holds an inclusive prefix
      int first_m = kLookWin;
      uint32_t first_mask = 0;
      bool stall = false;
#pragma unroll
      for (int m = 0; m < kLookWin; ++m) {
        const int64_t idx = base - lane - 32 * m;
        if (idx >= 0) {
          flag[m] = status_flag(w[m], epoch);
          val[m] = status_value(w[m]);
        } else {
          flag[m] = (uint32_t)kFlagInc;  // virtual inclusive zero before tile 0
          val[m] = 0;
        }
        const uint32_t inc_mask = __ballot_sync(0xffffffffu, flag[m] == kFlagInc);
        const uint32_t nr_mask = __ballot_sync(0xffffffffu, flag[m] == 0);
        if (first_m == kLookWin) {
          // lanes 0..first-inclusive of this slot (all lanes if none inclusive)
          const uint32_t upto = inc_mask ? ((2u << (__ffs(inc_mask) - 1)) - 1u) : 0xffffffffu;
          if (nr_mask & upto) stall = true;
          if (inc_mask) { first_m = m; first_mask = upto; }
        }
      }
      if (stall) {  // a needed predecessor is not ready: back off, re-read the window
        __nanosleep(200);
        continue;
      }
      uint64_t mine = 0;
#pragma unroll
      for (int m = 0; m < kLookWin; ++m) {
        if (m < first_m) mine += val[m];
        else if (m == first_m && ((first_mask >> lane) & 1u)) mine += val[m];
      }
      excl += warp_sum(mine);
      if (first_m < kLookWin) return excl;
      break;
    }
    base -= 32 * kLookWin;
  }
  return excl;
}

__host__ __device__ __forceinline__ int ilog2_ceil(uint64_t v) {
  int b = 0;
  while ((1ull << b) < v) ++b;
  return b;
}

}  // namespace evs
