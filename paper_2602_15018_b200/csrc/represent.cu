// Event representations and post-processing on device batches.
//
//   evs_accumulate      accumulate_events_to_image (model.py:249-262): signed
//                       polarity sum per pixel over t in [t_end - w, t_end).
//   evs_voxel           repo-defined 5-bin (B-bin) voxel grid: exact integer
//                       bilinear-in-time weights, one f32 rounding at the end.
//   evs_limit_bandwidth limit_bandwidth (model.py:215-246): keep the first
//                       floor(rate * window) events of every window that
//                       tiles forward from the first event.
//   evs_voxel_segments  the voxel grid over many device-counted segments (a
//                       step's S x T output rows, per-frame noise buffers)
//                       without a host round trip (EventSimulator.voxel_window).
// All accumulate with global int64 atomics (exact, order independent).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/evsim_b200.h"
#include "common.cuh"
#include "kernels.cuh"

namespace evs {

__global__ void __launch_bounds__(256) k_accumulate(int64_t n, const int64_t* __restrict__ t,
                                                    const uint16_t* __restrict__ x,
                                                    const uint16_t* __restrict__ y,
                                                    const int8_t* __restrict__ p, int64_t lo, int64_t hi,
                                                    int32_t W, unsigned long long* grid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ti = t[i];
    if (ti >= lo && ti < hi)  // model.py:259
      atomicAdd(grid + (int64_t)y[i] * W + x[i], (unsigned long long)(int64_t)p[i]);
  }
}

// floor(tau / D) to within +-1 without a 64-bit integer division (tau, D <
// 2^53 are exact doubles); the exact integer weight test below decides, so
// scanning b0-1 .. b0+2 visits every bin with weight > 0
__device__ __forceinline__ int64_t vox_bin_guess(int64_t tau, int64_t D) {
  return (int64_t)((double)tau / (double)D);
}

// voxel numerators: acc[b][pix] += p * max(0, D - |b*D - (B-1)(t - t0)|)
__global__ void __launch_bounds__(256) k_voxel_acc(int64_t n, const int64_t* __restrict__ t,
                                                   const uint16_t* __restrict__ x,
                                                   const uint16_t* __restrict__ y,
                                                   const int8_t* __restrict__ p, int64_t t0, int64_t t1,
                                                   int32_t B, int32_t W, int64_t P, long long* acc) {
  const int64_t D = t1 - t0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ti = t[i];
    if (ti < t0 || ti >= t1) continue;
    const int64_t tau = (int64_t)(B - 1) * (ti - t0);
    const int64_t pix = (int64_t)y[i] * W + x[i];
    const int64_t b0 = vox_bin_guess(tau, D);  // the bins with weight > 0 are among b0-1 .. b0+2
    for (int64_t b = b0 > 0 ? b0 - 1 : 0; b <= b0 + 2 && b < B; ++b) {
      int64_t d = b * D - tau;
      d = d < 0 ? -d : d;
      const int64_t w = D - d;
      if (w > 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + b * P + pix),
                           (unsigned long long)((int64_t)p[i] * w));
    }
  }
}

// the same numerators over many segments: segment s holds counts[s * cstride]
// events at offset s * seg_stride (evs_step output rows, per-frame noise buffers)
__global__ void __launch_bounds__(256) k_voxel_acc_seg(const int64_t* __restrict__ counts, int64_t cstride,
                                                       int64_t seg_stride, const int64_t* __restrict__ t,
                                                       const uint16_t* __restrict__ x,
                                                       const uint16_t* __restrict__ y,
                                                       const int8_t* __restrict__ p, int64_t t0, int64_t t1,
                                                       int32_t B, int32_t W, int64_t P, long long* acc) {
  const int64_t D = t1 - t0;
  const int64_t seg = blockIdx.y;
  int64_t n = counts[seg * cstride];
  if (seg_stride > 0 && n > seg_stride) n = seg_stride;  // (an overflowed noise buffer: redone by the caller)
  const int64_t base = seg * seg_stride;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + j;
    const int64_t ti = t[i];
    if (ti < t0 || ti >= t1) continue;
    const int64_t tau = (int64_t)(B - 1) * (ti - t0);
    const int64_t pix = (int64_t)y[i] * W + x[i];
    if ((uint64_t)pix >= (uint64_t)P) continue;  // (bounds: the caller's segments are sensor events)
    const int64_t b0 = vox_bin_guess(tau, D);
    for (int64_t b = b0 > 0 ? b0 - 1 : 0; b <= b0 + 2 && b < B; ++b) {
      int64_t d = b * D - tau;
      d = d < 0 ? -d : d;
      const int64_t w = D - d;
      if (w > 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + b * P + pix),
                           (unsigned long long)((int64_t)p[i] * w));
    }
  }
}

__global__ void __launch_bounds__(256) k_voxel_finalize(int64_t m, const long long* __restrict__ acc, int64_t D,
                                                        float* out) {
  const double inv = 1.0 / (double)D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)((double)acc[i] / (double)D);
  (void)inv;
}

// ---- voxel grid from a step's tile regions ---------------------------------
// The kept events of (segment, tile) are the first nkeep keys of its region
// (t_rel << 33 | y << 17 | x << 1 | p; capacity cut as in k_tile_order);
// t = seg_tbase + t_rel.  One CTA per 1024-pixel tile accumulates its own
// pixels' exact numerators in shared memory (no global atomics); every pixel
// of the tile is written, so the output needs no clearing.
//   NARROW ((B-1) * D < 2^30): 32-bit bin arithmetic and 32-bit shared
//   atomics, plus a per-pixel event count; a tile where count * D could reach
//   2^31 (never at camera rates) is redone with the 64-bit accumulators.
//   wide: 64-bit arithmetic and 64-bit shared atomics throughout.
struct VoxTileSrc {
  const uint64_t* src;
  int64_t nkeep, tb;
};
__device__ __forceinline__ VoxTileSrc vox_tile_src(const StepVoxArgs& a, int q, int f) {
  const int64_t seg = (int64_t)a.s * a.T + f;
  const int64_t sq = seg * a.ntiles + q;
  const int64_t nq = a.tile_count[sq];
  int64_t nkeep = a.cap - a.tile_base[sq];
  nkeep = nkeep < 0 ? 0 : (nkeep > nq ? nq : nkeep);
  const int64_t ov = a.tile_ovf[sq];
  VoxTileSrc r;
  r.src = ov >= 0 ? a.ovf_area + seg * a.ovf_cap + ov : a.region + sq * a.tile_cap;
  r.nkeep = nkeep;
  r.tb = a.seg_tbase[seg];
  return r;
}

__global__ void __launch_bounds__(256) k_step_voxel(StepVoxArgs a, int narrow) {
  extern __shared__ __align__(16) unsigned char vsm[];
  const int q = blockIdx.x, tid = threadIdx.x;
  const int64_t D = a.t1 - a.t0;
  const int TP = a.tile_px;  // pixels per tile (<= kGenTile)
  const int64_t tile0 = (int64_t)q * TP;
  const bool ok = *a.bad == kNoBad;
  __shared__ int s_wide;
  if (narrow) {
    int* acc = reinterpret_cast<int*>(vsm);        // [B][TP]
    int* cnt = acc + a.B * TP;                     // [TP]
    for (int i = tid; i < (a.B + 1) * TP; i += blockDim.x) acc[i] = 0;
    if (tid == 0) s_wide = 0;
    __syncthreads();
    const int d32 = (int)D;
    const float invD = 1.0f / (float)D;
    if (ok) {
      for (int f = 0; f < a.T; ++f) {
        const VoxTileSrc r = vox_tile_src(a, q, f);
        for (int64_t i = tid; i < r.nkeep; i += blockDim.x) {
          const uint64_t k = __ldcs(r.src + i);
          const int64_t t = r.tb + (int64_t)(k >> kKeyPixBits);
          if (t < a.t0 || t >= a.t1) continue;
          const int lp = (int)((int64_t)((k >> 17) & 0xffffu) * a.W + (int64_t)((k >> 1) & 0xffffu) - tile0);
          const int pol = (k & 1u) ? 1 : -1;
          const int tau = (a.B - 1) * (int)(t - a.t0);
          int b0 = (int)((float)tau * invD);  // floor(tau / D) within +-1, corrected below
          if (b0 * d32 > tau) --b0;
          else if ((b0 + 1) * d32 <= tau) ++b0;
          atomicAdd(cnt + lp, 1);
          for (int b = b0; b <= b0 + 1 && b < a.B; ++b) {
            const int d = b * d32 - tau;
            const int w = d32 - (d < 0 ? -d : d);
            if (w > 0) atomicAdd(acc + b * TP + lp, pol * w);
          }
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < TP; i += blockDim.x)
      if ((int64_t)cnt[i] * D >= (1ll << 31)) s_wide = 1;
    __syncthreads();
    if (!s_wide) {
      for (int i = tid; i < a.B * TP; i += blockDim.x) {
        const int b = i / TP, lp = i % TP;
        const int64_t pix = tile0 + lp;
        if (pix >= a.P) continue;
        const long long v = acc[i];
        if (a.out) a.out[(int64_t)b * a.P + pix] = (float)((double)v / (double)D);  // = k_voxel_finalize
        else a.acc_out[(int64_t)b * a.P + pix] = v;
      }
      return;
    }
    __syncthreads();  // (redo this tile below with 64-bit accumulators)
  }
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(vsm);  // [B][TP]
  for (int i = tid; i < a.B * TP; i += blockDim.x) acc[i] = 0ull;
  __syncthreads();
  if (ok) {
    for (int f = 0; f < a.T; ++f) {
      const VoxTileSrc r = vox_tile_src(a, q, f);
      for (int64_t i = tid; i < r.nkeep; i += blockDim.x) {
        const uint64_t k = __ldcs(r.src + i);
        const int64_t t = r.tb + (int64_t)(k >> kKeyPixBits);
        if (t < a.t0 || t >= a.t1) continue;
        const int lp = (int)((int64_t)((k >> 17) & 0xffffu) * a.W + (int64_t)((k >> 1) & 0xffffu) - tile0);
        const long long pol = (k & 1u) ? 1 : -1;
        const int64_t tau = (int64_t)(a.B - 1) * (t - a.t0);
        const int64_t b0 = tau / D;
        for (int64_t b = b0; b <= b0 + 1 && b < a.B; ++b) {
          int64_t d = b * D - tau;
          d = d < 0 ? -d : d;
          const int64_t w = D - d;
          if (w > 0) atomicAdd(acc + b * TP + lp, (unsigned long long)(pol * w));
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < a.B * TP; i += blockDim.x) {
    const int b = i / TP, lp = i % TP;
    const int64_t pix = tile0 + lp;
    if (pix >= a.P) continue;
    const long long v = (long long)acc[i];
    if (a.out) a.out[(int64_t)b * a.P + pix] = (float)((double)v / (double)D);  // = k_voxel_finalize
    else a.acc_out[(int64_t)b * a.P + pix] = v;
  }
}

cudaError_t launch_step_voxel(const StepVoxArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)a.B * kGenTile * sizeof(long long);  // >= the narrow (B + 1) x 4 B
  smem_optin(reinterpret_cast<const void*>(k_step_voxel));
  const int narrow = (int64_t)(a.B - 1) * (a.t1 - a.t0) < (1ll << 30) ? 1 : 0;
  k_step_voxel<<<a.ntiles, 256, smem, st>>>(a, narrow);
  return cudaGetLastError();
}

// ---- event histograms of every stream from a step's tile regions ------------
// accumulate_events_to_image (model.py:249-262) of each stream's events of the
// step with t in [lo, hi): grid (tile, stream), the tile's pixels summed in
// shared memory (|sum| <= events of the pixel: int32 is exact), int64 out.
__global__ void __launch_bounds__(256) k_step_hist(StepVoxArgs a, int64_t lo, int64_t hi, int64_t* out) {
  __shared__ int acc[kGenTile];
  const int q = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  for (int i = tid; i < kGenTile; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const int TP = a.tile_px;  // pixels per tile (<= kGenTile)
  const int64_t tile0 = (int64_t)q * TP;
  if (*a.bad == kNoBad) {
    StepVoxArgs b = a;
    b.s = s;
    for (int f = 0; f < a.T; ++f) {
      const VoxTileSrc r = vox_tile_src(b, q, f);
      for (int64_t i = tid; i < r.nkeep; i += blockDim.x) {
        const uint64_t k = __ldcs(r.src + i);
        const int64_t t = r.tb + (int64_t)(k >> kKeyPixBits);
        if (t < lo || t >= hi) continue;  // model.py:259
        const int lp = (int)((int64_t)((k >> 17) & 0xffffu) * a.W + (int64_t)((k >> 1) & 0xffffu) - tile0);
        atomicAdd(acc + lp, (k & 1u) ? 1 : -1);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < TP; i += blockDim.x) {
    const int64_t pix = tile0 + i;
    if (pix < a.P) out[(int64_t)s * a.P + pix] = acc[i];
  }
}

cudaError_t launch_step_hist(const StepVoxArgs& a, int S, int64_t lo, int64_t hi, int64_t* out, cudaStream_t st) {
  k_step_hist<<<dim3(a.ntiles, S), 256, 0, st>>>(a, lo, hi, out);
  return cudaGetLastError();
}

// ---- segment compaction -----------------------------------------------------
// out[prefix_g + i] = in[g * seg_stride + i] for i < counts[g], all four SoA
// arrays; prefix_g = sum of the earlier counts (each CTA sums them itself).
__global__ void __launch_bounds__(256) k_compact_segments(const int64_t* __restrict__ counts, int64_t seg_stride,
                                                          const int64_t* __restrict__ t, const uint16_t* __restrict__ x,
                                                          const uint16_t* __restrict__ y, const int8_t* __restrict__ p,
                                                          int64_t* ot, uint16_t* ox, uint16_t* oy, int8_t* op,
                                                          int64_t out_cap) {
  __shared__ int64_t s_pre[9];
  const int g = blockIdx.y, tid = threadIdx.x;
  int64_t part = 0;
  for (int j = tid; j < g; j += blockDim.x) part += counts[j];
  int64_t tot;
  block_excl_scan<256, int64_t>(part, s_pre, &tot);
  const int64_t pre = tot;
  int64_t n = counts[g];
  if (pre + n > out_cap) n = out_cap - pre;  // (caller falls back when the total exceeds out_cap)
  const int64_t src = (int64_t)g * seg_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ot[pre + i] = __ldcs(t + src + i);
    ox[pre + i] = __ldcs(x + src + i);
    oy[pre + i] = __ldcs(y + src + i);
    op[pre + i] = __ldcs(p + src + i);
  }
}

// ---- log_transform (model.py:28-39) -----------------------------------------
__global__ void __launch_bounds__(256) k_log_transform(int64_t n, const float* __restrict__ v, double eps,
                                                       double* __restrict__ out, int64_t* bad) {
  int64_t first = kNoBad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[i];
    if (!(x >= 0.f && x <= 1.f)) first = min(first, i);  // NaN / inf / out of range (model.py:33-38)
    out[i] = log((double)x + eps);                          // model.py:39, f64
  }
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if ((threadIdx.x & 31) == 0 && first != kNoBad)
    atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)first);
}

// ---- packed keys of a step's segments (gather payload) ---------------------
template <typename K>
__global__ void __launch_bounds__(256) k_pack_segments(const int64_t* __restrict__ counts, int64_t seg_stride,
                                                       const int64_t* __restrict__ t, const uint16_t* __restrict__ x,
                                                       const uint16_t* __restrict__ y, const int8_t* __restrict__ p,
                                                       int64_t t_base, int y_off, int ysh, int xsh, K* out,
                                                       int64_t* offs, int64_t out_cap) {
  __shared__ int64_t s_pre[9];
  const int g = blockIdx.y, tid = threadIdx.x;
  int64_t part = 0;
  for (int j = tid; j < g; j += blockDim.x) part += counts[j];
  int64_t tot;
  block_excl_scan<256, int64_t>(part, s_pre, &tot);
  const int64_t pre = tot;
  int64_t n = counts[g];
  if (blockIdx.x == 0 && tid == 0) {
    offs[g] = pre;
    if (g == gridDim.y - 1) offs[g + 1] = pre + n;
  }
  if (pre + n > out_cap) n = out_cap - pre;
  const int64_t src = (int64_t)g * seg_stride;
  const int tsh = ysh + xsh + 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t tr = (uint64_t)(__ldcs(t + src + i) - t_base);
    const uint64_t k = (tr << tsh) | ((uint64_t)(__ldcs(y + src + i) + y_off) << (xsh + 1)) |
                       ((uint64_t)__ldcs(x + src + i) << 1) | (__ldcs(p + src + i) > 0 ? 1u : 0u);
    out[pre + i] = (K)k;
  }
}

// ---- limit_bandwidth -------------------------------------------------------
// keep[i] = rank of i in its window < cap; per-block kept counts; unsorted flag
__global__ void __launch_bounds__(1024) k_lb_flags(int64_t n, const int64_t* __restrict__ t, int64_t window,
                                                   int64_t cap, uint8_t* keep, int64_t* blk, int64_t* flags) {
  __shared__ int64_t s_scan[33];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t k = 0;
  if (i < n) {
    const int64_t t0 = t[0], ti = t[i];
    if (i > 0 && ti < t[i - 1]) flags[0] = 1;  // model.py:232: requires a timestamp-sorted batch
    const int64_t w = (ti - t0) / window;
    const int64_t wstart = t0 + w * window;
    int64_t lo = 0, hi = i;  // first index with t >= wstart (sorted input)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (t[mid] < wstart) lo = mid + 1; else hi = mid;
    }
    k = (i - lo) < cap ? 1 : 0;
    keep[i] = (uint8_t)k;
  }
  int64_t tot;
  block_excl_scan<1024, int64_t>(k, s_scan, &tot);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_blocks(int64_t nb, int64_t* blk, int64_t* total) {
  __shared__ int64_t s_scan[33];
  __shared__ int64_t run;
  if (threadIdx.x == 0) run = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? blk[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<1024, int64_t>(v, s_scan, &tot);
    if (i < nb) blk[i] = run + ex;
    __syncthreads();
    if (threadIdx.x == 0) run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[0] = run;
}

__global__ void __launch_bounds__(1024) k_lb_scatter(int64_t n, const int64_t* __restrict__ t,
                                                     const uint16_t* __restrict__ x,
                                                     const uint16_t* __restrict__ y,
                                                     const int8_t* __restrict__ p, const uint8_t* keep,
                                                     const int64_t* blk, int64_t* ot, uint16_t* ox,
                                                     uint16_t* oy, int8_t* op) {
  __shared__ int64_t s_scan[33];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t k = i < n ? keep[i] : 0;
  int64_t tot;
  const int64_t ex = block_excl_scan<1024, int64_t>(k, s_scan, &tot);
  if (k) {
    const int64_t o = blk[blockIdx.x] + ex;
    ot[o] = t[i]; ox[o] = x[i]; oy[o] = y[i]; op[o] = p[i];
  }
}

}  // namespace evs

using namespace evs;

static inline unsigned grid_for(int64_t n, int64_t cap_blocks) {
  int64_t b = (n + 255) / 256;
  if (b > cap_blocks) b = cap_blocks;
  return (unsigned)(b < 1 ? 1 : b);
}

extern "C" {

evs_status evs_accumulate(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p,
                          int64_t window_us, int64_t t_end, int32_t width, int32_t height, int64_t* grid,
                          void* stream) {
  if (n < 0 || width < 1 || height < 1 || !grid) return EVS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(grid, 0, sizeof(int64_t) * (size_t)width * height, st) != cudaSuccess) return EVS_ERR_CUDA;
  if (n > 0)
    k_accumulate<<<grid_for(n, 148 * 16), 256, 0, st>>>(n, t, x, y, p, t_end - window_us, t_end, width,
                                                       reinterpret_cast<unsigned long long*>(grid));
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

size_t evs_voxel_workspace_bytes(int32_t bins, int32_t width, int32_t height) {
  return (size_t)bins * width * height * sizeof(long long);
}

evs_status evs_voxel(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p,
                     int64_t t0, int64_t t1, int32_t bins, int32_t width, int32_t height, float* out,
                     void* workspace, size_t ws_bytes, void* stream) {
  if (n < 0 || t1 <= t0 || bins < 2 || width < 1 || height < 1 || !out) return EVS_ERR_ARG;
  const int64_t P = (int64_t)width * height;
  if (!workspace || ws_bytes < (size_t)bins * P * sizeof(long long)) return EVS_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long* acc = static_cast<long long*>(workspace);
  if (cudaMemsetAsync(acc, 0, (size_t)bins * P * sizeof(long long), st) != cudaSuccess) return EVS_ERR_CUDA;
  if (n > 0) k_voxel_acc<<<grid_for(n, 148 * 16), 256, 0, st>>>(n, t, x, y, p, t0, t1, bins, width, P, acc);
  k_voxel_finalize<<<grid_for((int64_t)bins * P, 148 * 16), 256, 0, st>>>((int64_t)bins * P, acc, t1 - t0, out);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_voxel_segments(int32_t nseg, const int64_t* counts, int64_t counts_stride, int64_t seg_stride,
                              const int64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p,
                              int64_t t0, int64_t t1, int32_t bins, int32_t width, int32_t height,
                              int32_t flags, float* out, void* workspace, size_t ws_bytes, void* stream) {
  if (nseg < 0 || nseg > 65535 || t1 <= t0 || bins < 2 || width < 1 || height < 1) return EVS_ERR_ARG;
  if ((flags & EVS_VOXEL_FINALIZE) && !out) return EVS_ERR_ARG;
  if (nseg > 0 && (!counts || !t || !x || !y || !p || seg_stride < 0 || counts_stride < 1)) return EVS_ERR_ARG;
  const int64_t P = (int64_t)width * height;
  if (!workspace || ws_bytes < (size_t)bins * P * sizeof(long long)) return EVS_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long* acc = static_cast<long long*>(workspace);
  if ((flags & EVS_VOXEL_CLEAR) &&
      cudaMemsetAsync(acc, 0, (size_t)bins * P * sizeof(long long), st) != cudaSuccess)
    return EVS_ERR_CUDA;
  if (nseg > 0) {
    const int bx = (int)((148 * 8 + nseg - 1) / nseg);
    k_voxel_acc_seg<<<dim3(bx < 4 ? 4 : bx, nseg), 256, 0, st>>>(counts, counts_stride, seg_stride, t, x, y, p,
                                                               t0, t1, bins, width, P, acc);
  }
  if (flags & EVS_VOXEL_FINALIZE)
    k_voxel_finalize<<<grid_for((int64_t)bins * P, 148 * 16), 256, 0, st>>>((int64_t)bins * P, acc, t1 - t0, out);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_compact_segments(int32_t nseg, const int64_t* counts, int64_t seg_stride, const int64_t* t,
                                const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t* out_t,
                                uint16_t* out_x, uint16_t* out_y, int8_t* out_p, int64_t out_capacity,
                                void* stream) {
  if (nseg < 0 || nseg > 65535 || seg_stride < 0 || out_capacity < 0) return EVS_ERR_ARG;
  if (nseg == 0) return EVS_OK;
  if (!counts || !t || !x || !y || !p || !out_t || !out_x || !out_y || !out_p) return EVS_ERR_ARG;
  const int bx = (148 * 8 + nseg - 1) / nseg;
  k_compact_segments<<<dim3(bx < 2 ? 2 : bx, nseg), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, seg_stride, t, x, y, p, out_t, out_x, out_y, out_p, out_capacity);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_log_transform(int64_t n, const float* values, double log_eps, double* out, int64_t* bad_index,
                             void* stream) {
  if (n < 0 || !(log_eps > 0) || !bad_index) return EVS_ERR_ARG;
  if (n == 0) return EVS_OK;
  if (!values || !out) return EVS_ERR_ARG;
  k_log_transform<<<grid_for(n, 148 * 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, values, log_eps, out,
                                                                                        bad_index);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

evs_status evs_pack_segments(int32_t nseg, const int64_t* counts, int64_t seg_stride, const int64_t* t,
                             const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t t_base,
                             int32_t y_offset, int32_t key_bytes, int32_t ybits, int32_t xbits, void* out_keys,
                             int64_t* seg_offsets, int64_t out_capacity, void* stream) {
  if (nseg < 1 || nseg > 65535 || seg_stride < 0 || out_capacity < 0) return EVS_ERR_ARG;
  if (!counts || !t || !x || !y || !p || !out_keys || !seg_offsets) return EVS_ERR_ARG;
  if (ybits < 1 || xbits < 1 || ybits > 16 || xbits > 16 || y_offset < 0) return EVS_ERR_ARG;
  if (key_bytes == 8 && (ybits != 16 || xbits != 16)) return EVS_ERR_ARG;
  const int bx = (148 * 8 + nseg - 1) / nseg;
  const dim3 grid(bx < 2 ? 2 : bx, nseg);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (key_bytes == 4)
    k_pack_segments<uint32_t><<<grid, 256, 0, st>>>(counts, seg_stride, t, x, y, p, t_base, y_offset, ybits, xbits,
                                                   static_cast<uint32_t*>(out_keys), seg_offsets, out_capacity);
  else if (key_bytes == 8)
    k_pack_segments<uint64_t><<<grid, 256, 0, st>>>(counts, seg_stride, t, x, y, p, t_base, y_offset, ybits, xbits,
                                                   static_cast<uint64_t*>(out_keys), seg_offsets, out_capacity);
  else
    return EVS_ERR_ARG;
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

size_t evs_limit_bandwidth_workspace_bytes(int64_t n) {
  const int64_t nb = (n + 1023) / 1024 + 1;
  return (size_t)n + 16 + (size_t)nb * 8 + 64;
}

evs_status evs_limit_bandwidth(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                               const int8_t* p, int64_t cap, int64_t window_us, int64_t* ot, uint16_t* ox,
                               uint16_t* oy, int8_t* op, int64_t* meta_out, void* workspace, size_t ws_bytes,
                               void* stream) {
  if (n < 1 || window_us <= 0 || cap < 0 || !meta_out) return EVS_ERR_ARG;
  if (!workspace || ws_bytes < evs_limit_bandwidth_workspace_bytes(n)) return EVS_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nb = (n + 1023) / 1024;
  char* w = static_cast<char*>(workspace);
  int64_t* blk = reinterpret_cast<int64_t*>(w);
  uint8_t* keep = reinterpret_cast<uint8_t*>(w + ((nb + 1) * 8 + 63) / 64 * 64);
  // meta_out: [0] kept count, [1] unsorted flag
  if (cudaMemsetAsync(meta_out, 0, 2 * sizeof(int64_t), st) != cudaSuccess) return EVS_ERR_CUDA;
  k_lb_flags<<<(unsigned)nb, 1024, 0, st>>>(n, t, window_us, cap, keep, blk, meta_out + 1);
  k_scan_blocks<<<1, 1024, 0, st>>>(nb, blk, meta_out);
  k_lb_scatter<<<(unsigned)nb, 1024, 0, st>>>(n, t, x, y, p, keep, blk, ot, ox, oy, op);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

}  // extern "C"
