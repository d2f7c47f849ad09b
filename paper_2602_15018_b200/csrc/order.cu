// B200 (sm_100a) event-generation kernels.
//
//   k_prologue  : frame validation (reference ValueError semantics,
//                 model.py:28-39) + per-call accumulator reset.
//   (k_generate, K1, and the tile-order K2 live in k1_list.cu)
//   k_plan      : per-segment counts / capacity (parallel.py:261-273),
//                 histogram reduction + bin starts, work list for k_order.
//   k_hist      : digit histograms of a key array (generic sort passes).
//   k_order     : K2 -- one stable LSD radix pass (onesweep: warp match-any
//                 ranking, per-bin decoupled lookback across tiles) that
//                 turns pixel-major keys into canonical (t, y, x, p) order
//                 (canonical_sort, parallel.py:112-123).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace evs {

// ---------------------------------------------------------------------------
// prologue
// ---------------------------------------------------------------------------
template <bool VEC>
__global__ void __launch_bounds__(256) k_prologue(const float* __restrict__ frames, int64_t n,
                                                  int validate, int64_t* bad, int64_t* seg_res,
                                                  int nseg, StepDesc* desc, int64_t t_advance,
                                                  int64_t* zero2, int64_t n2) {
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) seg_res[i] = 0;
    for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) zero2[i] = 0;
    if (desc && threadIdx.x == 0) {  // advance the device clock for this step
      desc->cur_t0 = desc->next_t0;
      desc->next_t0 += t_advance;
      desc->cur_epoch = desc->next_epoch;
      desc->next_epoch += 8u;
    }
  }
  if (!validate) return;
  int64_t first = kNoBad;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (VEC) {
    const float4* f4 = reinterpret_cast<const float4*>(frames);
    const int64_t n4 = n >> 2;
    for (; i < n4; i += stride) {
      float4 v = __ldcs(f4 + i);
      if (!(v.x >= 0.f && v.x <= 1.f)) first = min(first, 4 * i + 0);
      else if (!(v.y >= 0.f && v.y <= 1.f)) first = min(first, 4 * i + 1);
      else if (!(v.z >= 0.f && v.z <= 1.f)) first = min(first, 4 * i + 2);
      else if (!(v.w >= 0.f && v.w <= 1.f)) first = min(first, 4 * i + 3);
    }
    for (int64_t j = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
      float v = frames[j];
      if (!(v >= 0.f && v <= 1.f)) first = min(first, j);
    }
  } else {
    for (; i < n; i += stride) {
      float v = frames[i];
      if (!(v >= 0.f && v <= 1.f)) first = min(first, i);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if ((threadIdx.x & 31) == 0 && first != kNoBad)
    atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)first);
}

cudaError_t launch_prologue(const float* frames, int64_t nframes_px, int64_t P, int validate,
                            int64_t* bad, int64_t* seg_res, int nseg, StepDesc* desc,
                            int64_t t_advance, int64_t* zero2, int64_t n2, cudaStream_t st) {
  (void)P;
  int64_t work = validate ? (nframes_px + 3) / 4 : 1;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  bool vec = ((uintptr_t)frames % 16) == 0;
  if (vec)
    k_prologue<true><<<(unsigned)blocks, 256, 0, st>>>(frames, nframes_px, validate, bad, seg_res, nseg,
                                                       desc, t_advance, zero2, n2);
  else
    k_prologue<false><<<(unsigned)blocks, 256, 0, st>>>(frames, nframes_px, validate, bad, seg_res, nseg,
                                                        desc, t_advance, zero2, n2);
  return cudaGetLastError();
}

// Raise a kernel's dynamic-smem limit once per (device, kernel) (smem_optin).
template <typename K>
static void ensure_smem(K k, size_t smem) {
  if (smem <= 48 * 1024) return;
  smem_optin(reinterpret_cast<const void*>(k));
}


// ---------------------------------------------------------------------------
// plan: counts, bin starts, work list
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_plan(PlanArgs a) {
  constexpr int NT = 256;
  __shared__ uint32_t s_scan32[NT / 32 + 1];
  __shared__ uint32_t s_run;
  const int seg = blockIdx.x, tid = threadIdx.x;
  const bool bad = *a.bad != kNoBad;
  const int64_t total = bad ? 0 : a.seg_total[seg];
  const int64_t written = total < a.cap ? total : a.cap;
  if (tid == 0 && a.out_count) {
    a.out_count[seg] = written;
    a.out_dropped[seg] = total - written;
  }
  if (a.hist) {
    const int NB = 1 << a.bits;
    const int per = (NB + NT - 1) / NT;
    uint32_t* h = const_cast<uint32_t*>(a.hist) + ((int64_t)seg * a.npass + a.pass) * kHistReps * NB;
    uint32_t c[8];
    uint32_t sum = 0;
    for (int j = 0; j < per && j < 8; ++j) {
      const int d = tid * per + j;
      uint32_t v = 0;
      if (d < NB) {
        for (int r = 0; r < kHistReps; ++r) {
          v += h[r * NB + d];
          if (a.zero_hist) h[r * NB + d] = 0;
        }
      }
      c[j] = bad ? 0 : v;
      sum += c[j];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan<NT, uint32_t>(sum, s_scan32, &tot);
    for (int j = 0; j < per && j < 8; ++j) {
      const int d = tid * per + j;
      if (d < NB) a.gstart[(int64_t)seg * NB + d] = ex;
      ex += c[j];
    }
  }
  if (seg == 0 && a.seg_tile_prefix) {
    if (tid == 0) s_run = 0;
    __syncthreads();
    for (int base = 0; base < a.nseg; base += NT) {
      const int i = base + tid;
      uint32_t nt = 0;
      if (i < a.nseg && !bad) {
        int64_t tt = a.seg_total[i];
        int64_t w = tt < a.cap ? tt : a.cap;
        nt = (uint32_t)((w + kOrdTile - 1) / kOrdTile);
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<NT, uint32_t>(nt, s_scan32, &tot);
      if (i < a.nseg) a.seg_tile_prefix[i] = s_run + ex;
      __syncthreads();
      if (tid == 0) s_run += tot;
      __syncthreads();
    }
    if (tid == 0) a.seg_tile_prefix[a.nseg] = s_run;
  }
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t st) {
  k_plan<<<a.nseg, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// generic digit histograms
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_hist(HistArgs a) {
  const int base_shift = a.base_shift;
  extern __shared__ uint32_t sh[];
  const int NB = 1 << a.bits;
  const int np = a.npass - a.pass0;
  for (int i = threadIdx.x; i < np * NB; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int seg = blockIdx.y;
  const int64_t n = a.seg_count[seg];
  const uint64_t* keys = a.keys + (int64_t)seg * a.seg_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    for (int p = 0; p < np; ++p) {
      const int sh_ = base_shift + (a.pass0 + p) * a.bits;
      atomicAdd(&sh[p * NB + (int)((k >> sh_) & (uint64_t)(NB - 1))], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < np * NB; i += blockDim.x) {
    const uint32_t c = sh[i];
    if (c) {
      const int p = a.pass0 + i / NB, d = i % NB;
      atomicAdd(a.hist + (((int64_t)seg * a.npass + p) * kHistReps + (blockIdx.x % kHistReps)) * NB + d, c);
    }
  }
}

cudaError_t launch_hist(const HistArgs& a, cudaStream_t st) {
  const int NB = 1 << a.bits;
  const size_t smem = (size_t)(a.npass - a.pass0) * NB * 4;
  dim3 grid(64, a.nseg);
  ensure_smem(k_hist, smem);
  k_hist<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2: one stable onesweep pass
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOrdThreads) k_order(OrderArgs a) {
  constexpr int NT = kOrdThreads, IPT = kOrdIpt, M = kOrdTile, NW = NT / 32;
  constexpr int MAXPER = (1 << kMaxDigitBits) / NT;  // bins per thread (<= 8)
  extern __shared__ __align__(16) unsigned char sm[];
  const int NB = 1 << a.bits;
  uint64_t* sorted = reinterpret_cast<uint64_t*>(sm);
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(sorted + M);  // [NW][NB]
  uint32_t* lstart = reinterpret_cast<uint32_t*>(wcnt + NW * NB);
  uint32_t* gbase = lstart + NB;
  __shared__ uint32_t s_w;
  __shared__ uint32_t s_scan[NW + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmask = (uint64_t)(NB - 1);
  const uint32_t epoch = a.desc ? a.desc->cur_epoch + a.epoch : a.epoch;

  for (;;) {
    const uint32_t total = a.seg_tile_prefix[a.nseg];
    if (tid == 0) {
      uint32_t w = atomicAdd(a.ctr, 1u);
      if (w == total + gridDim.x - 1) atomicExch(a.ctr, 0u);
      s_w = w;
    }
    __syncthreads();
    const uint32_t w = s_w;
    if (w >= total) break;
    int lo = 0, hi = a.nseg;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (a.seg_tile_prefix[mid] <= w) lo = mid; else hi = mid;
    }
    const int seg = lo;
    const int64_t tile = (int64_t)(w - a.seg_tile_prefix[seg]);
    const int64_t n = a.seg_count[seg];
    const int64_t kbase = tile * M;
    const int cnt = (int)((n - kbase) < M ? (n - kbase) : M);
    const uint64_t* kin = a.keys_in + (int64_t)seg * a.seg_stride + kbase;

    for (int d = lane; d < NB; d += 32) wcnt[warp * NB + d] = 0;
    __syncwarp();
    uint64_t key[IPT];
    uint32_t rank[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int idx = warp * 32 * IPT + k * 32 + lane;
      key[k] = idx < cnt ? __ldcs(kin + idx) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int idx = warp * 32 * IPT + k * 32 + lane;
      const bool valid = idx < cnt;
      const int d = valid ? (int)((key[k] >> a.shift) & dmask) : NB;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = wcnt[warp * NB + d];
        wcnt[warp * NB + d] = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      rank[k] = old + __popc(peers & lanemask_lt());
      __syncwarp();
    }
    __syncthreads();
    // per-bin warp offsets and tile totals
    for (int d = tid; d < NB; d += NT) {
      uint32_t acc = 0;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        uint32_t c = wcnt[w2 * NB + d];
        wcnt[w2 * NB + d] = (uint16_t)acc;
        acc += c;
      }
      gbase[d] = acc;  // tile total for bin d (temporarily)
    }
    __syncthreads();
    const int per = (NB + NT - 1) / NT;
    {
      uint32_t sum = 0;
      for (int j = 0; j < per; ++j) { int d = tid * per + j; if (d < NB) sum += gbase[d]; }
      uint32_t tot;
      uint32_t ex = block_excl_scan<NT, uint32_t>(sum, s_scan, &tot);
      for (int j = 0; j < per; ++j) { int d = tid * per + j; if (d < NB) { lstart[d] = ex; ex += gbase[d]; } }
    }
    __syncthreads();
    // per-bin decoupled lookback across this segment's tiles
    {
      uint64_t* stt = a.status + (int64_t)seg * a.max_tiles * NB;
      uint32_t tb[MAXPER];
      uint64_t ex[MAXPER];
      int64_t jj[MAXPER];
#pragma unroll
      for (int j = 0; j < MAXPER; ++j) {
        const int d = tid + j * NT;
        ex[j] = 0; jj[j] = tile - 1; tb[j] = 0;
        if (d < NB) {
          tb[j] = gbase[d];
          st_relaxed(stt + tile * NB + d, pack_status(tile == 0 ? kFlagInc : kFlagAgg, epoch, tb[j]));
        }
      }
      if (tile > 0) {
        bool pending = true;
        while (pending) {
          pending = false;
          uint64_t wv[MAXPER];
#pragma unroll
          for (int j = 0; j < MAXPER; ++j) {
            const int d = tid + j * NT;
            wv[j] = (d < NB && jj[j] >= 0) ? ld_relaxed(stt + jj[j] * NB + d) : 0ull;
          }
#pragma unroll
          for (int j = 0; j < MAXPER; ++j) {
            const int d = tid + j * NT;
            if (d < NB && jj[j] >= 0) {
              const uint32_t fl = status_flag(wv[j], epoch);
              if (fl == 0) { pending = true; __nanosleep(100); continue; }
              ex[j] += status_value(wv[j]);
              jj[j] = (fl == kFlagInc) ? -1 : jj[j] - 1;
              if (jj[j] >= 0) pending = true;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < MAXPER; ++j) {
          const int d = tid + j * NT;
          if (d < NB) st_relaxed(stt + tile * NB + d, pack_status(kFlagInc, epoch, ex[j] + tb[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < MAXPER; ++j) {
        const int d = tid + j * NT;
        if (d < NB) gbase[d] = a.gstart[(int64_t)seg * NB + d] + (uint32_t)ex[j] - lstart[d];
      }
    }
    __syncthreads();
    // local stable scatter into smem
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int idx = warp * 32 * IPT + k * 32 + lane;
      if (idx < cnt) {
        const int d = (int)((key[k] >> a.shift) & dmask);
        sorted[lstart[d] + wcnt[warp * NB + d] + rank[k]] = key[k];
      }
    }
    __syncthreads();
    const int64_t ob = (int64_t)seg * a.seg_stride;
    if (a.final_soa) {
      const int64_t tb0 = a.seg_tbase ? a.seg_tbase[seg] : 0;
      for (int i = tid; i < cnt; i += NT) {
        const uint64_t k = sorted[i];
        const int64_t g = ob + (int64_t)(uint32_t)(gbase[(int)((k >> a.shift) & dmask)] + (uint32_t)i);
        a.out_t[g] = tb0 + (int64_t)(k >> kKeyPixBits);
        a.out_x[g] = (uint16_t)((k >> 1) & 0xffffu);
        a.out_y[g] = (uint16_t)((k >> 17) & 0xffffu);
        a.out_p[g] = (k & 1u) ? (int8_t)1 : (int8_t)-1;
      }
    } else {
      for (int i = tid; i < cnt; i += NT) {
        const uint64_t k = sorted[i];
        a.keys_out[ob + (int64_t)(uint32_t)(gbase[(int)((k >> a.shift) & dmask)] + (uint32_t)i)] = k;
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_order(const OrderArgs& a, int sm_count, cudaStream_t st) {
  const int NB = 1 << a.bits;
  const size_t smem = (size_t)kOrdTile * 8 + (size_t)(kOrdThreads / 32) * NB * 2 + (size_t)NB * 8;
  ensure_smem(k_order, smem);
  // occupancy per digit width, cached (the query is slow relative to a launch)
  static int occ_cache[kMaxDigitBits + 1] = {0};
  int per_sm = occ_cache[a.bits];
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_order, kOrdThreads, smem);
    if (per_sm < 1) per_sm = 1;
    occ_cache[a.bits] = per_sm;
  }
  k_order<<<sm_count * per_sm, kOrdThreads, smem, st>>>(a);
  return cudaGetLastError();
}


}  // namespace evs
