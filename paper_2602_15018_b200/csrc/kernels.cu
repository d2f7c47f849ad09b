// B200 (sm_100a) event-generation kernels.
//
//   k_prologue  : frame validation (reference ValueError semantics,
//                 model.py:28-39) + per-call accumulator reset.
//   k_generate  : K1 -- fused log / threshold / crossing count / refractory /
//                 state update, warp-ballot chunk stats, block scan +
//                 decoupled-lookback placement of the variable-length
//                 per-pixel output in pixel-major (serial) order
//                 (model.py:79-171 == parallel.py:126-273), smem-staged
//                 coalesced writes, per-tile t_rel histogram.
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
                                                  int nseg, StepDesc* desc, int64_t t_advance) {
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) seg_res[i] = 0;
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
                            int64_t t_advance, cudaStream_t st) {
  (void)P;
  int64_t work = validate ? (nframes_px + 3) / 4 : 1;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  bool vec = ((uintptr_t)frames % 16) == 0;
  if (vec)
    k_prologue<true><<<(unsigned)blocks, 256, 0, st>>>(frames, nframes_px, validate, bad, seg_res, nseg,
                                                       desc, t_advance);
  else
    k_prologue<false><<<(unsigned)blocks, 256, 0, st>>>(frames, nframes_px, validate, bad, seg_res, nseg,
                                                        desc, t_advance);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K1: fused generate
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t t_rel_of(int j, double thd, double adiff, double dtd, int64_t dt) {
  // model.py:144-146: int(((j*th)/|diff|)*dt), clamped to dt-1
  int64_t tr = (int64_t)((((double)j * thd) / adiff) * dtd);
  return tr > dt - 1 ? dt - 1 : tr;
}

template <int MODE>
__device__ __forceinline__ void put_event(const GenArgs& a, int64_t segoff, int64_t g, uint64_t key,
                                          int64_t tprev) {
  if (MODE == 0) {
    a.out_t[segoff + g] = tprev + (int64_t)(key >> kKeyPixBits);
    a.out_x[segoff + g] = (uint16_t)((key >> 1) & 0xffffu);
    a.out_y[segoff + g] = (uint16_t)((key >> 17) & 0xffffu);
    a.out_p[segoff + g] = (key & 1u) ? (int8_t)1 : (int8_t)-1;
  } else {
    a.keys[segoff + g] = key;
  }
}

template <bool VEC, bool REFR, bool UNI, int MODE>
__global__ void __launch_bounds__(kGenThreads, 3) k_generate(GenArgs a) {
  constexpr int NT = kGenThreads, VPT = kGenVpt, TILE = kGenTile, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* stg = reinterpret_cast<uint64_t*>(smem_raw);  // [kGenStage]
  uint32_t* hs = reinterpret_cast<uint32_t*>(stg + kGenStage);
  __shared__ int64_t s_scan[NW + 1];
  __shared__ uint32_t s_id;
  __shared__ int64_t s_base;
  __shared__ int s_res;

  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    uint32_t id = atomicAdd(a.tile_ctr, 1u);
    if (id == gridDim.x - 1) atomicExch(a.tile_ctr, 0u);  // last fetch: reset for next launch
    s_id = id;
    s_res = 0;
  }
  const int NB = a.hist ? (1 << a.hist_bits) : 0;
  for (int d = tid; d < NB; d += NT) hs[d] = 0;
  __syncthreads();
  if (*a.bad != kNoBad) return;  // validation failed: state is not touched

  const uint32_t id = s_id;
  const int s = (int)(id / (uint32_t)a.ntiles);
  const int tile = (int)(id % (uint32_t)a.ntiles);
  const int64_t P = a.P;
  const uint32_t epoch = a.desc ? a.desc->cur_epoch : a.epoch;
  const int64_t clock_t0 = a.desc ? a.desc->cur_t0 : a.t0;
  const int64_t pix0 = (int64_t)tile * TILE + (int64_t)tid * VPT;
  const bool full = VEC && (pix0 + VPT <= P);
  float* refp = a.ref + (int64_t)s * P;
  int64_t* lastp = a.last + (int64_t)s * P;

  float r[VPT], thp[VPT], thn[VPT];
  int64_t lt[VPT];
  bool dirty[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) { r[k] = 0.f; lt[k] = 0; dirty[k] = false; thp[k] = a.thp_u; thn[k] = a.thn_u; }
  if (full) {
    float4 q = *reinterpret_cast<const float4*>(refp + pix0);
    r[0] = q.x; r[1] = q.y; r[2] = q.z; r[3] = q.w;
    if (REFR) {
      longlong2 l0 = *reinterpret_cast<const longlong2*>(lastp + pix0);
      longlong2 l1 = *reinterpret_cast<const longlong2*>(lastp + pix0 + 2);
      lt[0] = l0.x; lt[1] = l0.y; lt[2] = l1.x; lt[3] = l1.y;
    }
    if (!UNI) {
      float4 p4 = *reinterpret_cast<const float4*>(a.thp + (int64_t)s * P + pix0);
      float4 n4 = *reinterpret_cast<const float4*>(a.thn + (int64_t)s * P + pix0);
      thp[0] = p4.x; thp[1] = p4.y; thp[2] = p4.z; thp[3] = p4.w;
      thn[0] = n4.x; thn[1] = n4.y; thn[2] = n4.z; thn[3] = n4.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if (pix0 + k < P) {
        r[k] = refp[pix0 + k];
        if (REFR) lt[k] = lastp[pix0 + k];
        if (!UNI) { thp[k] = a.thp[(int64_t)s * P + pix0 + k]; thn[k] = a.thn[(int64_t)s * P + pix0 + k]; }
      }
    }
  }

  for (int f = 0; f < a.T; ++f) {
    const int seg = s * a.T + f;
    int64_t tprev, tnow;
    if (a.t_bounds) {
      tprev = a.t_bounds[(int64_t)s * (a.T + 1) + f];
      tnow = a.t_bounds[(int64_t)s * (a.T + 1) + f + 1];
    } else {
      tprev = clock_t0 + (int64_t)f * a.tick;
      tnow = tprev + a.tick;
    }
    const int64_t dt = tnow - tprev;
    const double dtd = (double)dt;
    const float* fr = a.frames + ((int64_t)s * a.T + f) * P;
    float v[VPT];
    if (full) {
      float4 q = __ldcs(reinterpret_cast<const float4*>(fr + pix0));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < VPT; ++k) v[k] = (pix0 + k < P) ? __ldcs(fr + pix0 + k) : 0.f;
    }

    // ---- lane math, count pass (model.py:124-163) ----
    double adiff[VPT];
    float thv[VPT];
    int nn[VPT], kept[VPT];
    int64_t last0[VPT];
    int tot = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      nn[k] = 0; kept[k] = 0; adiff[k] = 0.0; thv[k] = 1.f; last0[k] = lt[k];
      if (pix0 + k < P) {
        const double ln = log((double)v[k] + a.log_eps);  // model.py:39 (f64)
        const double ls = (double)r[k];
        const double diff = ln - ls;
        if (diff != 0.0) {
          const bool pos = diff > 0.0;
          const float th = pos ? thp[k] : thn[k];
          const double thd = (double)th;
          const double ad = pos ? diff : -diff;
          double q = ad / thd + 1e-4;  // model.py:137
          int n = q >= 2147483647.0 ? 2147483647 : (int)q;
          if (n > 0) {
            adiff[k] = ad; thv[k] = pos ? th : -th; nn[k] = n;
            int kc;
            if (REFR) {
              int64_t l = lt[k];
              kc = 0;
              for (int j = 1; j <= n; ++j) {
                int64_t t = tprev + t_rel_of(j, thd, ad, dtd, dt);
                if (t - l < a.refr) continue;  // model.py:148-149
                l = t;
                ++kc;
              }
              lt[k] = l;
            } else {
              kc = n;
              lt[k] = tprev + t_rel_of(n, thd, ad, dtd, dt);
            }
            kept[k] = kc;
            const double step = (double)n * thd;  // exact in f64
            r[k] = (float)(pos ? ls + step : ls - step);  // model.py:159-162
            dirty[k] = true;
            tot += kc;
          }
        }
      }
    }

    // ---- chunk reservations (warp ballot; 8 lanes = one 32-pixel chunk) ----
    {
      uint32_t m = __ballot_sync(0xffffffffu, tot > 0);
      if (lane == 0) {
        int c = ((m & 0xffu) != 0) + ((m & 0xff00u) != 0) + ((m & 0xff0000u) != 0) + ((m & 0xff000000u) != 0);
        if (c) atomicAdd(&s_res, c);
      }
    }

    // ---- block scan + decoupled lookback ----
    int64_t tile_total;
    const int64_t excl = block_excl_scan<NT, int64_t>((int64_t)tot, s_scan, &tile_total);
    if (tid < 32) {
      uint64_t* st = a.status + (int64_t)seg * a.ntiles;
      uint64_t ex = 0;
      if (tile == 0) {
        if (lane == 0) st_relaxed(st, pack_status(kFlagInc, epoch, (uint64_t)tile_total));
      } else {
        if (lane == 0) st_relaxed(st + tile, pack_status(kFlagAgg, epoch, (uint64_t)tile_total));
        ex = warp_lookback(st, tile, epoch);
        if (lane == 0) st_relaxed(st + tile, pack_status(kFlagInc, epoch, ex + (uint64_t)tile_total));
      }
      if (lane == 0) {
        s_base = (int64_t)ex;
        if (tile == a.ntiles - 1) a.seg_total[seg] = (int64_t)ex + tile_total;
        if (tile == 0) a.seg_tbase[seg] = tprev;
      }
    }
    __syncthreads();
    const int64_t base = s_base;
    int64_t nstore = a.cap - base;
    nstore = nstore < 0 ? 0 : (nstore > tile_total ? tile_total : nstore);
    const bool staged = nstore <= kGenStage;
    const int64_t segoff = (int64_t)seg * a.seg_stride;

    // ---- emission (pixel-major, chronological within a pixel) ----
    int64_t o = excl;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if (kept[k] > 0 && o < nstore) {
        const int64_t pix = pix0 + k;
        const uint64_t xy = ((uint64_t)(pix / a.W) << 17) | ((uint64_t)(pix % a.W) << 1) | (thv[k] > 0.f ? 1u : 0u);
        const double thd = (double)fabsf(thv[k]);
        int64_t l = last0[k];
        for (int j = 1; j <= nn[k] && o < nstore; ++j) {
          const int64_t tr = t_rel_of(j, thd, adiff[k], dtd, dt);
          if (REFR) {
            if (tprev + tr - l < a.refr) continue;
            l = tprev + tr;
          }
          const uint64_t key = ((uint64_t)tr << kKeyPixBits) | xy;
          if (staged) stg[o] = key;
          else put_event<MODE>(a, segoff, base + o, key, tprev);
          if (NB) atomicAdd(&hs[(uint32_t)tr & (uint32_t)(NB - 1)], 1u);
          ++o;
        }
      }
    }
    __syncthreads();
    if (staged) {
      for (int64_t i = tid; i < nstore; i += NT) put_event<MODE>(a, segoff, base + i, stg[i], tprev);
    }
    if (NB) {
      uint32_t* hg = a.hist + (((int64_t)seg * a.npass + 0) * kHistReps + (tile % kHistReps)) * NB;
      for (int d = tid; d < NB; d += NT) {
        uint32_t c = hs[d];
        if (c) { atomicAdd(hg + d, c); hs[d] = 0; }
      }
    }
    if (tid == 0 && s_res) { atomicAdd(reinterpret_cast<unsigned long long*>(a.seg_res + seg), (unsigned long long)s_res); s_res = 0; }
    __syncthreads();
  }

  // ---- state write-back (only pixels that crossed a threshold) ----
  if (full && dirty[0] && dirty[1] && dirty[2] && dirty[3]) {
    *reinterpret_cast<float4*>(refp + pix0) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<longlong2*>(lastp + pix0) = make_longlong2(lt[0], lt[1]);
    *reinterpret_cast<longlong2*>(lastp + pix0 + 2) = make_longlong2(lt[2], lt[3]);
  } else {
#pragma unroll
    for (int k = 0; k < VPT; ++k)
      if (dirty[k]) { refp[pix0 + k] = r[k]; lastp[pix0 + k] = lt[k]; }
  }
}

// Raise a kernel's dynamic-smem limit once per process (not per launch).
template <typename K>
static void ensure_smem(K k, size_t smem) {
  static const void* done[64];
  static int ndone = 0;
  if (smem <= 48 * 1024) return;
  const void* key = reinterpret_cast<const void*>(k);
  for (int i = 0; i < ndone; ++i)
    if (done[i] == key) return;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (ndone < 64) done[ndone++] = key;
}

template <bool VEC, bool REFR, bool UNI>
static cudaError_t gen_dispatch_mode(const GenArgs& a, unsigned grid, size_t smem, cudaStream_t st) {
  if (a.mode == 0) {
    auto k = k_generate<VEC, REFR, UNI, 0>;
    ensure_smem(k, smem);
    k<<<grid, kGenThreads, smem, st>>>(a);
  } else {
    auto k = k_generate<VEC, REFR, UNI, 1>;
    ensure_smem(k, smem);
    k<<<grid, kGenThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_generate(const GenArgs& a, int uniform_th, cudaStream_t st) {
  const unsigned grid = (unsigned)((int64_t)a.S * a.ntiles);
  const int NB = a.hist ? (1 << a.hist_bits) : 0;
  const size_t smem = (size_t)kGenStage * 8 + (size_t)NB * 4;
  bool vec = (a.P % 4 == 0) && ((uintptr_t)a.frames % 16 == 0) && ((uintptr_t)a.ref % 16 == 0) &&
             ((uintptr_t)a.last % 16 == 0) && (uniform_th || (((uintptr_t)a.thp % 16 == 0) && ((uintptr_t)a.thn % 16 == 0)));
  bool refr = a.refr > 0;
  if (vec) {
    if (refr) return uniform_th ? gen_dispatch_mode<true, true, true>(a, grid, smem, st) : gen_dispatch_mode<true, true, false>(a, grid, smem, st);
    return uniform_th ? gen_dispatch_mode<true, false, true>(a, grid, smem, st) : gen_dispatch_mode<true, false, false>(a, grid, smem, st);
  }
  if (refr) return uniform_th ? gen_dispatch_mode<false, true, true>(a, grid, smem, st) : gen_dispatch_mode<false, true, false>(a, grid, smem, st);
  return uniform_th ? gen_dispatch_mode<false, false, true>(a, grid, smem, st) : gen_dispatch_mode<false, false, false>(a, grid, smem, st);
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
              if (fl == 0) { pending = true; continue; }
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
