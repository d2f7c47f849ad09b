// K1 -- fused event generation for sm_100a (the reference's lane math,
// model.py:79-171 == parallel.py:126-273, for S streams x T frames).
//
// Per pixel (thread-owned, state held in registers across the T frames):
//   * f32 prefilter certifies "no crossing" (n == 0) without any FP64 work;
//   * f64 log via a 128-entry table + compensated degree-8 log1p (<= 1 ulp,
//     model.py:39), f64 diff against the f32 reference level;
//   * crossing count n = floor(|diff|/th + 1e-4) and event times
//     floor(((j*th)/|diff|)*dt) via reciprocals, falling back to the exact
//     IEEE division whenever the floor could differ (model.py:137, :144);
//   * refractory filter against last_event_t (model.py:148-150);
//   * state update ref = f32(ref + pol*n*th), last_event_t (model.py:159-163).
// Per tile: warp ballot per 32-pixel chunk (AggregationStats.reservation_count),
// block scan of the per-lane counts, decoupled lookback (wide windows) for the
// tile's pixel-major base, capacity cut at the first `cap` events
// (model.py:150-158), smem-staged coalesced writes, and a per-tile-group
// t_rel histogram row for the ordering pass (order.cu).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"
#include "log_table.h"

namespace evs {

struct LogTab {
  double c[128], invc[128], lh[128], ll[128];
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// log(x) for x > 0, <= 1 ulp (tools/gen_log_table.py documents the table).
__device__ __forceinline__ double fast_log(double x, const LogTab& T) {
  const uint64_t ix = (uint64_t)__double_as_longlong(x);
  if (ix < 0x0010000000000000ull || ix >= 0x7ff0000000000000ull) return log(x);  // subnormal / inf / nan
  const uint64_t tmp = ix - kLogOff;
  const int i = (int)((tmp >> (52 - kLogTableBits)) & ((1u << kLogTableBits) - 1));
  const int k = (int)((int64_t)tmp >> 52);
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
  const double c = T.c[i], invc = T.invc[i];
  const double d = z - c;  // exact (Sterbenz)
  const double rh = d * invc;
  const double rl = fma(-rh, c, d) * invc;  // r = rh + rl = (z - c) / c
  double q = -0.125;
  q = fma(q, rh, 1.0 / 7.0);
  q = fma(q, rh, -1.0 / 6.0);
  q = fma(q, rh, 0.2);
  q = fma(q, rh, -0.25);
  q = fma(q, rh, 1.0 / 3.0);
  q = fma(q, rh, -0.5);
  const double kd = (double)k;
  double s1, e1, s2, e2;
  two_sum(kd * kLn2Hi, T.lh[i], s1, e1);
  two_sum(s1, rh, s2, e2);
  double lo = e1 + e2 + (kd * kLn2Lo + T.ll[i]) + rl;
  lo = fma(rh * rh, q, lo);
  return s2 + lo;
}

// Newton-refined reciprocal (~1 ulp); only used where results are checked.
__device__ __forceinline__ double rcp_nr(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  return y;
}

// floor(v) of a value whose approximation `va` is within ~8 ulp; returns -1
// when an integer lies within the error band (caller then computes exactly).
__device__ __forceinline__ int64_t safe_floor(double va) {
  const double fl = floor(va);
  const double tol = va * 4e-15 + 1e-290;
  if (va - fl < tol || fl + 1.0 - va < tol) return -1;
  return (int64_t)fl;
}

__device__ __forceinline__ int64_t t_rel_exact(int j, double thd, double adiff, double dtd, int64_t dt) {
  // model.py:144-146: int(((j*th)/|diff|)*dt), clamped to dt-1 (IEEE division)
  int64_t tr = (int64_t)((((double)j * thd) / adiff) * dtd);
  return tr > dt - 1 ? dt - 1 : tr;
}

__device__ __forceinline__ int64_t t_rel_fast(int j, double thd, double adiff, double ra, double dtd, int64_t dt) {
  const int64_t f = safe_floor(((double)j * thd) * ra * dtd);
  if (f < 0) return t_rel_exact(j, thd, adiff, dtd, dt);
  return f > dt - 1 ? dt - 1 : f;
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

// Per-step constants of the lane math.
struct LaneCtx {
  double log_eps, rth_pos, rth_neg, dtd;
  int64_t tprev, dt, refr;
  float log_eps_f;
};

// One pixel of one frame (model.py:124-163).  Calls sink(key) for every
// refractory-surviving event in emission order (chronological), returns the
// number of such events, and produces the new (ref, last) in r_new / lt_new.
template <bool REFR, bool UNI, typename Sink>
__device__ __forceinline__ int lane_pixel(float v, float r, int64_t lt, float thp, float thn, uint64_t xy,
                                          const LaneCtx& c, const LogTab& T, float& r_new, int64_t& lt_new,
                                          Sink&& sink) {
  r_new = r;
  lt_new = lt;
  {
    // f32 prefilter: |__logf - ln| <= 2^-21 |ln| + 2^-22 and the f32 rounding of
    // v + eps are far inside the margin, so a pixel is skipped only when
    // |diff| < th (1 - 1e-4) surely holds (then n == 0: no event, no change).
    const float lf = __logf(v + c.log_eps_f);
    const float d32 = lf - r;
    const float th32 = d32 > 0.f ? thp : thn;
    if (fabsf(d32) + (2e-6f * fabsf(lf) + 2e-6f) < th32 * (1.0f - 1e-4f)) return 0;
  }
  const double ln = fast_log((double)v + c.log_eps, T);  // model.py:39 (f64)
  const double ls = (double)r;
  const double diff = ln - ls;
  if (diff == 0.0) return 0;
  const bool pos = diff > 0.0;
  const float th = pos ? thp : thn;
  const double thd = (double)th;
  const double ad = pos ? diff : -diff;
  // n = int(|diff|/th + 1e-4) (model.py:137)
  const double rth = UNI ? (pos ? c.rth_pos : c.rth_neg) : rcp_nr(thd);
  int64_t n64 = safe_floor(fma(ad, rth, 1e-4));
  if (n64 < 0) n64 = (int64_t)(ad / thd + 1e-4);
  if (n64 <= 0) return 0;
  const int n = n64 > 2147483647 ? 2147483647 : (int)n64;
  // t_rel(j) = int(((j*th)/|diff|)*dt) (model.py:144): j * u, exact fallback
  // whenever the floor of the approximation could differ from the reference's
  const double u = thd * rcp_nr(ad) * c.dtd;
  const uint64_t xyp = xy | (pos ? 1u : 0u);
  int kept = 0;
  int64_t l = lt;
  for (int j = 1; j <= n; ++j) {
    int64_t tr = safe_floor((double)j * u);
    if (tr < 0) tr = (int64_t)((((double)j * thd) / ad) * c.dtd);
    if (tr > c.dt - 1) tr = c.dt - 1;  // model.py:145-146
    if (REFR) {
      if (c.tprev + tr - l < c.refr) continue;  // model.py:148-149
    }
    l = c.tprev + tr;
    sink(((uint64_t)tr << kKeyPixBits) | xyp, kept);
    ++kept;
  }
  lt_new = l;
  const double step = (double)n * thd;          // exact in f64
  r_new = (float)(pos ? ls + step : ls - step);  // model.py:159-162
  return kept;
}

constexpr int kSlots = 16;  // per-lane event slots in smem (4 events per pixel)

template <bool VEC, bool REFR, bool UNI, int MODE>
__global__ void __launch_bounds__(kGenThreads, 3) k_generate(GenArgs a) {
  constexpr int NT = kGenThreads, VPT = kGenVpt, TILE = kGenTile, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* slots = reinterpret_cast<uint64_t*>(smem_raw);  // [kSlots][NT] (slot-major: no bank conflicts)
  uint64_t* stg = slots + kSlots * NT;                       // [kGenStage] compacted tile events
  __shared__ LogTab s_log;
  __shared__ int64_t s_scan[NW + 1];
  __shared__ int64_t s_base;
  __shared__ int s_res;

  const int tid = threadIdx.x, lane = tid & 31;
  // static tile order: blocks are dispatched in index order, so a tile's
  // lookback predecessors are always resident or finished
  const int s = (int)(blockIdx.x / (uint32_t)a.ntiles);
  const int tile = (int)(blockIdx.x % (uint32_t)a.ntiles);
  const int64_t P = a.P;
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
  const uint32_t epoch = a.desc ? a.desc->cur_epoch : a.epoch;
  const int64_t clock_t0 = a.desc ? a.desc->cur_t0 : a.t0;
  if (tid < 128) {
    s_log.c[tid] = kLogTable[tid][0];
    s_log.invc[tid] = kLogTable[tid][1];
    s_log.lh[tid] = kLogTable[tid][2];
    s_log.ll[tid] = kLogTable[tid][3];
  }
  if (tid == 0) s_res = 0;
  // key bits of the VPT pixels (y << 17 | x << 1), 32-bit coordinate math
  uint64_t xyk[VPT];
  {
    const uint32_t W = (uint32_t)a.W;
    uint32_t y = (uint32_t)pix0 / W;
    uint32_t x = (uint32_t)pix0 - y * W;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      xyk[k] = ((uint64_t)y << 17) | ((uint64_t)x << 1);
      if (++x == W) { x = 0; ++y; }
    }
  }
  const int NB = a.rows ? (1 << a.hist_bits) : 0;
  uint32_t* hrow = NB ? a.rows + ((int64_t)s * a.T * a.ngroups + tile / kGroupTiles) * NB : nullptr;
  __syncthreads();

  LaneCtx c;
  c.log_eps = a.log_eps; c.log_eps_f = a.log_eps_f; c.rth_pos = a.rth_pos; c.rth_neg = a.rth_neg;
  c.refr = a.refr;

  for (int f = 0; f < a.T; ++f) {
    const int seg = s * a.T + f;
    int64_t tnow;
    if (a.t_bounds) {
      c.tprev = a.t_bounds[(int64_t)s * (a.T + 1) + f];
      tnow = a.t_bounds[(int64_t)s * (a.T + 1) + f + 1];
    } else {
      c.tprev = clock_t0 + (int64_t)f * a.tick;
      tnow = c.tprev + a.tick;
    }
    c.dt = tnow - c.tprev;
    c.dtd = (double)c.dt;
    const float* fr = a.frames + ((int64_t)s * a.T + f) * P;
    float v[VPT];
    if (full) {
      float4 q = __ldcs(reinterpret_cast<const float4*>(fr + pix0));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < VPT; ++k) v[k] = (pix0 + k < P) ? __ldcs(fr + pix0 + k) : 0.f;
    }

    // ---- single pass: lane math, events straight into this lane's smem slots ----
    float rn[VPT];
    int64_t ltn[VPT];
    int tot = 0;  // events of this lane (sink calls)
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      rn[k] = r[k]; ltn[k] = lt[k];
      if (pix0 + k < P) {
        lane_pixel<REFR, UNI>(v[k], r[k], lt[k], thp[k], thn[k], xyk[k], c, s_log, rn[k], ltn[k],
                              [&](uint64_t key, int) {
                                if (tot < kSlots) slots[tot * NT + tid] = key;
                                ++tot;
                              });
      }
    }
    const bool overflow = __syncthreads_or(tot > kSlots) != 0;

    // ---- chunk reservations (warp ballot; 8 lanes = one 32-pixel chunk) ----
    {
      const uint32_t m = __ballot_sync(0xffffffffu, tot > 0);
      if (lane == 0) {
        const int cc = ((m & 0xffu) != 0) + ((m & 0xff00u) != 0) + ((m & 0xff0000u) != 0) + ((m & 0xff000000u) != 0);
        if (cc) atomicAdd(&s_res, cc);
      }
    }

    // ---- block scan, publish aggregate, compact slots -> stg, lookback ----
    int64_t tile_total;
    const int64_t excl = block_excl_scan<NT, int64_t>((int64_t)tot, s_scan, &tile_total);
    uint64_t* st = a.status + (int64_t)seg * a.ntiles;
    if (tid == 0) st_relaxed(st + tile, pack_status(tile == 0 ? kFlagInc : kFlagAgg, epoch, (uint64_t)tile_total));
    const bool compact = !overflow && tile_total <= kGenStage;
    if (compact)
      for (int e = 0; e < tot; ++e) stg[excl + e] = slots[e * NT + tid];
    if (tid < 32) {
      uint64_t ex = 0;
      if (tile > 0) {
        ex = warp_lookback(st, tile, epoch);
        if (lane == 0) st_relaxed(st + tile, pack_status(kFlagInc, epoch, ex + (uint64_t)tile_total));
      }
      if (lane == 0) {
        s_base = (int64_t)ex;
        if (tile == a.ntiles - 1) a.seg_total[seg] = (int64_t)ex + tile_total;
        if (tile == 0) a.seg_tbase[seg] = c.tprev;
        if (a.group_base && tile % kGroupTiles == 0)
          a.group_base[(int64_t)seg * a.ngroups + tile / kGroupTiles] = (int64_t)ex < a.cap ? (int64_t)ex : a.cap;
        if (s_res) {
          atomicAdd(reinterpret_cast<unsigned long long*>(a.seg_res + seg), (unsigned long long)s_res);
          s_res = 0;
        }
      }
    }
    __syncthreads();
    const int64_t base = s_base;
    int64_t nstore = a.cap - base;
    nstore = nstore < 0 ? 0 : (nstore > tile_total ? tile_total : nstore);
    const int64_t segoff = (int64_t)seg * a.seg_stride;
    uint32_t* hr = NB ? hrow + (int64_t)f * a.ngroups * NB : nullptr;
    auto store = [&](int64_t i, uint64_t key) {  // i: tile-local event index
      put_event<MODE>(a, segoff, base + i, key, c.tprev);
      if (NB) atomicAdd(hr + ((uint32_t)(key >> kKeyPixBits) & (uint32_t)(NB - 1)), 1u);
    };
    if (compact) {
      for (int64_t i = tid; i < nstore; i += NT) store(i, stg[i]);
    } else if (!overflow) {
      for (int e = 0; e < tot && excl + e < nstore; ++e) store(excl + e, slots[e * NT + tid]);
    } else {
      // a lane produced more than kSlots events: recompute from the unchanged
      // state and write straight to the global positions
      int64_t o = excl;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if (pix0 + k < P) {
          float r2;
          int64_t l2;
          lane_pixel<REFR, UNI>(v[k], r[k], lt[k], thp[k], thn[k], xyk[k], c, s_log, r2, l2,
                                [&](uint64_t key, int) {
                                  if (o < nstore) store(o, key);
                                  ++o;
                                });
        }
      }
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      dirty[k] |= (rn[k] != r[k]) || (ltn[k] != lt[k]);
      r[k] = rn[k];
      lt[k] = ltn[k];
    }
    __syncthreads();  // slots / stg / s_base reused by the next frame
  }

  // ---- state write-back (only pixels whose state changed) ----
  if (*a.bad != kNoBad) return;  // validation failed: state is not touched
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

// self-test: the fast log and CUDA's log side by side (tests/test_gpu_fastlog.py)
__global__ void k_selftest_log(const double* x, double* out_fast, double* out_ref, int64_t n) {
  __shared__ LogTab s_log;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    s_log.c[i] = kLogTable[i][0];
    s_log.invc[i] = kLogTable[i][1];
    s_log.lh[i] = kLogTable[i][2];
    s_log.ll[i] = kLogTable[i][3];
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    out_fast[i] = fast_log(x[i], s_log);
    out_ref[i] = log(x[i]);
  }
}

cudaError_t launch_selftest_log(const double* x, double* out_fast, double* out_ref, int64_t n, cudaStream_t st) {
  k_selftest_log<<<1024, 256, 0, st>>>(x, out_fast, out_ref, n);
  return cudaGetLastError();
}

template <typename K>
static void ensure_smem_gen(K k) {
  static const void* done[32];
  static int ndone = 0;
  const void* key = reinterpret_cast<const void*>(k);
  for (int i = 0; i < ndone; ++i)
    if (done[i] == key) return;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (ndone < 32) done[ndone++] = key;
}

template <bool VEC, bool REFR, bool UNI>
static cudaError_t gen_dispatch_mode(const GenArgs& a, unsigned grid, size_t smem, cudaStream_t st) {
  if (a.mode == 0) {
    auto k = k_generate<VEC, REFR, UNI, 0>;
    ensure_smem_gen(k);
    k<<<grid, kGenThreads, smem, st>>>(a);
  } else {
    auto k = k_generate<VEC, REFR, UNI, 1>;
    ensure_smem_gen(k);
    k<<<grid, kGenThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_generate(const GenArgs& a0, int uniform_th, cudaStream_t st) {
  GenArgs a = a0;
  a.rth_pos = 1.0 / (double)a.thp_u;  // IEEE reciprocals of the uniform thresholds
  a.rth_neg = 1.0 / (double)a.thn_u;
  const unsigned grid = (unsigned)((int64_t)a.S * a.ntiles);
  const int NB = a.rows ? (1 << a.hist_bits) : 0;
  (void)NB;
  const size_t smem = (size_t)kSlots * kGenThreads * 8 + (size_t)kGenStage * 8;
  const bool vec = (a.P % 4 == 0) && ((uintptr_t)a.frames % 16 == 0) && ((uintptr_t)a.ref % 16 == 0) &&
                   ((uintptr_t)a.last % 16 == 0) &&
                   (uniform_th || (((uintptr_t)a.thp % 16 == 0) && ((uintptr_t)a.thn % 16 == 0)));
  const bool refr = a.refr > 0;
  if (vec) {
    if (refr) return uniform_th ? gen_dispatch_mode<true, true, true>(a, grid, smem, st)
                                : gen_dispatch_mode<true, true, false>(a, grid, smem, st);
    return uniform_th ? gen_dispatch_mode<true, false, true>(a, grid, smem, st)
                      : gen_dispatch_mode<true, false, false>(a, grid, smem, st);
  }
  if (refr) return uniform_th ? gen_dispatch_mode<false, true, true>(a, grid, smem, st)
                              : gen_dispatch_mode<false, true, false>(a, grid, smem, st);
  return uniform_th ? gen_dispatch_mode<false, false, true>(a, grid, smem, st)
                    : gen_dispatch_mode<false, false, false>(a, grid, smem, st);
}

}  // namespace evs
