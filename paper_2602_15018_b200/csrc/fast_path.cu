// Fast canonical-order path of evs_step for sm_100a (t_now - t_prev <= 2048 us,
// the reference's render-rate regime: ticks of 1000 us in every BASELINE config).
//
//   k_fast_gen   (K1) one CTA per tile of G <= 2048 consecutive pixels of one
//                stream, all T frames of the call with the state in registers.
//                Per frame: certified f32 lane math (exact FP64 fallback),
//                block-scan compaction of the crossings into a pixel-major
//                smem list, stable bucket sort of the list in smem (warp
//                match-any ranks, buckets of 8 t_rel bins), coalesced write of
//                the sorted 4-byte keys to the tile's slot and of the tile's
//                bucket starts into a [bucket][tile] table.
//   k_fast_fix   per segment: counts / dropped (parallel.py:261-273), sorting of
//                tiles whose crossings overflowed the smem list, and the
//                capacity cut (first `cap` events in pixel-major order are kept,
//                model.py:150-158).  Exits at once in the common case.
//   k_fast_order (K2) one CTA per (segment, bucket): gathers the bucket's slice
//                of every tile (tile order = pixel order), stable counting sort
//                by t_rel within the bucket, and writes its contiguous range of
//                the canonical (t, y, x, p) output with coalesced stores.
//
// Lane math (model.py:124-163 / parallel.py:152-217).  The reference computes
// ln in f64, the crossing count floor(|d|/th + 1e-4) and the times
// floor(((j*th)/|d|)*dt) in f64.  Every observable (n, t_rel, the refractory
// filter, the new level f32(ls +- n*th)) depends on |d| only through those
// floors, so K1 evaluates them in f32 from a "lite" log (table + f32 log1p,
// |error| < 4e-9) and certifies each floor with an error band; a pixel whose
// band straddles an integer (about 1e-3 of the events) is recomputed with the
// exact path (<= 1 ulp f64 log and IEEE division, the formulas of the
// reference).  The new level is always computed in f64 from the certified n.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/evsim_b200.h"
#include "common.cuh"
#include "fast_path.cuh"
#include "log_table.h"
#include "lane_lite.cuh"

namespace evs {

// ---------------------------------------------------------------------------
// exact lane math (rare path): the reference's formulas with a <= 1 ulp log
// ---------------------------------------------------------------------------
__device__ __forceinline__ void two_sum_x(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// log(x), <= 1 ulp from CUDA's log (tests/test_gpu_fastlog.py checks the same
// construction); table read through L1 from global memory (rare path only).
__device__ __noinline__ double fast_log_g(double x) {
  const uint64_t ix = (uint64_t)__double_as_longlong(x);
  if (ix < 0x0010000000000000ull || ix >= 0x7ff0000000000000ull) return log(x);
  const uint64_t tmp = ix - kLogOff;
  const int i = (int)((tmp >> (52 - kLogTableBits)) & ((1u << kLogTableBits) - 1));
  const int k = (int)((int64_t)tmp >> 52);
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
  const double c = kLogTable[i][0], invc = kLogTable[i][1];
  const double d = z - c;
  const double rh = d * invc;
  const double rl = fma(-rh, c, d) * invc;
  double q = -0.125;
  q = fma(q, rh, 1.0 / 7.0);
  q = fma(q, rh, -1.0 / 6.0);
  q = fma(q, rh, 0.2);
  q = fma(q, rh, -0.25);
  q = fma(q, rh, 1.0 / 3.0);
  q = fma(q, rh, -0.5);
  const double kd = (double)k;
  double s1, e1, s2, e2;
  two_sum_x(kd * kLn2Hi, kLogTable[i][2], s1, e1);
  two_sum_x(s1, rh, s2, e2);
  double lo = e1 + e2 + (kd * kLn2Lo + kLogTable[i][3]) + rl;
  lo = fma(rh * rh, q, lo);
  return s2 + lo;
}

// n and the direction of one pixel with the reference's f64 formulas
// (model.py:125-137); returns n (0: no crossing) and |diff|, th.
__device__ __noinline__ int exact_count(float v, float r, float thp, float thn, double log_eps, bool& pos,
                                        double& ad, double& thd) {
  if (!(v >= 0.f && v <= 1.f)) return 0;  // invalid intensity: the call is rejected by validation
  const double ln = fast_log_g((double)v + log_eps);  // model.py:39
  const double diff = ln - (double)r;
  pos = diff > 0.0;
  if (!(diff != 0.0) || diff != diff) return 0;
  thd = (double)(pos ? thp : thn);
  ad = pos ? diff : -diff;
  const double q = __dadd_rn(__ddiv_rn(ad, thd), 1e-4);  // int(|diff|/th + 1e-4)
  if (!(q >= 1.0)) return 0;
  return q > (double)kMaxPixelCrossings ? 0 : (int)q;  // (beyond: corrupt level, no 32-bit overflow)
}
// t_rel of crossing j (model.py:144-146)
__device__ __forceinline__ int exact_trel(int j, double thd, double ad, double dtd, int dtm1) {
  const double a = __dmul_rn(__ddiv_rn(__dmul_rn((double)j, thd), ad), dtd);
  const int tr = a >= (double)dtm1 ? dtm1 : (int)a;
  return tr;
}

// ---------------------------------------------------------------------------
// certified f32 lane math
// ---------------------------------------------------------------------------
// |df - diff_ref| <= kEpsD + 3*2^-24*|df| (see the header comment of
// fast_path.cuh); diff_ref is the reference's f64 ln(v + eps) - ref.
// (kEpsD = 8e-9 enters the bands below as the 1e-8 terms.)

// All roundings below are explicit (_rn intrinsics / fmaf) so that no FMA
// contraction can differ between the passes that evaluate the same pixel
// (K1's count pass, its emission pass, and k_fast_redo): the decisions must
// be bit-identical wherever they are recomputed.
//
// Returns n (>= 0) or -1 when the exact path must decide.
__device__ __forceinline__ int lite_count(float v, float r, float thp, float thn, float rthp, float rthn,
                                          double log_eps, float dtf, const LiteTab& T, bool& pos, LiteOut& o) {
  const double x = __dadd_rn((double)v, log_eps);  // the reference's x exactly
  const uint64_t ix = (uint64_t)__double_as_longlong(x);
  if (ix < 0x0010000000000000ull || ix >= 0x7ff0000000000000ull) return -1;
  const uint64_t tmp = ix - kLogOff;
  const int i = (int)((tmp >> (52 - kLogTableBits)) & ((1u << kLogTableBits) - 1));
  const int k = (int)((int64_t)tmp >> 52);
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
  const double d = __dsub_rn(z, T.c[i]);                               // exact
  const float rf = __double2float_rn(__dmul_rn(d, T.invc[i]));          // |r| <= 2^-7
  float pf = fmaf(rf, 0.2f, -0.25f);
  pf = fmaf(pf, rf, 0.33333334f);
  pf = fmaf(pf, rf, -0.5f);
  pf = fmaf(pf, rf, 1.0f);
  pf = __fmul_rn(pf, rf);                                               // log1p(r), |err| < 2^-30
  const double dd = __dsub_rn(fma((double)k, 0.6931471805599453, T.lh[i]), (double)r);
  const float df = __fadd_rn(__double2float_rn(dd), pf);
  pos = df > 0.f;
  const float ad = fabsf(df);
  const float th = pos ? thp : thn;
  const float rth = pos ? rthp : rthn;
  const float q1 = fmaf(ad, rth, 1e-4f);  // |diff|/th + 1e-4 (model.py:137)
  const float dn = fmaf(q1, 6e-7f, fmaf(1e-8f, rth, 1e-10f));
  const float nlo = floorf(__fsub_rn(q1, dn)), nhi = floorf(__fadd_rn(q1, dn));
  if (nlo != nhi || q1 > 1e6f) return -1;
  const int n = (int)nlo;
  if (n <= 0) return 0;
  const float ra = rcp_approx(ad);
  o.uf = __fmul_rn(__fmul_rn(th, dtf), ra);
  o.erel = fmaf(1e-8f, ra, 1e-6f);
  return n;
}

// certified floor of j*uf clamped to dt-1; -1 if the band straddles
__device__ __forceinline__ int lite_trel(int j, const LiteOut& o, int dtm1) {
  const float a = __fmul_rn((float)j, o.uf);
  const float band = fmaf(a, o.erel, 1e-6f);
  const int lo = min((int)floorf(__fsub_rn(a, band)), dtm1);
  const int hi = min((int)floorf(__fadd_rn(a, band)), dtm1);
  return lo == hi ? lo : -1;
}

// One pixel, one frame (model.py:124-163): n (level steps), kept crossings
// after the refractory filter, and the last kept time.
struct PxStep {
  int n, kept, lnew;
  bool pos, exact;
  LiteOut lo;
};

// Exact path of one pixel-frame (rare; kept out of line so the hot loop stays small).
template <bool REFR>
__device__ __forceinline__ void exact_step(float v, float r, int lrel, float thp, float thn, const FrameCtx& c,
                                        PxStep& o) {
  double ad = 0.0, thd = 0.0;
  const int n = exact_count(v, r, thp, thn, c.log_eps, o.pos, ad, thd);
  int kept = 0, l = lrel;
  for (int j = 1; j <= n; ++j) {
    const int tr = exact_trel(j, thd, ad, c.dtd, c.dtm1);
    if (REFR && c.tpr + tr - l < c.refr) continue;
    l = c.tpr + tr;
    ++kept;
  }
  o.n = n > 0 ? n : 0;
  o.kept = kept;
  o.lnew = l;
  o.exact = true;
}

// Exact-path crossings of one pixel appended to a key list (rare path).
template <bool REFR>
__device__ __forceinline__ int exact_emit(float v, float rold, int lold, float thp, float thn, const FrameCtx& c,
                                       uint32_t xyp, uint32_t* list, int off) {
  double ad = 0.0, thd = 0.0;
  bool pos;
  const int n = exact_count(v, rold, thp, thn, c.log_eps, pos, ad, thd);
  int l = lold;
  for (int j = 1; j <= n; ++j) {
    const int tr = exact_trel(j, thd, ad, c.dtd, c.dtm1);
    if (REFR) {
      if (c.tpr + tr - l < c.refr) continue;
      l = c.tpr + tr;
    }
    list[off++] = ((uint32_t)tr << 12) | xyp;
  }
  return off;
}

template <bool REFR, bool PREF>
__device__ __forceinline__ void px_step(float v, float r, int lrel, float thp, float thn, float rthp, float rthn,
                                        const FrameCtx& c, const LiteTab& T, PxStep& o) {
  o.n = 0;
  o.kept = 0;
  o.lnew = lrel;
  o.exact = false;
  if (PREF) {
    // f32 prefilter: |__logf - ln| <= 2^-21 |ln| + 2^-22 and the f32 rounding of
    // v + eps are far inside the margin, so a skipped pixel surely has n == 0
    const float lf = __logf(v + c.log_eps_f);
    const float d32 = lf - r;
    const float th32 = d32 > 0.f ? thp : thn;
    if (fabsf(d32) + (2e-6f * fabsf(lf) + 2e-6f) < th32 * (1.0f - 1e-4f)) return;
  }
  int n = lite_count(v, r, thp, thn, rthp, rthn, c.log_eps, c.dtf, T, o.pos, o.lo);
  bool exact = n < 0;
  int kept = 0, l = lrel;
  if (!exact && n > 0) {
    for (int j = 1; j <= n; ++j) {
      const int tr = lite_trel(j, o.lo, c.dtm1);
      if (tr < 0) { exact = true; break; }
      if (REFR && c.tpr + tr - l < c.refr) continue;  // model.py:148-149
      l = c.tpr + tr;
      ++kept;
    }
  }
  if (exact) {
    exact_step<REFR>(v, r, lrel, thp, thn, c, o);
    return;
  }
  o.n = n > 0 ? n : 0;
  o.kept = kept;
  o.lnew = l;
}

// The kept crossing times of a pixel (chronological), as decided by px_step.
// The kept crossings of a lite-path pixel (chronological), as px_step decided.
template <bool REFR, typename Sink>
__device__ __forceinline__ void px_emit(int lold, int n, const LiteOut& lo, const FrameCtx& c, Sink&& sink) {
  int l = lold;
  for (int j = 1; j <= n; ++j) {
    // certified in px_step: floor(j*uf) lies inside the band, so it is the value
    const int tr = min((int)floorf(__fmul_rn((float)j, lo.uf)), c.dtm1);
    if (REFR) {
      if (c.tpr + tr - l < c.refr) continue;
      l = c.tpr + tr;
    }
    sink(tr);
  }
}

// Rare pixels (band straddles an integer, n > 2): the general path, out of
// line so that the unrolled per-pixel code stays small and spill-free.
struct SlowRes {
  int n, kept, lnew;
  bool pos;
};
template <bool REFR>
__device__ __forceinline__ SlowRes slow_step(float v, float r, int lrel, float thp, float thn, float rthp, float rthn,
                                          const FrameCtx& c, const LiteTab& T) {
  PxStep o;
  px_step<REFR, false>(v, r, lrel, thp, thn, rthp, rthn, c, T, o);
  return SlowRes{o.n, o.kept, o.lnew, o.pos};
}
template <bool REFR>
__device__ __forceinline__ void slow_emit(float v, float r, int lrel, float thp, float thn, float rthp, float rthn,
                                       const FrameCtx& c, const LiteTab& T, uint32_t xy, uint32_t* list, int off) {
  PxStep o;
  px_step<REFR, false>(v, r, lrel, thp, thn, rthp, rthn, c, T, o);
  const uint32_t xyp = xy | (o.pos ? 1u : 0u);
  if (o.exact)
    exact_emit<REFR>(v, r, lrel, thp, thn, c, xyp, list, off);
  else
    px_emit<REFR>(lrel, o.n, o.lo, c, [&](int tr) { list[off++] = ((uint32_t)tr << 12) | xyp; });
}
template <typename T>
__device__ __forceinline__ T sel4(const T (&a)[4], int k) {
  return k == 0 ? a[0] : (k == 1 ? a[1] : (k == 2 ? a[2] : a[3]));
}
template <typename T>
__device__ __forceinline__ void set4(T (&a)[4], int k, T v) {
  a[0] = k == 0 ? v : a[0]; a[1] = k == 1 ? v : a[1]; a[2] = k == 2 ? v : a[2]; a[3] = k == 3 ? v : a[3];
}

// ---------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t frame_tprev(const FastArgs& a, int s, int f, int64_t t0c) {
  return a.t_bounds ? a.t_bounds[(int64_t)s * (a.T + 1) + f] : t0c + (int64_t)f * a.tick;
}
__device__ __forceinline__ int64_t frame_tnow(const FastArgs& a, int s, int f, int64_t t0c) {
  return a.t_bounds ? a.t_bounds[(int64_t)s * (a.T + 1) + f + 1] : t0c + (int64_t)(f + 1) * a.tick;
}
__device__ __forceinline__ FrameCtx frame_ctx(const FastArgs& a, int s, int f, int64_t t0c, int64_t tb) {
  FrameCtx c;
  const int64_t tprev = frame_tprev(a, s, f, t0c);
  const int dt = (int)(frame_tnow(a, s, f, t0c) - tprev);
  c.log_eps = a.log_eps;
  c.log_eps_f = a.log_eps_f;
  c.dtd = (double)dt;
  c.dtf = (float)dt;
  c.dtm1 = dt - 1;
  c.tpr = (int)(tprev - tb);
  c.refr = a.refr;
  return c;
}
__device__ __forceinline__ int clamp_rel(int64_t d) {
  return d < -(1ll << 30) ? -(1 << 30) : (d > (1ll << 30) ? (1 << 30) : (int)d);
}

// K1.  Thread t of a tile owns pixels t + k*NT (k < VPT): for each k a warp
// handles 32 consecutive pixels (one 32-pixel chunk of the reference), so a
// tile's pixel order is (k, warp, lane) and its crossings form NG = VPT*NW
// "groups" (k, warp) whose lists concatenate in pixel order.  The per-pixel
// loop is rolled (small hot code: the instruction cache is the limiter) and
// the state stays in registers (select chains instead of dynamic indexing).
template <bool REFR, bool UNI>
__global__ void __launch_bounds__(kFNT, kFCtasPerSm) k_fast_gen(FastArgs a) {
  constexpr int NT = kFNT, VPT = kFVpt, NW = NT / 32, NG = VPT * NW, KB = kFMaxBuckets;
  constexpr int GCAP = kFListCap / NG;  // crossings per group held in smem
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_list = reinterpret_cast<uint32_t*>(smem_raw);   // [NG][GCAP] pixel-major keys per group
  uint32_t* s_sorted = s_list + kFListCap;                      // [kFListCap] bucket-sorted keys of the tile
  uint16_t* s_gc = reinterpret_cast<uint16_t*>(s_sorted + kFListCap);  // [NG][KB] per-group bucket counters
  __shared__ LiteTab s_tab;
  __shared__ uint32_t s_bstart[KB + 1];
  __shared__ int s_gn[NG];         // crossings per group (this frame)
  __shared__ uint32_t s_res2[2];   // reservation chunks, per frame parity
  __shared__ int s_ovf2[2];        // a group list overflowed, per frame parity
  __shared__ int s_scan[NW + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = blockIdx.x / a.ntiles;
  const int tile = blockIdx.x % a.ntiles;
  const int64_t P = a.P;
  const int64_t tile0 = (int64_t)tile * a.G;
  const int gt = (int)min((int64_t)a.G, P - tile0);  // pixels of this tile
  float* refp = a.ref + (int64_t)s * P + tile0;
  int64_t* lastp = a.last + (int64_t)s * P + tile0;
  const int64_t t0c = a.desc ? a.desc->cur_t0 : a.t0;
  const int64_t tb = frame_tprev(a, s, 0, t0c);  // time base of the relative times
  const int nbk = a.nbk;

  // ---- state into registers ----
  float r4[VPT], thp4[VPT], thn4[VPT], rthp4[VPT], rthn4[VPT];
  int l4[VPT];
  uint32_t dirty = 0;  // bit k: level changed, bit 4+k: last event changed
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int lp = tid + k * NT;
    r4[k] = 0.f; l4[k] = -(1 << 30);
    thp4[k] = a.thp_u; thn4[k] = a.thn_u; rthp4[k] = a.rthp_u; rthn4[k] = a.rthn_u;
    if (lp < gt) {
      r4[k] = __ldcg(refp + lp);
      if (REFR) l4[k] = clamp_rel(__ldcg(lastp + lp) - tb);
      if (!UNI) {
        thp4[k] = a.thp[(int64_t)s * P + tile0 + lp];
        thn4[k] = a.thn[(int64_t)s * P + tile0 + lp];
        rthp4[k] = __frcp_rn(thp4[k]);
        rthn4[k] = __frcp_rn(thn4[k]);
      }
    }
  }
  for (int i = tid; i < NG * KB / 2; i += NT) reinterpret_cast<uint32_t*>(s_gc)[i] = 0u;
  if (tid < 2) { s_res2[tid] = 0; s_ovf2[tid] = 0; }
  load_lite_tab(s_tab);

  auto load_frame = [&](int f, float* dst) {
    const float* fr = a.frames + ((int64_t)s * a.T + f) * P + tile0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) dst[k] = (tid + k * NT < gt) ? __ldcs(fr + tid + k * NT) : 1.0f;
  };
  float vn4[VPT];
  load_frame(0, vn4);
  __syncthreads();

  for (int f = 0; f < a.T; ++f) {
    const int seg = s * a.T + f;
    const int64_t st_idx = (int64_t)seg * a.ntiles + tile;
    const FrameCtx c = frame_ctx(a, s, f, t0c, tb);
    uint32_t& s_res = s_res2[f & 1];
    int& s_ovf = s_ovf2[f & 1];
    float v4[VPT], ro4[VPT];
    int lo4[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) { v4[k] = vn4[k]; ro4[k] = r4[k]; lo4[k] = l4[k]; }
    if (f + 1 < a.T) load_frame(f + 1, vn4);

    // ---- 1. per pixel (rolled): lane math, state, crossings into the group lists ----
    // each warp clears its own groups' bucket counters (no other warp touches
    // them before this frame's barrier A)
#pragma unroll
    for (int k = 0; k < VPT; ++k)
      for (int b = lane; b < nbk; b += 32) s_gc[(k * NW + warp) * KB + b] = 0;
    __syncwarp();
    uint32_t chg = 0;
#pragma unroll 1
    for (int k = 0; k < VPT; ++k) {
      const int lp = tid + k * NT;
      const int g = k * NW + warp;
      uint32_t* glist = s_list + g * GCAP;
      const float v = sel4(v4, k), r = sel4(r4, k), thp = sel4(thp4, k), thn = sel4(thn4, k);
      const float rthp = sel4(rthp4, k), rthn = sel4(rthn4, k);
      const int l = sel4(l4, k);
      uint32_t res = 0;
      int n = 0, kept = 0, ln = l;
      bool pos = false;
      if (lp < gt) {
        res = px_fast2<REFR>(v, r, l, thp, thn, rthp, rthn, c, s_tab, ln);
        if (res & kF2Slow) {
          const SlowRes o = slow_step<REFR>(v, r, l, thp, thn, rthp, rthn, c, s_tab);
          n = o.n; kept = o.kept; ln = o.lnew; pos = o.pos;
        } else {
          n = (int)((res >> 25) & 3u);
          kept = (int)((res >> 22) & 1u) + (int)((res >> 23) & 1u);
          pos = (res & kF2Pos) != 0;
        }
        if (n > 0) {
          // new level f32(ls +- n*th) (model.py:159-162); n*th is exact in f64
          const double step = __dmul_rn((double)n, (double)(pos ? thp : thn));
          set4(r4, k, __double2float_rn(pos ? __dadd_rn((double)r, step) : __dsub_rn((double)r, step)));
          chg |= 1u << k;
        }
        if (kept > 0) { set4(l4, k, ln); chg |= 16u << k; }
      }
      // group list: warp scan of the kept counts
      int off = warp_incl_scan(kept);
      const int gn = __shfl_sync(0xffffffffu, off, 31);
      off -= kept;
      const uint32_t anyk = __ballot_sync(0xffffffffu, kept > 0);
      if (lane == 0) {
        s_gn[g] = gn;
        if (anyk) atomicAdd(&s_res, 1u);  // one 32-pixel chunk with kept events
        if (gn > GCAP) s_ovf = 1;
      }
      if (gn <= GCAP && kept > 0) {
        const uint32_t xyp = ((uint32_t)lp << 1) | (pos ? 1u : 0u);
        if (!(res & kF2Slow)) {
          if (res & kF2K1) glist[off++] = ((res & 0x7ffu) << 12) | xyp;
          if (res & kF2K2) glist[off++] = (((res >> 11) & 0x7ffu) << 12) | xyp;
        } else {
          slow_emit<REFR>(v, r, l, thp, thn, rthp, rthn, c, s_tab, (uint32_t)lp << 1, glist, off);
        }
      }
      __syncwarp();
      if (gn <= GCAP) {  // bucket counts of the group (warp-aggregated)
        uint16_t* gc = s_gc + g * KB;
        for (int base = 0; base < gn; base += 32) {
          const int i = base + lane;
          const bool valid = i < gn;
          const uint32_t active = __ballot_sync(0xffffffffu, valid);
          if (valid) {
            const int bk = (int)(glist[i] >> 15);
            const uint32_t peers = __match_any_sync(active, bk);
            if (lane == __ffs(peers) - 1) gc[bk] = (uint16_t)(gc[bk] + __popc(peers));
          }
          __syncwarp();  // the next round's leader may update the same counter
        }
      }
    }
    dirty |= chg;
    __syncthreads();  // A
    if (s_ovf) {  // block-uniform, rare: k_fast_redo regenerates this tile-frame
      float* sr = a.snap_ref + st_idx * a.G;
      int* sl = a.snap_last + st_idx * a.G;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int lp = tid + k * NT;
        if (lp < gt) { sr[lp] = ro4[k]; sl[lp] = lo4[k]; }
      }
      for (int i = tid; i < NG * KB / 2; i += NT) reinterpret_cast<uint32_t*>(s_gc)[i] = 0u;
      if (tid == 0) {
        int total = 0;
        for (int g = 0; g < NG; ++g) total += s_gn[g];
        a.tile_src[st_idx] = kSrcRedo;
        a.rows[((int64_t)seg * (nbk + 1) + nbk) * a.ntiles + tile] = (uint32_t)total;
        if (s_res) atomicAdd(reinterpret_cast<unsigned long long*>(a.seg_res + seg), (unsigned long long)s_res);
        s_res = 0;
      }
      __syncthreads();  // everyone has read s_ovf; counters are zero again
      if (tid == 0) s_ovf = 0;  // (this parity slot is next used by frame f + 2)
      continue;
    }

    // ---- 2. bucket starts: column prefix over the groups, scan over buckets ----
    int total = 0;
    {
      uint32_t tot = 0;
      if (tid < nbk) {
        for (int g = 0; g < NG; ++g) {
          const uint32_t cc = s_gc[g * KB + tid];
          s_gc[g * KB + tid] = (uint16_t)tot;
          tot += cc;
        }
      }
      const uint32_t bst = (uint32_t)block_excl_scan<NT, int>((int)tot, s_scan, &total);
      if (tid < nbk) {
        for (int g = 0; g < NG; ++g) s_gc[g * KB + tid] = (uint16_t)(s_gc[g * KB + tid] + bst);
        s_bstart[tid] = bst;
        const uint32_t cb = tot;
        if (cb) atomicAdd(a.btot + (int64_t)seg * nbk + tid, cb);
      }
      if (tid == 0) s_bstart[nbk] = (uint32_t)total;
    }
    __syncthreads();  // B

    // ---- 3. stable rank (warp match-any over each of the warp's groups) ----
#pragma unroll 1
    for (int k = 0; k < VPT; ++k) {
      const int g = k * NW + warp;
      const uint32_t* glist = s_list + g * GCAP;
      uint16_t* gc = s_gc + g * KB;
      const int gn = s_gn[g];
      for (int base = 0; base < gn; base += 32) {
        const int i = base + lane;
        const bool valid = i < gn;
        const uint32_t active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          const uint32_t key = glist[i];
          const int bk = (int)(key >> 15);
          const uint32_t peers = __match_any_sync(active, bk);
          const int leader = __ffs(peers) - 1;
          uint32_t bpos = 0;
          if (lane == leader) {
            bpos = gc[bk];
            gc[bk] = (uint16_t)(bpos + __popc(peers));
          }
          bpos = __shfl_sync(active, bpos, leader);
          s_sorted[bpos + __popc(peers & lanemask_lt())] = key;
        }
        __syncwarp();  // the next round's leader may update the same counter
      }
    }
    __syncthreads();  // C

    // ---- 4. sorted keys and bucket starts out; reset the counters ----
    {
      uint32_t* dst = a.keys + st_idx * kFListCap;
      const int n4 = total >> 2;
      for (int i = tid; i < n4; i += NT)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(s_sorted)[i];
      for (int i = 4 * n4 + tid; i < total; i += NT) dst[i] = s_sorted[i];
      uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * a.ntiles + tile;
      for (int b = tid; b <= nbk; b += NT) rows[(int64_t)b * a.ntiles] = s_bstart[b];
      if (tid == 0) {
        a.tile_src[st_idx] = kSrcSlot;
        if (s_res) atomicAdd(reinterpret_cast<unsigned long long*>(a.seg_res + seg), (unsigned long long)s_res);
        s_res = 0;
      }
    }
  }

  // ---- state write-back (the prologue validated every frame of the call) ----
  if (*a.bad == kNoBad) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int lp = tid + k * NT;
      if (dirty & (1u << k)) refp[lp] = r4[k];
      if (dirty & (16u << k)) lastp[lp] = tb + l4[k];
    }
  }
}

// ---------------------------------------------------------------------------
// fixup (one CTA per segment): totals, counts / dropped, capacity cut, and the
// work list of tile-frames K1 could not hold (regenerated by k_fast_redo)
// ---------------------------------------------------------------------------
constexpr int kFixNT = 512;

__device__ __forceinline__ const uint32_t* tile_keys(const FastArgs& a, int seg, int q) {
  const int64_t st = (int64_t)seg * a.ntiles + q;
  const int64_t src = a.tile_src[st];
  return src < 0 ? a.keys + st * kFListCap : a.area_sorted + (int64_t)seg * a.cap + src;
}

__global__ void __launch_bounds__(kFixNT) k_fast_fix(FastArgs a) {
  constexpr int NT = kFixNT;
  __shared__ int64_t s_scan64[NT / 32 + 1];
  __shared__ int s_scan[NT / 32 + 1];
  __shared__ uint32_t s_hist[kFMaxBuckets + 1];
  __shared__ int s_qcut;
  __shared__ int64_t s_qbase;
  const int seg = blockIdx.x, tid = threadIdx.x;
  const int nbk = a.nbk, nt = a.ntiles;
  uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * nt;
  const int64_t* src = a.tile_src + (int64_t)seg * nt;
  if (*a.bad != kNoBad) {
    if (tid == 0) { a.out_count[seg] = 0; a.out_dropped[seg] = 0; a.redo_n[seg] = 0; }
    return;
  }
  const int64_t cap = a.cap;
  if (tid == 0) s_qcut = nt;
  // pixel-major base of every tile; the tile holding the cut; the redo list
  int64_t run = 0;
  int redo_run = 0;
  int64_t area_run = 0;
  for (int q0 = 0; q0 < nt; q0 += NT) {
    const int q = q0 + tid;
    const int64_t c = q < nt ? (int64_t)rows[(int64_t)nbk * nt + q] : 0;
    int64_t tt;
    const int64_t base = run + block_excl_scan<NT, int64_t>(c, s_scan64, &tt);
    run += tt;
    const bool redo = q < nt && src[q] == kSrcRedo && base < cap;
    const int64_t lim = redo ? (base + c > cap ? cap - base : c) : 0;
    if (q < nt && base < cap && base + c > cap) s_qcut = q;  // unique
    int ntt;
    const int rex = block_excl_scan<NT, int>(redo ? 1 : 0, s_scan, &ntt);
    int64_t att;
    const int64_t aex = block_excl_scan<NT, int64_t>(lim, s_scan64, &att);
    if (redo) {
      int* item = a.redo_items + ((int64_t)seg * nt + redo_run + rex) * 2;
      item[0] = q;
      item[1] = (int)(area_run + aex);
      a.redo_lim[(int64_t)seg * nt + q] = (int)lim;
    }
    redo_run += ntt;
    area_run += att;
  }
  const int64_t total = run;
  __syncthreads();
  const int qc = s_qcut;
  if (total > cap) {
    // capacity (model.py:150-158): tiles after the cut keep nothing
    for (int q = qc + 1; q < nt; ++q)
      for (int b = tid; b <= nbk; b += NT) rows[(int64_t)b * nt + q] = 0;
    if (src[qc] != kSrcRedo) {
      // cut inside a K1 tile list: keep its first `keepn` events in pixel-major
      // order = order by (pixel, t_rel); identical keys are interchangeable
      if (tid == 0) {
        int64_t r2 = 0;
        for (int q = 0; q < qc; ++q) r2 += rows[(int64_t)nbk * nt + q];
        s_qbase = r2;
      }
      __syncthreads();
      const int64_t keepn = cap - s_qbase;
      const int n = (int)rows[(int64_t)nbk * nt + qc];
      uint32_t* list = a.keys + ((int64_t)seg * nt + qc) * kFListCap;
      for (int i = tid; i < n; i += NT) {
        const uint32_t ki = list[i];
        const uint32_t pi = ((ki >> 1) & 0x7ffu) << 12 | (ki >> 12);
        int rank = 0;
        for (int j = 0; j < n; ++j) {
          const uint32_t kj = list[j] & 0x7fffffffu;
          const uint32_t pj = ((kj >> 1) & 0x7ffu) << 12 | (kj >> 12);
          rank += (pj < pi) || (pj == pi && j < i);
        }
        if (rank < keepn) list[i] = ki | 0x80000000u;
      }
      __syncthreads();
      // stable in-place compaction of the kept keys, then the tile's bucket starts
      for (int b = tid; b <= nbk; b += NT) s_hist[b] = 0;
      int kr = 0;
      for (int base = 0; base < n; base += NT) {
        const int i = base + tid;
        const uint32_t k = i < n ? list[i] : 0u;
        const int keep = (k >> 31) & 1;
        int tt;
        const int ex = block_excl_scan<NT, int>(keep, s_scan, &tt);
        if (keep) {
          list[kr + ex] = k & 0x7fffffffu;
          atomicAdd(&s_hist[(k & 0x7fffffffu) >> 15], 1u);
        }
        kr += tt;
        __syncthreads();
      }
      const int cc = tid < nbk ? (int)s_hist[tid] : 0;
      int tt;
      const int ex = block_excl_scan<NT, int>(cc, s_scan, &tt);
      if (tid < nbk) rows[(int64_t)tid * nt + qc] = (uint32_t)ex;
      if (tid == 0) rows[(int64_t)nbk * nt + qc] = (uint32_t)tt;
    }
    __syncthreads();
    for (int k = tid; k < nbk; k += NT) {
      uint32_t acc = 0;
      for (int q = 0; q < nt; ++q)
        if (src[q] != kSrcRedo) acc += rows[(int64_t)(k + 1) * nt + q] - rows[(int64_t)k * nt + q];
      a.btot[(int64_t)seg * nbk + k] = acc;
    }
  }
  if (tid == 0) {
    const int64_t written = total < cap ? total : cap;
    a.out_count[seg] = written;
    a.out_dropped[seg] = total - written;
    a.redo_n[seg] = redo_run;
  }
}

// ---------------------------------------------------------------------------
// redo: regenerate a tile-frame whose crossings overflowed K1's shared list,
// from the state snapshot K1 left, keeping at most its capacity share; stable
// bucket sort into the segment's overflow area.  Grid (kRedoCtas, nseg).
// ---------------------------------------------------------------------------
constexpr int kRedoNT = 256, kRedoCtas = 8;

template <bool REFR>
__global__ void __launch_bounds__(kRedoNT) k_fast_redo(FastArgs a) {
  constexpr int NT = kRedoNT, PPT = (kFGmax + NT - 1) / NT;
  __shared__ int s_scan[NT / 32 + 1];
  __shared__ uint32_t s_hist[kFMaxBuckets + 1];
  __shared__ LiteTab s_tab;
  const int seg = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  if (*a.bad != kNoBad) return;
  const int nitems = a.redo_n[seg];
  if (blockIdx.x >= nitems) return;
  load_lite_tab(s_tab);
  __syncthreads();
  const int s = seg / a.T, f = seg % a.T;
  const int nbk = a.nbk, nt = a.ntiles;
  const int64_t t0c = a.desc ? a.desc->cur_t0 : a.t0;
  const int64_t tb = frame_tprev(a, s, 0, t0c);
  const FrameCtx c = frame_ctx(a, s, f, t0c, tb);
  uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * nt;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int q = a.redo_items[((int64_t)seg * nt + it) * 2];
    const int aoff = a.redo_items[((int64_t)seg * nt + it) * 2 + 1];
    const int lim = a.redo_lim[(int64_t)seg * nt + q];
    const int64_t st_idx = (int64_t)seg * nt + q;
    const int64_t tile0 = (int64_t)q * a.G;
    const int gt = (int)min((int64_t)a.G, a.P - tile0);
    const float* sr = a.snap_ref + st_idx * a.G;
    const int* sl = a.snap_last + st_idx * a.G;
    const float* fr = a.frames + ((int64_t)s * a.T + f) * a.P + tile0;
    const float* tp = a.thp ? a.thp + (int64_t)s * a.P + tile0 : nullptr;
    const float* tn = a.thn ? a.thn + (int64_t)s * a.P + tile0 : nullptr;
    uint32_t* un = a.area_unsorted + (int64_t)seg * a.cap + aoff;
    uint32_t* so = a.area_sorted + (int64_t)seg * a.cap + aoff;
    // pass 1: pixel-major emission (thread owns PPT consecutive pixels)
    int cnt = 0;
    const int lp0 = tid * PPT;
    for (int k = 0; k < PPT; ++k) {
      const int lp = lp0 + k;
      if (lp >= gt) break;
      const float thp = tp ? tp[lp] : a.thp_u, thn = tn ? tn[lp] : a.thn_u;
      const float rthp = tp ? __frcp_rn(thp) : a.rthp_u, rthn = tn ? __frcp_rn(thn) : a.rthn_u;
      PxStep o;
      px_step<REFR, kFPrefilter>(fr[lp], sr[lp], sl[lp], thp, thn, rthp, rthn, c, s_tab, o);
      cnt += o.kept;
    }
    int total;
    int off = block_excl_scan<NT, int>(cnt, s_scan, &total);
    for (int k = 0; k < PPT && off < lim; ++k) {
      const int lp = lp0 + k;
      if (lp >= gt) break;
      const float thp = tp ? tp[lp] : a.thp_u, thn = tn ? tn[lp] : a.thn_u;
      const float rthp = tp ? __frcp_rn(thp) : a.rthp_u, rthn = tn ? __frcp_rn(thn) : a.rthn_u;
      PxStep o;
      px_step<REFR, kFPrefilter>(fr[lp], sr[lp], sl[lp], thp, thn, rthp, rthn, c, s_tab, o);
      if (o.kept == 0) continue;
      const uint32_t xyp = ((uint32_t)lp << 1) | (o.pos ? 1u : 0u);
      if (o.exact) {
        // regenerate into a small local buffer-free path: count, then write those below lim
        double ad = 0.0, thd = 0.0;
        bool p2;
        const int n = exact_count(fr[lp], sr[lp], thp, thn, c.log_eps, p2, ad, thd);
        int l = sl[lp];
        for (int j = 1; j <= n; ++j) {
          const int tr = exact_trel(j, thd, ad, c.dtd, c.dtm1);
          if (REFR) {
            if (c.tpr + tr - l < c.refr) continue;
            l = c.tpr + tr;
          }
          if (off < lim) un[off] = ((uint32_t)tr << 12) | xyp;
          ++off;
        }
      } else {
        px_emit<REFR>(sl[lp], o.n, o.lo, c, [&](int tr) {
          if (off < lim) un[off] = ((uint32_t)tr << 12) | xyp;
          ++off;
        });
      }
    }
    for (int b = tid; b <= nbk; b += NT) s_hist[b] = 0;
    __syncthreads();
    for (int i = tid; i < lim; i += NT) atomicAdd(&s_hist[un[i] >> 15], 1u);
    __syncthreads();
    {
      const int cc = tid < nbk ? (int)s_hist[tid] : 0;
      int tt;
      const int ex = block_excl_scan<NT, int>(cc, s_scan, &tt);
      if (tid < nbk) {
        if (cc) atomicAdd(a.btot + (int64_t)seg * nbk + tid, (uint32_t)cc);
        s_hist[tid] = (uint32_t)ex;
        rows[(int64_t)tid * nt + q] = (uint32_t)ex;
      }
      if (tid == 0) rows[(int64_t)nbk * nt + q] = (uint32_t)lim;
    }
    __syncthreads();
    if (tid < 32) {  // one warp in list order: stable
      for (int base = 0; base < lim; base += 32) {
        const int i = base + lane;
        const bool valid = i < lim;
        const uint32_t active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          const uint32_t key = un[i];
          const int bk = (int)(key >> 15);
          const uint32_t peers = __match_any_sync(active, bk);
          const int leader = __ffs(peers) - 1;
          uint32_t bpos = 0;
          if (lane == leader) { bpos = s_hist[bk]; s_hist[bk] = bpos + __popc(peers); }
          bpos = __shfl_sync(active, bpos, leader);
          so[bpos + __popc(peers & lanemask_lt())] = key;
        }
        __syncwarp();
      }
    }
    if (tid == 0) a.tile_src[st_idx] = aoff;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2: one CTA per (segment, bucket of 8 t_rel bins)
// ---------------------------------------------------------------------------
// Gather entry: pixel (24 bits) | p << 24 | (t_rel & 7) << 25.
__device__ __forceinline__ uint32_t gentry(uint32_t key, uint32_t gpx0) {
  return (gpx0 + ((key >> 1) & 0x7ffu)) | ((key & 1u) << 24) | (((key >> 12) & 7u) << 25);
}

// Per-warp bin counts of s_g[lo, hi) (lane v < 8 returns the count of bin v).
__device__ __forceinline__ uint32_t warp_bin_counts(const uint32_t* s_g, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  uint32_t my = 0;
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const uint32_t b = i < hi ? (s_g[i] >> 25) & 7u : 8u;
#pragma unroll
    for (uint32_t v = 0; v < 8; ++v) {
      const uint32_t m = __ballot_sync(0xffffffffu, b == v);
      if (lane == (int)v) my += __popc(m);
    }
  }
  return my;
}

// plan (one CTA per segment): split the buckets into pieces of about kOCap
// events.  A bucket above kOCap ("big") is cut at tile boundaries; its pieces
// get per-bin counts from k_fast_count so each can place its events.
constexpr int kPlanNT = 256;
__global__ void __launch_bounds__(kPlanNT) k_fast_plan(FastArgs a) {
  constexpr int NT = kPlanNT;
  __shared__ int s_len[kFMaxTiles];
  __shared__ uint32_t s_bt[kFMaxBuckets];
  __shared__ int s_scan[NT / 32 + 1];
  __shared__ int s_np;
  const int seg = blockIdx.x, tid = threadIdx.x;
  const int nbk = a.nbk, nt = a.ntiles;
  const uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * nt;
  int* pc = a.pieces + (int64_t)seg * a.maxp * 8;
  for (int k = tid; k < nbk; k += NT) s_bt[k] = a.btot[(int64_t)seg * nbk + k];
  __syncthreads();
  // small buckets (<= kOCap events): one piece each, written in parallel
  {
    int run = 0;
    for (int k0 = 0; k0 < nbk; k0 += NT) {
      const int k = k0 + tid;
      const bool small = k < nbk && s_bt[k] > 0 && s_bt[k] <= (uint32_t)kOCap;
      int tt;
      const int ex = run + block_excl_scan<NT, int>(small ? 1 : 0, s_scan, &tt);
      if (small) {
        int* e = pc + ex * 8;
        e[0] = k; e[1] = 0; e[2] = nt; e[3] = ex; e[4] = ex + 1; e[5] = 0;
      }
      run += tt;
    }
    if (tid == 0) s_np = run;
    __syncthreads();
  }
  for (int k = 0; k < nbk; ++k) {
    if (s_bt[k] <= (uint32_t)kOCap) continue;  // (uniform)
    // big bucket: a piece starts where floor(prefix / kSplit) advances (tile
    // granularity, so a piece holds <= kSplit + one slice; k_fast_order walks a
    // piece larger than kOCap in chunks)
    constexpr int kSplit = kOCap - 1024;
    const int j0 = s_np;
    for (int q = tid; q < nt; q += NT)
      s_len[q] = (int)(rows[(int64_t)(k + 1) * nt + q] - rows[(int64_t)k * nt + q]);
    __syncthreads();
    int run = 0, nb = 0;
    for (int q0 = 0; q0 < nt; q0 += NT) {
      const int q = q0 + tid;
      const int len = q < nt ? s_len[q] : 0;
      int tt;
      const int pre = run + block_excl_scan<NT, int>(len, s_scan, &tt);
      const int plen = (q > 0 && q < nt) ? s_len[q - 1] : 0;  // tile q-1 starts at pre - plen
      const bool start = q < nt && (q == 0 || (pre / kSplit) != ((pre - plen) / kSplit));
      int ns;
      const int ex = nb + block_excl_scan<NT, int>(start ? 1 : 0, s_scan, &ns);
      if (start) {
        int* e = pc + (j0 + ex) * 8;
        e[0] = k; e[1] = q; e[3] = j0; e[5] = 1;
      }
      run += tt;
      nb += ns;
    }
    __syncthreads();
    for (int jj = j0 + tid; jj < j0 + nb; jj += NT) {
      int* e = pc + jj * 8;
      e[2] = jj + 1 < j0 + nb ? pc[(jj + 1) * 8 + 1] : nt;
      e[4] = j0 + nb;
    }
    __syncthreads();
    if (tid == 0) s_np = j0 + nb;
    __syncthreads();
  }
  if (tid == 0) a.npieces[seg] = s_np;
}

// per-bin counts of every piece of a big bucket
__global__ void __launch_bounds__(kONT) k_fast_count(FastArgs a) {
  constexpr int NT = kONT;
  __shared__ uint32_t s_c[8];
  const int seg = blockIdx.y, tid = threadIdx.x;
  if (*a.bad != kNoBad) return;
  const int np = a.npieces[seg];
  const int nbk = a.nbk, nt = a.ntiles;
  const uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * nt;
  for (int j = blockIdx.x; j < np; j += gridDim.x) {
    const int* e = a.pieces + ((int64_t)seg * a.maxp + j) * 8;
    if (!e[5]) continue;
    const int k = e[0], qa = e[1], qb = e[2];
    if (tid < 8) s_c[tid] = 0;
    __syncthreads();
    uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = qa + tid; q < qb; q += NT) {
      const uint32_t s0 = rows[(int64_t)k * nt + q], s1 = rows[(int64_t)(k + 1) * nt + q];
      if (s1 == s0) continue;
      const uint32_t* src = tile_keys(a, seg, q);
      for (uint32_t i = s0; i < s1; ++i) {
        const uint32_t b = (__ldg(src + i) >> 12) & 7u;
#pragma unroll
        for (int v = 0; v < 8; ++v) c[v] += b == (uint32_t)v;
      }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint32_t w = warp_sum(c[v]);
      if ((tid & 31) == 0 && w) atomicAdd(&s_c[v], w);
    }
    __syncthreads();
    if (tid < 8) a.pcnt[((int64_t)seg * a.maxp + j) * 8 + tid] = s_c[tid];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kONT, 2) k_fast_order(FastArgs a) {
  constexpr int NT = kONT, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_g = reinterpret_cast<uint32_t*>(smem_raw);  // [kOCap] gathered entries
  uint32_t* s_s = s_g + kOCap;                             // [kOCap] bin-sorted entries
  int* s_goff = reinterpret_cast<int*>(s_s + kOCap);       // [ntiles + 1] gather offsets
  uint32_t* s_src = reinterpret_cast<uint32_t*>(s_goff + a.ntiles + 1);  // [ntiles] slice start
  __shared__ int s_scan[NW + 1];
  __shared__ uint32_t s_wc[NW][8];   // per-warp bin counts -> per-warp bin offsets
  __shared__ uint32_t s_cbs[9];      // bin starts within the chunk (+ total)
  __shared__ int64_t s_pbs[8];       // bin starts of this piece's events within the bucket
  __shared__ int64_t s_kbase[kFMaxBuckets + 1];  // bucket bases within the segment

  const int seg = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*a.bad != kNoBad) return;
  const int np = a.npieces[seg];
  if ((int)blockIdx.x >= np) return;
  const int nbk = a.nbk, nt = a.ntiles;
  const int s = seg / a.T, f = seg % a.T;
  const uint32_t* rows = a.rows + (int64_t)seg * (nbk + 1) * nt;
  const int64_t t0c = a.desc ? a.desc->cur_t0 : a.t0;
  const int64_t tprev = frame_tprev(a, s, f, t0c);
  const uint32_t* keys_seg = a.keys + (int64_t)seg * nt * kFListCap;
  const uint32_t* area_seg = a.area_sorted + (int64_t)seg * a.cap;
  {
    // bucket bases: exclusive scan of the bucket totals
    const uint32_t* bt = a.btot + (int64_t)seg * nbk;
    int tt;
    const int c = tid < nbk ? (int)bt[tid] : 0;
    const int ex = block_excl_scan<NT, int>(c, s_scan, &tt);
    if (tid < nbk) s_kbase[tid] = ex;
    if (tid == 0) s_kbase[nbk] = tt;
    __syncthreads();
  }
  const int W = a.W;
  const float winv = 1.0f / (float)W;

  for (int j = blockIdx.x; j < np; j += gridDim.x) {
    const int* pe = a.pieces + ((int64_t)seg * a.maxp + j) * 8;
    const int k = pe[0], qa = pe[1], qb = pe[2], j0 = pe[3], j1 = pe[4], big = pe[5];
    // slices of the piece's tiles (bit 31 of s_src: in the overflow area)
    int run = 0;
    for (int q0 = qa; q0 < qb; q0 += NT) {
      const int q = q0 + tid;
      int len = 0;
      if (q < qb) {
        const uint32_t s0 = rows[(int64_t)k * nt + q];
        const uint32_t s1 = rows[(int64_t)(k + 1) * nt + q];
        len = (int)(s1 - s0);
        if (len > 0) {
          const int64_t src = a.tile_src[(int64_t)seg * nt + q];
          s_src[q] = src < 0 ? (uint32_t)(q * kFListCap) + s0 : (0x80000000u | (uint32_t)(src + s0));
        }
      }
      int tt;
      const int ex = block_excl_scan<NT, int>(len, s_scan, &tt);
      if (q < qb) s_goff[q] = run + ex;
      run += tt;
    }
    const int total = run;
    if (tid == 0) s_goff[qb] = total;
    if (big && tid < 8) {
      // this piece's bin starts within the bucket: all pieces' counts of lower
      // bins + earlier pieces' counts of the same bin
      const uint32_t* pcn = a.pcnt + (int64_t)seg * a.maxp * 8;
      int64_t below = 0, before = 0;
      for (int jj = j0; jj < j1; ++jj) {
        for (int v = 0; v < tid; ++v) below += pcn[jj * 8 + v];
        if (jj < j) before += pcn[jj * 8 + tid];
      }
      s_pbs[tid] = below + before;
    }
    __syncthreads();
    const int64_t ob = (int64_t)seg * a.seg_stride + s_kbase[k];
    const int64_t tbin0 = tprev + 8 * k;

    for (int g0 = 0; g0 < total; g0 += kOCap) {
      const int n = min(kOCap, total - g0);
      // gather: thread t takes entries [t*m, t*m + m) of the chunk (one binary
      // search for its first tile, then walks forward): all loads independent
      {
        const int m = (n + NT - 1) / NT;
        const int i0 = min(n, tid * m), i1 = min(n, i0 + m);
        if (i0 < i1) {
          int lo = qa, hi = qb - 1;  // last tile with goff <= g0 + i0
          const int gi0 = g0 + i0;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_goff[mid] <= gi0) lo = mid; else hi = mid - 1;
          }
          int q = lo;
          int qend = s_goff[q + 1];
          uint32_t so = s_src[q];
          const uint32_t* srcp = ((so >> 31) ? area_seg + (so & 0x7fffffffu) : keys_seg + so) - s_goff[q];
          uint32_t gpx0 = (uint32_t)q * (uint32_t)a.G;
          for (int i = i0; i < i1; ++i) {
            const int gi = g0 + i;
            while (gi >= qend) {
              ++q;
              qend = s_goff[q + 1];
              so = s_src[q];
              srcp = ((so >> 31) ? area_seg + (so & 0x7fffffffu) : keys_seg + so) - s_goff[q];
              gpx0 = (uint32_t)q * (uint32_t)a.G;
            }
            s_g[i] = gentry(__ldg(srcp + gi), gpx0);
          }
        }
      }
      __syncthreads();
      // stable partition by bin: per-warp counts, offsets, ballot ranks
      const int per = ((n + NW - 1) / NW + 31) & ~31;
      const int lo = min(n, warp * per), hi = min(n, lo + per);
      {
        const uint32_t my = warp_bin_counts(s_g, lo, hi);
        if (lane < 8) s_wc[warp][lane] = my;
      }
      __syncthreads();
      if (tid < 8) {
        uint32_t acc = 0;
        for (int w = 0; w < NW; ++w) { const uint32_t c = s_wc[w][tid]; s_wc[w][tid] = acc; acc += c; }
        s_cbs[tid] = acc;
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t acc = 0;
        for (int b = 0; b < 8; ++b) { const uint32_t c = s_cbs[b]; s_cbs[b] = acc; acc += c; }
        s_cbs[8] = acc;
      }
      __syncthreads();
      {
        uint32_t runb = lane < 8 ? s_cbs[lane] + s_wc[warp][lane] : 0u;  // lane v: next slot of bin v
        for (int base = lo; base < hi; base += 32) {
          const int i = base + lane;
          const bool valid = i < hi;
          const uint32_t e = valid ? s_g[i] : 0u;
          const uint32_t b = valid ? (e >> 25) & 7u : 8u;
          uint32_t mine = 0, mv = 0;
#pragma unroll
          for (uint32_t v = 0; v < 8; ++v) {
            const uint32_t m = __ballot_sync(0xffffffffu, b == v);
            mine = b == v ? m : mine;
            mv = lane == (int)v ? m : mv;
          }
          const uint32_t slot = __shfl_sync(0xffffffffu, runb, (int)(b & 7u));
          if (valid) s_s[slot + __popc(mine & lanemask_lt())] = e;
          runb += __popc(mv);
        }
      }
      __syncthreads();
      const bool contiguous = !big && total <= kOCap;
      for (int i = tid; i < n; i += NT) {
        const uint32_t e = s_s[i];
        const uint32_t b = (e >> 25) & 7u;
        // big pieces / later chunks: bin runs at the piece's bin starts (+ events
        // of this bin in earlier chunks, accumulated in s_pbs)
        const int64_t o = contiguous ? ob + i : ob + s_pbs[b] + (i - (int)s_cbs[b]);
        const uint32_t gp = e & 0xffffffu;
        uint32_t y = (uint32_t)((float)gp * winv);
        if (y * (uint32_t)W > gp) --y;
        else if ((y + 1) * (uint32_t)W <= gp) ++y;
        a.out_t[o] = tbin0 + (int64_t)b;
        a.out_x[o] = (uint16_t)(gp - y * (uint32_t)W);
        a.out_y[o] = (uint16_t)y;
        a.out_p[o] = (e >> 24) & 1u ? (int8_t)1 : (int8_t)-1;
      }
      __syncthreads();
      if (!contiguous && tid < 8) s_pbs[tid] += s_cbs[tid + 1] - s_cbs[tid];
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename K>
static void ensure_smem_fast(K k, size_t bytes) {
  static const void* done[16];
  static int ndone = 0;
  const void* key = reinterpret_cast<const void*>(k);
  for (int i = 0; i < ndone; ++i)
    if (done[i] == key) return;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (ndone < 16) done[ndone++] = key;
}

size_t fast_gen_smem() { return (size_t)2 * kFListCap * 4 + (size_t)kFVpt * (kFNT / 32) * kFMaxBuckets * 2; }
size_t fast_order_smem(int ntiles) { return (size_t)2 * kOCap * 4 + (size_t)(2 * ntiles + 1) * 4; }

cudaError_t launch_fast_gen(const FastArgs& a, cudaStream_t st) {
  const size_t smem = fast_gen_smem();
  const unsigned grid = (unsigned)((int64_t)a.S * a.ntiles);
  const bool uni = a.thp == nullptr;
  const bool refr = a.refr > 0;
#define EVS_FAST_GEN(R, U)                        \
  {                                               \
    auto kf = k_fast_gen<R, U>;                   \
    ensure_smem_fast(kf, fast_gen_smem()); \
    kf<<<grid, kFNT, smem, st>>>(a);              \
  }
  if (refr) {
    if (uni) EVS_FAST_GEN(true, true) else EVS_FAST_GEN(true, false)
  } else {
    if (uni) EVS_FAST_GEN(false, true) else EVS_FAST_GEN(false, false)
  }
#undef EVS_FAST_GEN
  return cudaGetLastError();
}

cudaError_t launch_fast_fix(const FastArgs& a, int nseg, cudaStream_t st) {
  k_fast_fix<<<nseg, kFixNT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fast_redo(const FastArgs& a, int nseg, cudaStream_t st) {
  dim3 grid(kRedoCtas, nseg);
  if (a.refr > 0) k_fast_redo<true><<<grid, kRedoNT, 0, st>>>(a);
  else k_fast_redo<false><<<grid, kRedoNT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fast_plan(const FastArgs& a, int nseg, cudaStream_t st) {
  k_fast_plan<<<nseg, kPlanNT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fast_order(const FastArgs& a, int nseg, cudaStream_t st) {
  k_fast_count<<<dim3(16, nseg), kONT, 0, st>>>(a);
  const size_t smem = fast_order_smem(a.ntiles);
  ensure_smem_fast(k_fast_order, fast_order_smem(kFMaxTiles));
  // one CTA per piece in the common case (pieces = buckets); big buckets add
  // pieces that the CTAs pick up round-robin
  dim3 grid(a.nbk + 8, nseg);
  k_fast_order<<<grid, kONT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace evs
