// Certified f32 lane math shared by the event-generation kernels (k1_list.cu,
// fast_path.cu).  See fast_path.cuh for the error model: every observable of
// a pixel-frame (n, the crossing times, the refractory filter, the new level)
// depends on the f64 difference |ln(v + eps) - ref| only through floors, which
// are evaluated in f32 from a "lite" log and certified with an error band; a
// straddling band marks the pixel "slow" and the caller takes the exact f64
// path (the reference's formulas, model.py:124-163).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "log_table.h"

namespace evs {

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct LiteOut {
  float uf;    // t_rel(j) ~ j * uf
  float erel;  // relative band of j * uf
};

// Table of the lite log (shared memory): c_i, 1/c_i, log(c_i) (hi part).
struct LiteTab {
  double c[128], invc[128], lh[128];
};
__device__ __forceinline__ void load_lite_tab(LiteTab& t) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    t.c[i] = kLogTable[i][0];
    t.invc[i] = kLogTable[i][1];
    t.lh[i] = kLogTable[i][2];
  }
}

// Per-frame constants of the lane math.
struct FrameCtx {
  double log_eps, dtd;
  float log_eps_f, dtf;
  int dtm1, tpr, refr;  // tpr: frame start relative to the call's time base
};

// Straight-line lane math for the common case n <= 2 (no loops, no branches):
// the same certified f32 evaluation as lite_count / lite_trel.  Returns
//   bits 0-10 t_rel(1), 11-21 t_rel(2), 22 kept(1), 23 kept(2), 24 pos,
//   25-26 n (0..2), 31 slow (band straddles an integer, n > 2, or x outside
//   the table's range: px_step decides),
// and the last kept time in lnew.  dt <= 2048 (11-bit t_rel).
constexpr uint32_t kF2Slow = 0x80000000u, kF2K1 = 1u << 22, kF2K2 = 1u << 23, kF2Pos = 1u << 24;
template <bool REFR>
__device__ __forceinline__ uint32_t px_fast2(float v, float r, int lrel, float thp, float thn, float rthp,
                                             float rthn, const FrameCtx& c, const LiteTab& T, int& lnew) {
  const double x = __dadd_rn((double)v, c.log_eps);
  const uint64_t ix = (uint64_t)__double_as_longlong(x);
  const bool bad_x = ix < 0x0010000000000000ull || ix >= 0x7ff0000000000000ull;
  const uint64_t tmp = ix - kLogOff;
  const int i = (int)((tmp >> (52 - kLogTableBits)) & ((1u << kLogTableBits) - 1));
  const int k = (int)((int64_t)tmp >> 52);
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
  const double d = __dsub_rn(z, T.c[i]);
  const float rf = __double2float_rn(__dmul_rn(d, T.invc[i]));
  float pf = fmaf(rf, 0.2f, -0.25f);
  pf = fmaf(pf, rf, 0.33333334f);
  pf = fmaf(pf, rf, -0.5f);
  pf = fmaf(pf, rf, 1.0f);
  pf = __fmul_rn(pf, rf);
  const double dd = __dsub_rn(fma((double)k, 0.6931471805599453, T.lh[i]), (double)r);
  const float df = __fadd_rn(__double2float_rn(dd), pf);
  const bool pos = df > 0.f;
  const float ad = fabsf(df);
  const float th = pos ? thp : thn;
  const float rth = pos ? rthp : rthn;
  const float q1 = fmaf(ad, rth, 1e-4f);
  const float dn = fmaf(q1, 6e-7f, fmaf(1e-8f, rth, 1e-10f));
  const float nlo = floorf(__fsub_rn(q1, dn)), nhi = floorf(__fadd_rn(q1, dn));
  const int n = (int)nlo;
  const float ra = rcp_approx(ad);
  const float uf = __fmul_rn(__fmul_rn(th, c.dtf), ra);
  const float erel = fmaf(1e-8f, ra, 1e-6f);
  const float a1 = __fmul_rn(1.0f, uf), a2 = __fmul_rn(2.0f, uf);
  const float b1 = fmaf(a1, erel, 1e-6f), b2 = fmaf(a2, erel, 1e-6f);
  const int t1 = min((int)floorf(__fsub_rn(a1, b1)), c.dtm1), t1h = min((int)floorf(__fadd_rn(a1, b1)), c.dtm1);
  const int t2 = min((int)floorf(__fsub_rn(a2, b2)), c.dtm1), t2h = min((int)floorf(__fadd_rn(a2, b2)), c.dtm1);
  const bool slow = bad_x | (nlo != nhi) | (q1 > 1e6f) | (n > 2) | ((n >= 1) & (t1 != t1h)) |
                    ((n >= 2) & (t2 != t2h));
  const bool k1 = (n >= 1) && (!REFR || c.tpr + t1 - lrel >= c.refr);
  const int l1 = k1 ? c.tpr + t1 : lrel;
  const bool k2 = (n >= 2) && (!REFR || c.tpr + t2 - l1 >= c.refr);
  lnew = k2 ? c.tpr + t2 : l1;
  return (slow ? kF2Slow : 0u) | ((uint32_t)(t1 & 0x7ff)) | ((uint32_t)(t2 & 0x7ff) << 11) | (k1 ? kF2K1 : 0u) |
         (k2 ? kF2K2 : 0u) | (pos ? kF2Pos : 0u) | ((uint32_t)(n & 3) << 25);
}

}  // namespace evs
