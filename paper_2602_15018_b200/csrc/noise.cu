// Exact background noise on the GPU: inject_noise_events (model.py:174-212)
// reproduced draw-for-draw from numpy's Generator(PCG64(SeedSequence(seed))).
//
// numpy consumes one sequential PCG64 stream: P Poisson counts (multiplication
// method for lam < 10, PTRS for lam >= 10), then `total` doubles for the
// timestamps, then buffered Lemire bytes of u32 draws for the polarities
// (SURVEY.md Appendix B).  The GPU evaluates the stream in parallel:
//   A  each thread jumps (LCG jump-ahead) to its chunk and counts the pixel
//      terminators / events in the part of the stream it owns;
//   B  one block scans those counts and locates the P-th terminator (the
//      number of Poisson draws D);
//   C  threads re-walk their chunks and label every event with its pixel;
//   D  per event, jump to draw D + k (timestamp) and to the polarity byte;
//   E  per event, rank within its pixel by (t_rel, draw order) -> output.
// The multiplication method is sequential within a pixel; a pixel can only
// continue past a draw U > exp(-lam), so every draw U <= exp(-lam) ends a
// pixel and the stream splits into independent segments at those draws.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/evsim_b200.h"
#include "common.cuh"
#include "kernels.cuh"

namespace evs {

typedef unsigned __int128 u128;
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}
__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double u_double(uint64_t v) {  // numpy next_double
  return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}
// state after n LCG steps from s (jump-ahead by repeated squaring)
__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, uint64_t n) {
  u128 am = 1, ag = 0;              // accumulated: s' = am*s + ag*inc
  u128 cm = pcg_mult(), cg = 1;     // current power-of-two step
  while (n) {
    if (n & 1) { am = am * cm; ag = ag * cm + cg; }
    cg = (cm + 1) * cg;
    cm = cm * cm;
    n >>= 1;
  }
  return am * s + ag * inc;
}

struct NoiseArgs {
  int64_t P, W, dt, t_prev;
  double lam, enlam;
  int ptrs;
  double slam, loglam, pa, pb, log_invalpha, vr;
  uint64_t s_hi, s_lo, i_hi, i_lo;
  int64_t L, nthreads, cap;
  int64_t* n_term;  // [nthreads] per-walker counts (pass A)
  int64_t* n_ev;    // [nthreads] per-walker counts (pass A)
  int64_t* blk_term;  // [nblk] per-256-walker-block totals -> exclusive prefix (k_noise_scan)
  int64_t* blk_ev;
  int64_t nblk;
  int64_t* meta;    // [0] D (draws used by the counts) [1] total events [2] insufficient [3] overflow
  int32_t* ev_pix;  // [cap]
  int32_t* ev_trel; // [cap]
  int8_t* ev_pol;   // [cap]
  int order;
  int64_t* out_t;
  uint16_t* out_x;
  uint16_t* out_y;
  int8_t* out_p;
  uint64_t* out_key;
};

__device__ __forceinline__ u128 s0_of(const NoiseArgs& a) { return ((u128)a.s_hi << 64) | a.s_lo; }
__device__ __forceinline__ u128 inc_of(const NoiseArgs& a) { return ((u128)a.i_hi << 64) | a.i_lo; }

// numpy random_loggam, rounding each operation like the host C code (no FMA)
__device__ double np_loggam(double x) {
  const double a[10] = {8.333333333333333e-02, -2.777777777777778e-03, 7.936507936507937e-04,
                        -5.952380952380952e-04, 8.417508417508418e-04, -1.917526917526918e-03,
                        6.410256410256410e-03, -2.955065359477124e-02, 1.796443723688307e-01,
                        -1.39243221690590e+00};
  if (x == 1.0 || x == 2.0) return 0.0;
  const int64_t n = x < 7.0 ? (int64_t)(7 - x) : 0;
  double x0 = __dadd_rn(x, (double)n);
  const double r = __ddiv_rn(1.0, x0);
  const double x2 = __dmul_rn(r, r);
  const double lg2pi = 1.8378770664093453e+00;
  double gl0 = a[9];
  for (int k = 8; k >= 0; --k) { gl0 = __dmul_rn(gl0, x2); gl0 = __dadd_rn(gl0, a[k]); }
  double gl = __dadd_rn(__ddiv_rn(gl0, x0), __dmul_rn(0.5, lg2pi));
  gl = __dadd_rn(gl, __dmul_rn(__dadd_rn(x0, -0.5), log(x0)));
  gl = __dadd_rn(gl, -x0);
  if (x < 7.0)
    for (int64_t k = 1; k <= n; ++k) { gl = __dadd_rn(gl, -log(__dadd_rn(x0, -1.0))); x0 = __dadd_rn(x0, -1.0); }
  return gl;
}

// one PTRS trial from the pair (u0, u1); returns k >= 0 on accept, -1 on reject
__device__ __forceinline__ int64_t ptrs_trial(const NoiseArgs& a, uint64_t u0, uint64_t u1) {
  const double U = __dadd_rn(u_double(u0), -0.5);
  const double V = u_double(u1);
  const double us = __dadd_rn(0.5, -fabs(U));
  const double t = __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, a.pa), us), a.pb), U), a.lam), 0.43);
  const int64_t k = (int64_t)floor(t);
  if (us >= 0.07 && V <= a.vr) return k;
  if (k < 0 || (us < 0.013 && V > us)) return -1;
  const double lhs = __dadd_rn(__dadd_rn(log(V), a.log_invalpha),
                               -log(__dadd_rn(__ddiv_rn(a.pa, __dmul_rn(us, us)), a.pb)));
  const double rhs = __dadd_rn(__dadd_rn(-a.lam, __dmul_rn((double)k, a.loglam)), -np_loggam((double)k + 1));
  return lhs <= rhs ? k : -1;
}

// Walk thread c's part of the stream.  EMIT=false: count terminators/events.
// EMIT=true: label events with pixels (needs the exclusive prefixes).
template <bool EMIT>
__device__ __forceinline__ void noise_walk_body(const NoiseArgs& a, int64_t c, int64_t term0, int64_t ev0,
                                                int64_t& term, int64_t& ev) {
  const u128 inc = inc_of(a);
  term = 0;
  ev = 0;
  if (EMIT && term0 >= a.P) return;
  if (a.ptrs) {
    const int64_t m0 = c * a.L;
    u128 s = pcg_advance(s0_of(a), inc, (uint64_t)(2 * m0));
    for (int64_t m = m0; m < m0 + a.L; ++m) {
      s = s * pcg_mult() + inc;
      const uint64_t u0 = xsl_rr(s);
      s = s * pcg_mult() + inc;
      const uint64_t u1 = xsl_rr(s);
      const int64_t k = ptrs_trial(a, u0, u1);
      if (k < 0) continue;
      if (EMIT) {
        const int64_t pix = term0 + term;
        for (int64_t i = 0; i < k; ++i)
          if (ev0 + ev + i < a.cap) a.ev_pix[ev0 + ev + i] = (int32_t)pix;
        if (pix == a.P - 1) { a.meta[0] = 2 * (m + 1); a.meta[1] = ev0 + ev + k; ev += k; ++term; return; }
      }
      ev += k;
      ++term;
    }
  } else {
    const int64_t d0 = c * a.L, d1 = d0 + a.L;
    u128 s = pcg_advance(s0_of(a), inc, (uint64_t)d0);
    int64_t d = d0;
    // skip to the first segment start owned by this thread
    if (c > 0) {
      for (;;) {
        if (d >= d1) return;  // no non-candidate in this chunk: an earlier thread owns it
        s = s * pcg_mult() + inc;
        const double U = u_double(xsl_rr(s));
        ++d;
        if (!(U > a.enlam)) break;  // non-candidate: always ends a pixel
      }
    }
    // resolve segments until a non-candidate at index >= d1 ends the region
    double prod = 1.0;
    for (;;) {
      s = s * pcg_mult() + inc;
      const double U = u_double(xsl_rr(s));
      const int64_t dd = d++;
      prod *= U;
      if (prod > a.enlam) {  // pixel continues: one more event
        if (EMIT && ev0 + ev < a.cap) a.ev_pix[ev0 + ev] = (int32_t)(term0 + term);
        ++ev;
      } else {
        prod = 1.0;
        if (EMIT && term0 + term == a.P - 1) { a.meta[0] = dd + 1; a.meta[1] = ev0 + ev; ++term; return; }
        ++term;
        if (dd >= d1 && !(U > a.enlam)) break;
      }
    }
  }
}

// Pass A (EMIT=false): per-walker counts and their per-block totals.  Pass B
// (EMIT=true): each walker's exclusive prefix = block prefix (k_noise_scan)
// + in-block scan, then the labelling walk.
template <bool EMIT>
__device__ __forceinline__ void noise_walk(const NoiseArgs& a) {
  __shared__ int64_t s1[9], s2[9];
  if (blockIdx.x >= a.nblk) return;  // (batched launch: a smaller frame)
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool mine = c < a.nthreads;
  int64_t term = 0, ev = 0;
  if (!EMIT) {
    if (mine) {
      noise_walk_body<false>(a, c, 0, 0, term, ev);
      a.n_term[c] = term;
      a.n_ev[c] = ev;
    }
    int64_t tt, te;
    block_excl_scan<256, int64_t>(term, s1, &tt);
    block_excl_scan<256, int64_t>(ev, s2, &te);
    if (threadIdx.x == 0) { a.blk_term[blockIdx.x] = tt; a.blk_ev[blockIdx.x] = te; }
    return;
  }
  const int64_t rt = mine ? a.n_term[c] : 0, re = mine ? a.n_ev[c] : 0;
  int64_t tt, te;
  const int64_t t0 = block_excl_scan<256, int64_t>(rt, s1, &tt) + a.blk_term[blockIdx.x];
  const int64_t e0 = block_excl_scan<256, int64_t>(re, s2, &te) + a.blk_ev[blockIdx.x];
  if (mine) noise_walk_body<true>(a, c, t0, e0, term, ev);
}

// single-block exclusive scan of the walker-block totals (blk_term, blk_ev);
// flags a too-short stream.  Chunks of kNsChunk blocks: coalesced loads into shared memory, each thread
// sums its kNsPer consecutive entries, one block scan per array, prefixes
// written back through shared memory with coalesced stores.
constexpr int kNsPer = 4, kNsChunk = 1024 * kNsPer;
__device__ __forceinline__ void noise_scan(const NoiseArgs& a) {
  extern __shared__ __align__(16) unsigned char nsm[];
  int64_t* sT = reinterpret_cast<int64_t*>(nsm);  // [kNsChunk]
  int64_t* sE = sT + kNsChunk;                    // [kNsChunk]
  __shared__ int64_t s1[33], s2[33];
  const int tid = threadIdx.x;
  if (tid == 0) { a.meta[0] = -1; a.meta[1] = 0; a.meta[2] = 0; a.meta[3] = 0; }
  const int64_t n = a.nblk;
  int64_t run_t = 0, run_e = 0;
  for (int64_t base = 0; base < n; base += kNsChunk) {
#pragma unroll
    for (int j = 0; j < kNsPer; ++j) {
      const int64_t i = base + j * 1024 + tid;
      sT[j * 1024 + tid] = i < n ? a.blk_term[i] : 0;
      sE[j * 1024 + tid] = i < n ? a.blk_ev[i] : 0;
    }
    __syncthreads();
    int64_t vt[kNsPer], ve[kNsPer], st = 0, se = 0;
#pragma unroll
    for (int j = 0; j < kNsPer; ++j) {
      vt[j] = sT[tid * kNsPer + j];
      ve[j] = sE[tid * kNsPer + j];
      st += vt[j];
      se += ve[j];
    }
    int64_t tt, te;
    int64_t xt = block_excl_scan<1024, int64_t>(st, s1, &tt) + run_t;
    int64_t xe = block_excl_scan<1024, int64_t>(se, s2, &te) + run_e;
#pragma unroll
    for (int j = 0; j < kNsPer; ++j) {
      sT[tid * kNsPer + j] = xt;
      sE[tid * kNsPer + j] = xe;
      xt += vt[j];
      xe += ve[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kNsPer; ++j) {
      const int64_t i = base + j * 1024 + tid;
      if (i < n) { a.blk_term[i] = sT[j * 1024 + tid]; a.blk_ev[i] = sE[j * 1024 + tid]; }
    }
    run_t += tt;
    run_e += te;
    __syncthreads();  // before the next chunk overwrites sT / sE
  }
  if (tid == 0 && run_t < a.P) a.meta[2] = 1;  // not enough draws: caller retries bigger
}

// per event: timestamp draw D + k and polarity byte k of the u32 stream
__device__ __forceinline__ void noise_draws(const NoiseArgs& a) {
  const int64_t total = a.meta[1], D = a.meta[0];
  if (a.meta[2] || D < 0) return;
  if (total > a.cap) { if (blockIdx.x == 0 && threadIdx.x == 0) a.meta[3] = 1; return; }
  const u128 inc = inc_of(a);
  constexpr int64_t E = 16;  // events per thread (sequential draws after one jump)
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * E;
  if (k0 >= total) return;
  const int64_t k1 = k0 + E < total ? k0 + E : total;
  u128 s = pcg_advance(s0_of(a), inc, (uint64_t)(D + k0));
  for (int64_t k = k0; k < k1; ++k) {  // model.py:201: t_rel = floor(U * dt)
    s = s * pcg_mult() + inc;
    a.ev_trel[k] = (int32_t)floor(u_double(xsl_rr(s)) * (double)a.dt);
  }
  // model.py:202: integers(0, 2, int8): u32 m = k/4 is the low (m even) or
  // high half of u64 number D + total + m/2; byte k%4; value = byte >> 7
  const int64_t q0 = k0 / 8;
  u128 s2 = pcg_advance(s0_of(a), inc, (uint64_t)(D + total + q0));
  uint64_t cur = 0;
  int64_t cur_q = -1;
  for (int64_t k = k0; k < k1; ++k) {
    const int64_t q = k / 8;
    while (cur_q < q) { s2 = s2 * pcg_mult() + inc; cur = xsl_rr(s2); ++cur_q; cur_q = cur_q < q0 ? q0 : cur_q; }
    const uint8_t byte = (uint8_t)(cur >> (8 * (k % 8)));
    a.ev_pol[k] = (int8_t)(2 * (byte >> 7) - 1);
  }
}

// per event: rank within its pixel (reference order: t_rel, then draw order;
// merge order: polarity, t_rel, draw order) and write the output
__device__ __forceinline__ void noise_place(const NoiseArgs& a) {
  const int64_t total = a.meta[1];
  if (a.meta[2] || a.meta[3] || a.meta[0] < 0) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pix = a.ev_pix[k];
    const int32_t tk = a.ev_trel[k];
    const int8_t pk = a.ev_pol[k];
    int64_t lo = k, hi = k + 1;
    while (lo > 0 && a.ev_pix[lo - 1] == pix) --lo;
    while (hi < total && a.ev_pix[hi] == pix) ++hi;
    int64_t rank = 0;
    for (int64_t j = lo; j < hi; ++j) {
      if (j == k) continue;
      const int32_t tj = a.ev_trel[j];
      bool before;
      if (a.order == 1) {
        const int8_t pj = a.ev_pol[j];
        before = (pj < pk) || (pj == pk && (tj < tk || (tj == tk && j < k)));
      } else {
        before = tj < tk || (tj == tk && j < k);
      }
      rank += before;
    }
    const int64_t o = lo + rank;
    const int64_t x = pix % a.W, y = pix / a.W;
    if (a.order == 1) {
      a.out_key[o] = ((uint64_t)(uint32_t)tk << kKeyPixBits) | ((uint64_t)y << 17) | ((uint64_t)x << 1) |
                     (pk > 0 ? 1u : 0u);
    } else {
      a.out_t[o] = a.t_prev + tk;
      a.out_x[o] = (uint16_t)x;
      a.out_y[o] = (uint16_t)y;
      a.out_p[o] = pk;
    }
  }
}

// Up to kNoiseBatch frames per launch (grid.y = frame): each frame's own
// NoiseArgs; the per-frame walks are short, so batching fills the GPU.
constexpr int kNoiseBatch = 16;
struct NoiseBatch {
  NoiseArgs a[kNoiseBatch];
};
template <bool EMIT>
__global__ void __launch_bounds__(256) k_noise_walk(const __grid_constant__ NoiseBatch b) { noise_walk<EMIT>(b.a[blockIdx.y]); }
__global__ void __launch_bounds__(1024) k_noise_scan(const __grid_constant__ NoiseBatch b) { noise_scan(b.a[blockIdx.y]); }
__global__ void __launch_bounds__(256) k_noise_draws(const __grid_constant__ NoiseBatch b) { noise_draws(b.a[blockIdx.y]); }
__global__ void __launch_bounds__(256) k_noise_place(const __grid_constant__ NoiseBatch b) { noise_place(b.a[blockIdx.y]); }

}  // namespace evs

using namespace evs;

namespace {

struct NoiseLayout {
  int64_t L, nthreads, cap, nblk;
  size_t n_term, n_ev, blk_term, blk_ev, meta, ev_pix, ev_trel, ev_pol, total;
};

constexpr size_t kAl = 256;
inline size_t al(size_t v) { return (v + kAl - 1) / kAl * kAl; }

bool noise_layout(const evs_noise_params* p, NoiseLayout* L) {
  if (!p || p->width < 1 || p->height < 1 || p->t_now <= p->t_prev || !(p->lam > 0)) return false;
  const int64_t P = (int64_t)p->width * p->height;
  const bool ptrs = p->lam >= 10;
  L->L = ptrs ? 32 : 64;  // draws per walker (16 measured no faster: the jump-ahead then dominates)
  // trials needed: P terminators; mult: P + events draws; PTRS: ~P/acceptance pairs
  const double mean_ev = p->lam * (double)P;
  const double draws = ptrs ? 1.5 * (double)P + 64.0 * std::sqrt((double)P) + 4096.0
                            : (double)P + mean_ev + 12.0 * std::sqrt(mean_ev + 1.0) + 4096.0;
  const double scale = p->draw_scale > 1.0 ? p->draw_scale : 1.0;
  L->nthreads = (int64_t)(draws * scale / (double)L->L) + 1;
  L->cap = p->capacity > 0 ? p->capacity : (int64_t)(mean_ev + 12.0 * std::sqrt(mean_ev + 1.0) + 1024.0);
  size_t off = 0;
  L->n_term = off; off = al(off + (size_t)L->nthreads * 8);
  L->n_ev = off; off = al(off + (size_t)L->nthreads * 8);
  L->nblk = (L->nthreads + 255) / 256;
  L->blk_term = off; off = al(off + (size_t)L->nblk * 8);
  L->blk_ev = off; off = al(off + (size_t)L->nblk * 8);
  L->meta = off; off = al(off + 8 * 8);
  L->ev_pix = off; off = al(off + (size_t)L->cap * 4);
  L->ev_trel = off; off = al(off + (size_t)L->cap * 4);
  L->ev_pol = off; off = al(off + (size_t)L->cap);
  L->total = off;
  return true;
}

template <typename T>
T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

}  // namespace

extern "C" {

size_t evs_noise_workspace_bytes(const evs_noise_params* p) {
  NoiseLayout L;
  return noise_layout(p, &L) ? L.total : 0;
}

int64_t evs_noise_capacity(const evs_noise_params* p) {
  NoiseLayout L;
  return noise_layout(p, &L) ? L.cap : -1;
}

static NoiseArgs noise_args(const evs_noise_params* p, const NoiseLayout& L, void* ws, int64_t* ev_t,
                            uint16_t* ev_x, uint16_t* ev_y, int8_t* ev_p, uint64_t* ev_key, int64_t* meta_out) {
  NoiseArgs a;
  memset(&a, 0, sizeof(a));
  a.P = (int64_t)p->width * p->height;
  a.W = p->width;
  a.dt = p->t_now - p->t_prev;
  a.t_prev = p->t_prev;
  a.lam = p->lam;
  a.enlam = p->enlam;
  a.ptrs = p->lam >= 10;
  if (a.ptrs) {  // numpy random_poisson_ptrs constants, host libm like numpy
    a.slam = std::sqrt(p->lam);
    a.loglam = std::log(p->lam);
    a.pb = 0.931 + 2.53 * a.slam;
    a.pa = -0.059 + 0.02483 * a.pb;
    const double invalpha = 1.1239 + 1.1328 / (a.pb - 3.4);
    a.vr = 0.9277 - 3.6224 / (a.pb - 2);
    a.log_invalpha = std::log(invalpha);
  }
  a.s_hi = p->pcg[0]; a.s_lo = p->pcg[1]; a.i_hi = p->pcg[2]; a.i_lo = p->pcg[3];
  a.L = L.L; a.nthreads = L.nthreads; a.cap = L.cap;
  a.n_term = at<int64_t>(ws, L.n_term);
  a.n_ev = at<int64_t>(ws, L.n_ev);
  a.blk_term = at<int64_t>(ws, L.blk_term);
  a.blk_ev = at<int64_t>(ws, L.blk_ev);
  a.nblk = L.nblk;
  a.meta = meta_out ? meta_out : at<int64_t>(ws, L.meta);
  a.ev_pix = at<int32_t>(ws, L.ev_pix);
  a.ev_trel = at<int32_t>(ws, L.ev_trel);
  a.ev_pol = at<int8_t>(ws, L.ev_pol);
  a.order = p->order;
  a.out_t = ev_t; a.out_x = ev_x; a.out_y = ev_y; a.out_p = ev_p; a.out_key = ev_key;
  return a;
}

// the five passes over nf frames of one batch (grid.y = frame)
static cudaError_t launch_noise(const NoiseBatch& b, const NoiseLayout* Ls, int nf, cudaStream_t st) {
  int64_t gw = 1, gd = 1, gp = 1;
  for (int f = 0; f < nf; ++f) {
    const NoiseLayout& L = Ls[f];
    gw = std::max<int64_t>(gw, (L.nthreads + 255) / 256);
    gd = std::max<int64_t>(gd, (L.cap / 16 + 255) / 256 + 1);
    gp = std::max<int64_t>(gp, L.cap < 148 * 1024 ? (L.cap + 255) / 256 + 1 : 148 * 4);
  }
  k_noise_walk<false><<<dim3((unsigned)gw, nf), 256, 0, st>>>(b);
  {
    const int smem = 2 * kNsChunk * (int)sizeof(int64_t);
    smem_optin(reinterpret_cast<const void*>(k_noise_scan));
    k_noise_scan<<<dim3(1, nf), 1024, smem, st>>>(b);
  }
  k_noise_walk<true><<<dim3((unsigned)gw, nf), 256, 0, st>>>(b);
  k_noise_draws<<<dim3((unsigned)gd, nf), 256, 0, st>>>(b);
  k_noise_place<<<dim3((unsigned)gp, nf), 256, 0, st>>>(b);
  return cudaGetLastError();
}

evs_status evs_noise(const evs_noise_params* p, int64_t* ev_t, uint16_t* ev_x, uint16_t* ev_y, int8_t* ev_p,
                     uint64_t* ev_key, int64_t* meta_out, void* ws, size_t ws_bytes, void* stream) {
  NoiseLayout L;
  if (!noise_layout(p, &L)) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  if (p->order == 1 ? !ev_key : (!ev_t || !ev_x || !ev_y || !ev_p)) return EVS_ERR_ARG;
  NoiseBatch b;
  memset(&b, 0, sizeof(b));
  b.a[0] = noise_args(p, L, ws, ev_t, ev_x, ev_y, ev_p, ev_key, meta_out);
  return launch_noise(b, &L, 1, static_cast<cudaStream_t>(stream)) == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

size_t evs_noise_batch_workspace_bytes(const evs_noise_params* ps, int32_t nf) {
  size_t total = 0;
  for (int32_t f = 0; f < nf; ++f) {
    NoiseLayout L;
    if (!noise_layout(ps + f, &L)) return 0;
    total += L.total;
  }
  return total;
}

evs_status evs_noise_batch(const evs_noise_params* ps, int32_t nf, int64_t* ev_t, uint16_t* ev_x, uint16_t* ev_y,
                           int8_t* ev_p, int64_t ev_stride, int64_t* meta_out, void* ws, size_t ws_bytes,
                           void* stream) {
  if (!ps || nf < 0 || !ev_t || !ev_x || !ev_y || !ev_p || !meta_out || ev_stride < 0) return EVS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int32_t f0 = 0; f0 < nf; f0 += kNoiseBatch) {
    const int n = std::min<int>(kNoiseBatch, nf - f0);
    NoiseBatch b;
    memset(&b, 0, sizeof(b));
    NoiseLayout Ls[kNoiseBatch];
    size_t off = 0;
    for (int f = 0; f < f0; ++f) {  // workspace offset of this batch's first frame
      NoiseLayout L;
      if (!noise_layout(ps + f, &L)) return EVS_ERR_ARG;
      off += L.total;
    }
    for (int j = 0; j < n; ++j) {
      const evs_noise_params* p = ps + f0 + j;
      if (!noise_layout(p, &Ls[j]) || p->order != 0) return EVS_ERR_ARG;
      if (!ws || ws_bytes < off + Ls[j].total) return EVS_ERR_WORKSPACE;
      if (Ls[j].cap > ev_stride) return EVS_ERR_ARG;  // each frame's capacity must fit its row
      const int64_t r = (int64_t)(f0 + j) * ev_stride;
      b.a[j] = noise_args(p, Ls[j], static_cast<char*>(ws) + off, ev_t + r, ev_x + r, ev_y + r, ev_p + r,
                          nullptr, meta_out + 4 * (int64_t)(f0 + j));
      off += Ls[j].total;
    }
    if (launch_noise(b, Ls, n, st) != cudaSuccess) return EVS_ERR_CUDA;
  }
  return EVS_OK;
}

}  // extern "C"
