// canonical_sort of an arbitrary device batch (parallel.py:112-123) and
// host-side numpy SeedSequence->PCG64 seeding (for the noise path).
//
// The batch is packed into 64-bit keys ((t - t_min) << 33 | y << 17 | x << 1 |
// (p > 0)) whose unsigned order is exactly the reference lexsort order
// (t, y, x, p); the keys are sorted with LSD onesweep passes (k_order) over
// all key bits and unpacked into SoA by the last pass.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/evsim_b200.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace evs;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
template <typename T>
T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

__global__ void __launch_bounds__(256) k_batch_stats(int64_t n, const int64_t* __restrict__ t,
                                                     const uint16_t* __restrict__ x,
                                                     const uint16_t* __restrict__ y,
                                                     const int8_t* __restrict__ p, int64_t* out) {
  // out: [0] min t (as order-preserving u64), [1] max t, [2] max x, [3] max y, [4] bad p
  uint64_t tmin = ~0ull, tmax = 0;
  uint32_t xm = 0, ym = 0, badp = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = (uint64_t)t[i] ^ 0x8000000000000000ull;
    tmin = u < tmin ? u : tmin;
    tmax = u > tmax ? u : tmax;
    xm = max(xm, (uint32_t)x[i]);
    ym = max(ym, (uint32_t)y[i]);
    badp |= (p[i] != 1 && p[i] != -1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t a = __shfl_xor_sync(0xffffffffu, tmin, o), b = __shfl_xor_sync(0xffffffffu, tmax, o);
    tmin = a < tmin ? a : tmin;
    tmax = b > tmax ? b : tmax;
    xm = max(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    ym = max(ym, __shfl_xor_sync(0xffffffffu, ym, o));
    badp |= __shfl_xor_sync(0xffffffffu, badp, o);
  }
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out);
    atomicMin(o + 0, tmin);
    atomicMax(o + 1, tmax);
    atomicMax(o + 2, (unsigned long long)xm);
    atomicMax(o + 3, (unsigned long long)ym);
    if (badp) atomicOr(o + 4, 1ull);
  }
}

__global__ void k_stats_init(int64_t* out) {
  out[0] = (int64_t)~0ull; out[1] = 0; out[2] = 0; out[3] = 0; out[4] = 0;
}
__global__ void k_stats_fini(int64_t* out) {
  out[0] = (int64_t)((uint64_t)out[0] ^ 0x8000000000000000ull);
  out[1] = (int64_t)((uint64_t)out[1] ^ 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256) k_pack(int64_t n, const int64_t* __restrict__ t,
                                              const uint16_t* __restrict__ x,
                                              const uint16_t* __restrict__ y,
                                              const int8_t* __restrict__ p, int64_t t_min,
                                              uint64_t* keys, int64_t* meta, uint32_t* hist,
                                              int64_t hist_words) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i0 == 0) { meta[0] = n; meta[1] = t_min; meta[2] = kNoBad; }
  // the workspace may be reused with another layout: clear the histogram region
  for (int64_t i = i0; i < hist_words; i += (int64_t)gridDim.x * blockDim.x) hist[i] = 0;
  for (int64_t i = i0; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)(t[i] - t_min) << kKeyPixBits) | ((uint64_t)y[i] << 17) |
              ((uint64_t)x[i] << 1) | (p[i] > 0 ? 1u : 0u);
}

struct SortLayout {
  int npass, bits, NB;
  int64_t max_tiles;
  size_t ctr, meta, hist, gstart, prefix, status, keysA, keysB, total;
};

bool sort_layout(int64_t n, int64_t t_span, SortLayout* L) {
  if (n < 0 || t_span < 0 || t_span >= (1ll << 31)) return false;
  int tbits = ilog2_ceil((uint64_t)t_span + 1);
  int total_bits = kKeyPixBits + tbits;
  L->npass = (total_bits + kMaxDigitBits - 1) / kMaxDigitBits;
  L->bits = (total_bits + L->npass - 1) / L->npass;
  L->NB = 1 << L->bits;
  L->max_tiles = (n + kOrdTile - 1) / kOrdTile;
  size_t off = 0;
  L->ctr = off; off = align_up(off + 64 * 4);
  L->meta = off; off = align_up(off + 8 * 8);
  L->hist = off; off = align_up(off + (size_t)L->npass * kHistReps * L->NB * 4);
  L->gstart = off; off = align_up(off + (size_t)L->NB * 4);
  L->prefix = off; off = align_up(off + 2 * 4);
  L->status = off; off = align_up(off + (size_t)L->max_tiles * L->NB * 8);
  L->keysA = off; off = align_up(off + (size_t)n * 8);
  L->keysB = off; off = align_up(off + (size_t)n * 8);
  L->total = off;
  return true;
}

int sm_count_current() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

extern "C" {

evs_status evs_batch_stats(int64_t n, const int64_t* t, const uint16_t* x, const uint16_t* y,
                           const int8_t* p, int64_t* out5, void* stream) {
  if (n < 0 || !out5) return EVS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_stats_init<<<1, 1, 0, st>>>(out5);
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    k_batch_stats<<<(unsigned)blocks, 256, 0, st>>>(n, t, x, y, p, out5);
  }
  k_stats_fini<<<1, 1, 0, st>>>(out5);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

size_t evs_sort_workspace_bytes(int64_t n, int64_t t_span) {
  SortLayout L;
  if (!sort_layout(n, t_span, &L)) return 0;
  return L.total;
}

evs_status evs_canonical_sort(int64_t n, int64_t* t, uint16_t* x, uint16_t* y, int8_t* p,
                              int64_t t_min, int64_t t_span, uint32_t epoch, void* ws,
                              size_t ws_bytes, void* stream) {
  SortLayout L;
  if (!sort_layout(n, t_span, &L)) return EVS_ERR_UNSUPPORTED;
  if (n == 0) return EVS_OK;
  if (!t || !x || !y || !p) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  if (epoch == 0 || epoch + EVS_EPOCHS_PER_CALL > EVS_EPOCH_LIMIT) return EVS_ERR_ARG;
  if (L.npass + 1 > (int)EVS_EPOCHS_PER_CALL) return EVS_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* meta = at<int64_t>(ws, L.meta);
  uint64_t* kA = at<uint64_t>(ws, L.keysA);
  uint64_t* kB = at<uint64_t>(ws, L.keysB);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_pack<<<(unsigned)blocks, 256, 0, st>>>(n, t, x, y, p, t_min, kA, meta, at<uint32_t>(ws, L.hist),
                                           (int64_t)L.npass * kHistReps * L.NB);
  HistArgs h;
  h.nseg = 1; h.keys = kA; h.seg_stride = n; h.seg_count = meta; h.npass = L.npass; h.pass0 = 0;
  h.bits = L.bits; h.base_shift = 0; h.hist = at<uint32_t>(ws, L.hist);
  if (launch_hist(h, st) != cudaSuccess) return EVS_ERR_CUDA;
  const int sms = sm_count_current();
  for (int pass = 0; pass < L.npass; ++pass) {
    PlanArgs pl;
    memset(&pl, 0, sizeof(pl));
    pl.nseg = 1; pl.cap = n; pl.seg_total = meta; pl.hist = h.hist; pl.npass = L.npass; pl.pass = pass;
    pl.bits = L.bits; pl.gstart = at<uint32_t>(ws, L.gstart);
    pl.seg_tile_prefix = at<uint32_t>(ws, L.prefix); pl.bad = meta + 2; pl.zero_hist = 1;
    if (launch_plan(pl, st) != cudaSuccess) return EVS_ERR_CUDA;
    OrderArgs o;
    memset(&o, 0, sizeof(o));
    o.nseg = 1; o.keys_in = (pass % 2 == 0) ? kA : kB; o.keys_out = (pass % 2 == 0) ? kB : kA;
    o.seg_stride = n; o.seg_count = meta; o.seg_tile_prefix = pl.seg_tile_prefix; o.gstart = pl.gstart;
    o.shift = pass * L.bits; o.bits = L.bits; o.status = at<uint64_t>(ws, L.status);
    o.max_tiles = L.max_tiles; o.ctr = at<uint32_t>(ws, L.ctr) + pass; o.epoch = epoch + pass;
    o.final_soa = pass == L.npass - 1; o.out_t = t; o.out_x = x; o.out_y = y; o.out_p = p;
    o.seg_tbase = meta + 1;
    if (launch_order(o, sms, st) != cudaSuccess) return EVS_ERR_CUDA;
  }
  return EVS_OK;
}

}  // extern "C"

namespace {

__device__ __forceinline__ uint64_t ckey(const int64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p,
                                         int64_t i, int64_t tmin) {
  return ((uint64_t)(t[i] - tmin) << kKeyPixBits) | ((uint64_t)y[i] << 17) | ((uint64_t)x[i] << 1) |
         (p[i] > 0 ? 1u : 0u);
}

// B[j] goes to j + upper_bound(A, B[j]); records the split for the A pass
__global__ void __launch_bounds__(256) k_merge_b(int64_t na, const int64_t* at, const uint16_t* ax,
                                                 const uint16_t* ay, const int8_t* ap, int64_t nb,
                                                 const int64_t* bt, const uint16_t* bx, const uint16_t* by,
                                                 const int8_t* bp, int64_t tmin, int64_t* ub, int64_t* ot,
                                                 uint16_t* ox, uint16_t* oy, int8_t* op) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t kb = ckey(bt, bx, by, bp, j, tmin);
    int64_t lo = 0, hi = na;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ckey(at, ax, ay, ap, mid, tmin) <= kb) lo = mid + 1; else hi = mid;
    }
    ub[j] = lo;
    const int64_t o = j + lo;
    ot[o] = bt[j]; ox[o] = bx[j]; oy[o] = by[j]; op[o] = bp[j];
  }
}

// A[i] goes to i + #{j : ub[j] <= i}
__global__ void __launch_bounds__(256) k_merge_a(int64_t na, const int64_t* at, const uint16_t* ax,
                                                 const uint16_t* ay, const int8_t* ap, int64_t nb,
                                                 const int64_t* ub, int64_t* ot, uint16_t* ox, uint16_t* oy,
                                                 int8_t* op) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ub[mid] <= i) lo = mid + 1; else hi = mid;
    }
    const int64_t o = i + lo;
    ot[o] = at[i]; ox[o] = ax[i]; oy[o] = ay[i]; op[o] = ap[i];
  }
}

}  // namespace

extern "C" {

evs_status evs_merge_canonical(int64_t na, const int64_t* at, const uint16_t* ax, const uint16_t* ay,
                               const int8_t* ap, int64_t nb, const int64_t* bt, const uint16_t* bx,
                               const uint16_t* by, const int8_t* bp, int64_t t_min, int64_t* out_t,
                               uint16_t* out_x, uint16_t* out_y, int8_t* out_p, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (na < 0 || nb < 0) return EVS_ERR_ARG;
  if (nb > 0 && (!workspace || workspace_bytes < (size_t)nb * 8)) return EVS_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* ub = static_cast<int64_t*>(workspace);
  auto grid = [](int64_t n) { int64_t b = (n + 255) / 256; return (unsigned)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b)); };
  if (nb > 0)
    k_merge_b<<<grid(nb), 256, 0, st>>>(na, at, ax, ay, ap, nb, bt, bx, by, bp, t_min, ub, out_t, out_x, out_y, out_p);
  if (na > 0) k_merge_a<<<grid(na), 256, 0, st>>>(na, at, ax, ay, ap, nb, ub, out_t, out_x, out_y, out_p);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

// numpy SeedSequence(entropy).generate_state(4, uint64) + PCG64 srandom_r.
void evs_seed_pcg64(const uint32_t* words, int32_t nwords, uint64_t out[4]) {
  struct Hasher {
    uint32_t c;
    uint32_t operator()(uint32_t v) {
      v ^= c;
      c *= 0x931e8875u;
      v *= c;
      return v ^ (v >> 16);
    }
  } hm{0x43b0d7e5u};
  auto mix = [](uint32_t a, uint32_t b) {
    uint32_t r = 0xca01f9ddu * a - 0x4973f715u * b;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hm(i < nwords ? words[i] : 0u);
  for (int src = 0; src < 4; ++src)
    for (int dst = 0; dst < 4; ++dst)
      if (src != dst) pool[dst] = mix(pool[dst], hm(pool[src]));
  for (int src = 4; src < nwords; ++src)
    for (int dst = 0; dst < 4; ++dst) pool[dst] = mix(pool[dst], hm(words[src]));
  uint32_t c = 0x8b51f9ddu, w32[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ c;
    c *= 0x58f38dedu;
    v *= c;
    w32[i] = v ^ (v >> 16);
  }
  typedef unsigned __int128 u128;
  const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  const u128 initstate = ((u128)(((uint64_t)w32[1] << 32) | w32[0]) << 64) | (((uint64_t)w32[3] << 32) | w32[2]);
  const u128 initseq = ((u128)(((uint64_t)w32[5] << 32) | w32[4]) << 64) | (((uint64_t)w32[7] << 32) | w32[6]);
  const u128 inc = (initseq << 1) | 1u;
  u128 s = inc;  // state 0 stepped once: 0 * mult + inc
  s += initstate;
  s = s * mult + inc;
  out[0] = (uint64_t)(s >> 64); out[1] = (uint64_t)s;
  out[2] = (uint64_t)(inc >> 64); out[3] = (uint64_t)inc;
}

}  // extern "C"
