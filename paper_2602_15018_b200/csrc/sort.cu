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
  size_t permA, permB, soa;  // general path only
};

bool sort_layout_bits(int64_t n, int total_bits, SortLayout* L) {
  if (n < 0 || total_bits < 1 || total_bits > 64) return false;
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
  L->permA = L->permB = L->soa = 0;
  L->total = off;
  return true;
}

bool sort_layout(int64_t n, int64_t t_span, SortLayout* L) {
  if (n < 0 || t_span < 0 || t_span >= (1ll << 31)) return false;
  return sort_layout_bits(n, kKeyPixBits + ilog2_ceil((uint64_t)t_span + 1), L);
}

// General canonical_sort (any uint64 t, any int8 polarity): four stable LSD
// passes over 32-bit digits (polarity, then (y, x), then t's low and high
// words), each a full sort of 64-bit keys digit << 32 | previous position.
bool sort_layout_general(int64_t n, SortLayout* L) {
  if (n < 0 || n >= (1ll << 32)) return false;
  if (!sort_layout_bits(n, 64, L)) return false;
  size_t off = L->total;
  L->permA = off; off = align_up(off + (size_t)n * 4);
  L->permB = off; off = align_up(off + (size_t)n * 4);
  L->soa = off; off = align_up(off + (size_t)n * 13);
  L->total = off;
  return true;
}

// key of element e for LSD pass `which` (0: polarity, 1: (y, x), 2: t low word,
// 3: t high word); r = its position in the order sorted so far
__device__ __forceinline__ uint64_t general_digit(int which, const int64_t* t, const uint16_t* x,
                                                  const uint16_t* y, const int8_t* p, int64_t e) {
  switch (which) {
    case 0: return (uint64_t)((uint8_t)p[e] ^ 0x80u);  // int8 order as unsigned
    case 1: return ((uint64_t)y[e] << 16) | x[e];
    case 2: return (uint64_t)t[e] & 0xffffffffull;     // t as uint64 (parallel.py:116)
    default: return (uint64_t)t[e] >> 32;
  }
}

__global__ void __launch_bounds__(256) k_general_keys(int64_t n, int which, const uint32_t* perm,
                                                      const int64_t* t, const uint16_t* x, const uint16_t* y,
                                                      const int8_t* p, uint64_t* keys) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = perm ? (int64_t)perm[r] : r;
    keys[r] = (general_digit(which, t, x, y, p, e) << 32) | (uint64_t)r;
  }
}

// after a pass: the element now at position r2 was at position (key & 0xffffffff)
__global__ void __launch_bounds__(256) k_general_perm(int64_t n, const uint64_t* sorted, const uint32_t* perm_old,
                                                      uint32_t* perm_new) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t prev = (uint32_t)sorted[r];
    perm_new[r] = perm_old ? perm_old[prev] : prev;
  }
}

__global__ void __launch_bounds__(256) k_general_gather(int64_t n, const uint32_t* perm, const int64_t* ti,
                                                        const uint16_t* xi, const uint16_t* yi, const int8_t* pi,
                                                        int64_t* t, uint16_t* x, uint16_t* y, int8_t* p) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = perm[r];
    t[r] = ti[e]; x[r] = xi[e]; y[r] = yi[e]; p[r] = pi[e];
  }
}

// Full sort of n 64-bit keys in kA (low `bits` bits significant); returns the
// buffer holding the result (kA or kB).  The status words are cleared first,
// so any epochs >= 1 are fresh.
cudaError_t sort_keys64(int64_t n, int total_bits, void* ws, const SortLayout& L, int64_t* meta, uint64_t* kA,
                        uint64_t* kB, uint64_t** result, cudaStream_t st);

int sm_count_current() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

cudaError_t sort_keys64(int64_t n, int total_bits, void* ws, const SortLayout& L, int64_t* meta, uint64_t* kA,
                        uint64_t* kB, uint64_t** result, cudaStream_t st) {
  const int npass = (total_bits + L.bits - 1) / L.bits;
  cudaMemsetAsync(at<uint32_t>(ws, L.hist), 0, (size_t)L.npass * kHistReps * L.NB * 4, st);
  cudaMemsetAsync(at<uint64_t>(ws, L.status), 0, (size_t)L.max_tiles * L.NB * 8, st);
  HistArgs h;
  h.nseg = 1; h.keys = kA; h.seg_stride = n; h.seg_count = meta; h.npass = npass; h.pass0 = 0;
  h.bits = L.bits; h.base_shift = 0; h.hist = at<uint32_t>(ws, L.hist);
  cudaError_t e = launch_hist(h, st);
  if (e != cudaSuccess) return e;
  const int sms = sm_count_current();
  for (int pass = 0; pass < npass; ++pass) {
    PlanArgs pl;
    memset(&pl, 0, sizeof(pl));
    pl.nseg = 1; pl.cap = n; pl.seg_total = meta; pl.hist = h.hist; pl.npass = npass; pl.pass = pass;
    pl.bits = L.bits; pl.gstart = at<uint32_t>(ws, L.gstart);
    pl.seg_tile_prefix = at<uint32_t>(ws, L.prefix); pl.bad = meta + 2; pl.zero_hist = 1;
    if ((e = launch_plan(pl, st)) != cudaSuccess) return e;
    OrderArgs o;
    memset(&o, 0, sizeof(o));
    o.nseg = 1; o.keys_in = (pass % 2 == 0) ? kA : kB; o.keys_out = (pass % 2 == 0) ? kB : kA;
    o.seg_stride = n; o.seg_count = meta; o.seg_tile_prefix = pl.seg_tile_prefix; o.gstart = pl.gstart;
    o.shift = pass * L.bits; o.bits = L.bits; o.status = at<uint64_t>(ws, L.status);
    o.max_tiles = L.max_tiles; o.ctr = at<uint32_t>(ws, L.ctr) + pass; o.epoch = 1 + pass;
    o.final_soa = 0;
    if ((e = launch_order(o, sms, st)) != cudaSuccess) return e;
  }
  *result = (npass % 2 == 0) ? kA : kB;
  return cudaSuccess;
}

__global__ void k_general_meta(int64_t* meta, int64_t n) { meta[0] = n; meta[1] = 0; meta[2] = kNoBad; }

}  // namespace

extern "C" {

size_t evs_sort_general_workspace_bytes(int64_t n) {
  SortLayout L;
  if (!sort_layout_general(n, &L)) return 0;
  return L.total;
}

evs_status evs_canonical_sort_general(int64_t n, int64_t* t, uint16_t* x, uint16_t* y, int8_t* p, void* ws,
                                      size_t ws_bytes, void* stream) {
  SortLayout L;
  if (!sort_layout_general(n, &L)) return EVS_ERR_UNSUPPORTED;
  if (n == 0) return EVS_OK;
  if (!t || !x || !y || !p) return EVS_ERR_ARG;
  if (!ws || ws_bytes < L.total) return EVS_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* meta = at<int64_t>(ws, L.meta);
  uint64_t* kA = at<uint64_t>(ws, L.keysA);
  uint64_t* kB = at<uint64_t>(ws, L.keysB);
  uint32_t* perm[2] = {at<uint32_t>(ws, L.permA), at<uint32_t>(ws, L.permB)};
  char* soa = at<char>(ws, L.soa);
  int64_t* t0 = reinterpret_cast<int64_t*>(soa);
  uint16_t* x0 = reinterpret_cast<uint16_t*>(soa + (size_t)n * 8);
  uint16_t* y0 = x0 + n;
  int8_t* p0 = reinterpret_cast<int8_t*>(y0 + n);
  cudaMemcpyAsync(t0, t, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(x0, x, (size_t)n * 2, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(y0, y, (size_t)n * 2, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(p0, p, (size_t)n, cudaMemcpyDeviceToDevice, st);
  k_general_meta<<<1, 1, 0, st>>>(meta, n);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const uint32_t* cur = nullptr;  // identity
  int which_buf = 0;
  static const int kBits[4] = {40, 64, 64, 64};  // digit bits + 32 position bits
  for (int which = 0; which < 4; ++which) {
    k_general_keys<<<(unsigned)blocks, 256, 0, st>>>(n, which, cur, t0, x0, y0, p0, kA);
    uint64_t* sorted = nullptr;
    if (sort_keys64(n, kBits[which], ws, L, meta, kA, kB, &sorted, st) != cudaSuccess) return EVS_ERR_CUDA;
    k_general_perm<<<(unsigned)blocks, 256, 0, st>>>(n, sorted, cur, perm[which_buf]);
    cur = perm[which_buf];
    which_buf ^= 1;
  }
  k_general_gather<<<(unsigned)blocks, 256, 0, st>>>(n, cur, t0, x0, y0, p0, t, x, y, p);
  return cudaGetLastError() == cudaSuccess ? EVS_OK : EVS_ERR_CUDA;
}

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

}  // extern "C"

namespace {

// k-way stable merge of sorted runs of int64 keys (row bands of one sensor,
// bands.py): key i of run b goes to (i - start_b) + #keys <= it in runs before
// b + #keys < it in runs after b (binary searches; ties keep run order).
constexpr int kMaxRuns = 64;
__global__ void __launch_bounds__(256) k_merge_runs(int nruns, const int64_t* __restrict__ offs,
                                                    const int64_t* __restrict__ in, int64_t* __restrict__ out) {
  __shared__ int64_t s_off[kMaxRuns + 1];
  for (int i = threadIdx.x; i <= nruns; i += blockDim.x) s_off[i] = offs[i];
  __syncthreads();
  const int64_t n = s_off[nruns];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int b = 0;
    while (s_off[b + 1] <= i) ++b;
    const int64_t k = in[i];
    int64_t pos = i - s_off[b];
    for (int r = 0; r < nruns; ++r) {
      if (r == b) continue;
      int64_t lo = s_off[r], hi = s_off[r + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int64_t v = in[mid];
        if (r < b ? v <= k : v < k) lo = mid + 1; else hi = mid;
      }
      pos += lo - s_off[r];
    }
    out[pos] = k;
  }
}

}  // namespace

extern "C" {

evs_status evs_merge_runs(int32_t nruns, const int64_t* run_offsets, int64_t n, const int64_t* keys_in,
                          int64_t* keys_out, void* stream) {
  if (nruns < 1 || nruns > kMaxRuns || n < 0 || !run_offsets) return EVS_ERR_ARG;
  if (n == 0) return EVS_OK;
  if (!keys_in || !keys_out || keys_in == keys_out) return EVS_ERR_ARG;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_merge_runs<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(nruns, run_offsets, keys_in,
                                                                                keys_out);
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
