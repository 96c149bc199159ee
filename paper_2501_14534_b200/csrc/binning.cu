// binning.cu — tile binning and the (tile | depth | index) sort (R5).
//
// Reference: bin_tiles (rasterizer.py:95-148) emits one instance per covered
// tile (row-major within the Gaussian's rect), then np.lexsort((gid, depth,
// tile)) and a bincount/cumsum for the CSR offsets.
//
// B200 design: a stable LSD radix sort of the key
//     tile << 64 | orderable(float64 depth)
// whose value is the Gaussian index (the north star's 64-bit tile|depth key with
// the depth widened to float64 so ties break exactly like the reference's float64
// lexsort).  Because every instance of a Gaussian carries the same depth, the
// eight 8-bit depth passes commute with duplication: they run over the M
// on-screen GAUSSIANS (M <= n items) instead of the I instances (I = 27*n at c3),
// and only the ceil(log2 tiles) tile bits are sorted at instance granularity
// (2 passes at 1080p).  Stability of every pass plus
// index-ordered emission gives exactly lexsort's (tile, depth, index) order,
// bit-identical to the oracle.
//
// Pass kernels are reduce-then-scan (histogram, device scan of the digit x block
// matrix, rank + scatter).  Ranking inside a block is warp-synchronous multisplit
// with __match_any_sync, then a shared-memory reorder so the scatter writes
// contiguous runs per digit.  Item counts may live on the device (grids are
// sized for the capacity; blocks past the live count do nothing) so nothing
// here needs a host round trip except the one instance count the caller reads
// between tgs_bin_gaussians and tgs_bin_instances.
#include "tgs_common.cuh"
#include "tgs_math.cuh"

namespace tgs {

constexpr int kBlock = 256;
constexpr int kIPT = 16;
constexpr int kTile = kBlock * kIPT;  // 4096 items per block
constexpr int kWarps = kBlock / 32;

__device__ __forceinline__ uint32_t live_count(const uint32_t *nd, uint32_t nh) { return nd ? *nd : nh; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of one value per thread across the block; returns the block total via *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *warp_sums, uint32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  const uint32_t warp_off = warp ? warp_sums[warp - 1] : 0u;
  if (total) *total = warp_sums[nw - 1];
  const uint32_t res = warp_off + x - v;
  __syncthreads();
  return res;
}

// ---------------------------------------------------------------- scan (u32)
__global__ void __launch_bounds__(kBlock) k_scan_reduce(const uint32_t *__restrict__ in, uint32_t nh,
                                                        const uint32_t *nd, uint32_t *__restrict__ partials) {
  __shared__ uint32_t ws[32];
  const uint32_t n = live_count(nd, nh);
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  uint32_t s = 0;
  if (base < n) {
    const uint32_t end = (uint32_t)tmin<uint64_t>(base + kTile, n);
    for (uint32_t j = (uint32_t)base + threadIdx.x; j < end; j += kBlock) s += in[j];
  }
  uint32_t tot;
  block_exclusive_scan(s, ws, &tot);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_partials(uint32_t *partials, int nb, uint32_t *total_u32,
                                                        int64_t *total_i64) {
  __shared__ uint32_t ws[32];
  uint32_t carry = 0;
  for (int c = 0; c < nb; c += 1024) {
    const int j = c + threadIdx.x;
    const uint32_t v = j < nb ? partials[j] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(v, ws, &tot);
    if (j < nb) partials[j] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (total_u32) *total_u32 = carry;
    if (total_i64) *total_i64 = (int64_t)carry;
  }
}

__global__ void __launch_bounds__(kBlock) k_scan_down(const uint32_t *in, uint32_t *out, uint32_t nh,
                                                      const uint32_t *nd, const uint32_t *__restrict__ partials) {
  __shared__ uint32_t tile[kTile];
  __shared__ uint32_t ws[32];
  const uint32_t n = live_count(nd, nh);
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  if (base >= n) return;
  const uint32_t cnt = (uint32_t)tmin<uint64_t>(kTile, n - base);
  for (uint32_t j = threadIdx.x; j < kTile; j += kBlock) tile[j] = j < cnt ? in[base + j] : 0u;
  __syncthreads();
  uint32_t local[kIPT], s = 0;
#pragma unroll
  for (int k = 0; k < kIPT; ++k) {
    local[k] = tile[threadIdx.x * kIPT + k];
    s += local[k];
  }
  uint32_t run = block_exclusive_scan(s, ws, nullptr) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kIPT; ++k) {
    tile[threadIdx.x * kIPT + k] = run;
    run += local[k];
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += kBlock) out[base + j] = tile[j];
}

struct ScanPlan {
  int nb;
  uint32_t *partials;
};

inline size_t scan_ws_bytes(uint64_t cap) { return align_up((ceil_div<uint64_t>(cap, kTile) + 1) * 4); }

// In-place capable exclusive scan of `cap` (host) or *nd (device, <= cap) items.
inline void device_scan(const uint32_t *in, uint32_t *out, uint64_t cap, const uint32_t *nd, uint32_t *partials,
                        uint32_t *total_u32, int64_t *total_i64, cudaStream_t st) {
  const int nb = (int)ceil_div<uint64_t>(cap, kTile);
  if (nb == 0) {
    k_scan_partials<<<1, 1024, 0, st>>>(partials, 0, total_u32, total_i64);
    return;
  }
  k_scan_reduce<<<nb, kBlock, 0, st>>>(in, (uint32_t)cap, nd, partials);
  k_scan_partials<<<1, 1024, 0, st>>>(partials, nb, total_u32, total_i64);
  k_scan_down<<<nb, kBlock, 0, st>>>(in, out, (uint32_t)cap, nd, partials);
}

// ------------------------------------------------------------ radix passes
// Stable LSD pass over digit [shift, shift+nbits) of K-typed keys (uint32 or
// uint64) with one uint32 payload.  IPT items per thread (tile = 256*IPT).
template <typename K, int IPT>
__global__ void __launch_bounds__(kBlock) k_radix_hist(const K *__restrict__ keys, uint32_t nh,
                                                       const uint32_t *nd, int shift, int nbits,
                                                       uint32_t *__restrict__ hist, int nblocks) {
  constexpr int TILE = kBlock * IPT;
  __shared__ uint32_t h[256];
  const int bins = 1 << nbits;
  const uint32_t mask = bins - 1;
  for (int d = threadIdx.x; d < bins; d += kBlock) h[d] = 0;
  __syncthreads();
  const uint32_t n = live_count(nd, nh);
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  if (base < n) {
#pragma unroll 4
    for (int r = 0; r < IPT; ++r) {
      const uint64_t j = base + (uint64_t)r * kBlock + threadIdx.x;
      const bool ok = j < n;
      const uint32_t okmask = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const uint32_t d = (uint32_t)(keys[j] >> shift) & mask;
        // warp-aggregated shared atomics: one add per distinct digit per warp
        const uint32_t peers = __match_any_sync(okmask, d);
        if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[d], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += kBlock) hist[(size_t)d * nblocks + blockIdx.x] = h[d];
}

template <typename K, int IPT>
__global__ void __launch_bounds__(kBlock) k_radix_scatter(const K *__restrict__ keys_in,
                                                          const uint32_t *__restrict__ vals_in,
                                                          K *__restrict__ keys_out,
                                                          uint32_t *__restrict__ vals_out, uint32_t nh,
                                                          const uint32_t *nd, int shift, int nbits,
                                                          const uint32_t *__restrict__ hist_scanned, int nblocks) {
  constexpr int TILE = kBlock * IPT;
  __shared__ K ks[TILE];
  __shared__ uint32_t vs[TILE];
  __shared__ uint32_t wcnt[kWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t gbase[256];
  __shared__ uint32_t wsum[32];
  const uint32_t n = live_count(nd, nh);
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  if (base >= n) return;
  const int bins = 1 << nbits;
  const uint32_t mask = bins - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < kWarps * 256; j += kBlock) (&wcnt[0][0])[j] = 0;
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  K key[IPT];
  uint32_t val[IPT];
  uint16_t rank[IPT];
  const uint64_t wbase = base + (uint64_t)warp * (IPT * 32);
  // warp-synchronous multisplit: ranks are stable in index order (warp-major,
  // then round, then lane), matching the block's item order
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint64_t j = wbase + r * 32 + lane;
    const bool ok = j < n;
    key[r] = ok ? keys_in[j] : (K)0;
    val[r] = ok ? vals_in[j] : 0u;
    const uint32_t okmask = __ballot_sync(0xffffffffu, ok);
    rank[r] = 0;
    if (ok) {
      const uint32_t d = (uint32_t)(key[r] >> shift) & mask;
      const uint32_t peers = __match_any_sync(okmask, d);
      const uint32_t prev = wcnt[warp][d];
      rank[r] = (uint16_t)(prev + __popc(peers & lt));
      __syncwarp(okmask);
      if (lane == __ffs(peers) - 1) wcnt[warp][d] = prev + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per-digit exclusive prefix over warps, then over digits (block-local start)
  uint32_t dtotal = 0;
  if (threadIdx.x < (unsigned)bins) {
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = dtotal;
      dtotal += c;
    }
  }
  const uint32_t ds = block_exclusive_scan(threadIdx.x < (unsigned)bins ? dtotal : 0u, wsum, nullptr);
  if (threadIdx.x < (unsigned)bins) {
    dstart[threadIdx.x] = ds;
    gbase[threadIdx.x] = hist_scanned[(size_t)threadIdx.x * nblocks + blockIdx.x];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint64_t j = wbase + r * 32 + lane;
    if (j < n) {
      const uint32_t d = (uint32_t)(key[r] >> shift) & mask;
      const uint32_t p = dstart[d] + wcnt[warp][d] + rank[r];
      ks[p] = key[r];
      vs[p] = val[r];
    }
  }
  __syncthreads();
  // contiguous runs per digit -> coalesced scatter
  const uint32_t cnt = (uint32_t)tmin<uint64_t>(TILE, n - base);
  for (uint32_t j = threadIdx.x; j < cnt; j += kBlock) {
    const K k = ks[j];
    const uint32_t d = (uint32_t)(k >> shift) & mask;
    const uint32_t o = gbase[d] + (j - dstart[d]);
    if (keys_out) keys_out[o] = k;
    vals_out[o] = vs[j];
  }
}

struct RadixScratch {
  uint32_t *hist;      // 256 * nblocks
  uint32_t *partials;  // scan partials for hist
};

template <typename K>
constexpr int ipt_for() {
  return sizeof(K) == 8 ? 8 : kIPT;  // 64-bit keys: 2048-item tiles keep smem at 24 KB + counters
}

template <typename K>
inline uint64_t radix_blocks(uint64_t cap) {
  return ceil_div<uint64_t>(cap, (uint64_t)kBlock * ipt_for<K>());
}

// One stable pass over digit [shift, shift+nbits).
template <typename K>
inline void radix_pass(const K *kin, const uint32_t *vin, K *kout, uint32_t *vout, uint64_t cap, const uint32_t *nd,
                       int shift, int nbits, RadixScratch sc, cudaStream_t st) {
  constexpr int IPT = ipt_for<K>();
  const int nb = (int)radix_blocks<K>(cap);
  if (nb == 0) return;
  k_radix_hist<K, IPT><<<nb, kBlock, 0, st>>>(kin, (uint32_t)cap, nd, shift, nbits, sc.hist, nb);
  device_scan(sc.hist, sc.hist, (uint64_t)(1 << nbits) * nb, nullptr, sc.partials, nullptr, nullptr, st);
  k_radix_scatter<K, IPT><<<nb, kBlock, 0, st>>>(kin, vin, kout, vout, (uint32_t)cap, nd, shift, nbits, sc.hist,
                                                 nb);
}

// ------------------------------------------------------- Gaussian stage
struct Band {
  int W, H, ts, tiles_x, tiles_y, row_begin, row_end;
};

// Band-restricted tile count of Gaussian i (0 when off-screen / not visible).
__device__ __forceinline__ int band_rect(const float *sp, const Band &b, int &x0, int &y0, int &x1, int &y1) {
  const float4 a = reinterpret_cast<const float4 *>(sp)[0];
  const float4 c = reinterpret_cast<const float4 *>(sp)[2];
  const int n = tile_rect(a.x, a.y, c.z, b.W, b.H, b.ts, b.tiles_x, b.tiles_y, x0, y0, x1, y1);
  if (n == 0) return 0;
  y0 = max(y0, b.row_begin);
  y1 = min(y1, b.row_end - 1);
  return y1 >= y0 ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0;
}

__global__ void k_select(const float *__restrict__ splats, const int32_t *__restrict__ tiles_touched, int64_t n,
                         Band b, uint32_t *__restrict__ cnt, uint32_t *__restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c = 0;
  if (tiles_touched[i] > 0) {
    int x0, y0, x1, y1;
    c = (uint32_t)band_rect(splats + 12 * i, b, x0, y0, x1, y1);
  }
  cnt[i] = c;
  flag[i] = c > 0;
}

__global__ void k_compact(const float *__restrict__ splats, const uint64_t *__restrict__ depth_keys,
                          const uint32_t *__restrict__ cnt, const uint32_t *__restrict__ pos, int64_t n,
                          uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || cnt[i] == 0) return;
  const uint32_t p = pos[i];
  keys[p] = depth_keys ? depth_keys[i] : orderable_key64((double)splats[12 * i + 9]);
  vals[p] = (uint32_t)i;
}

__global__ void k_gather_counts(const uint32_t *__restrict__ ids, const uint32_t *__restrict__ cnt, int64_t cap,
                                const uint32_t *nd, uint32_t *__restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap || j >= (int64_t)*nd) return;
  out[j] = cnt[ids[j]];
}

// Warp-cooperative expansion: each warp owns 32 depth-ordered Gaussians and
// emits their band tiles row-major with lane-strided, coalesced stores.
__global__ void k_duplicate(const float *__restrict__ splats, const uint32_t *__restrict__ ids,
                            const uint32_t *__restrict__ inst_off, int64_t cap, const uint32_t *nd, Band b,
                            uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = *nd;
  const int lane = threadIdx.x & 31;
  int x0 = 0, y0 = 0, x1 = -1, y1 = -1, cnt = 0;
  uint32_t g = 0, off = 0;
  if (j < m && j < cap) {
    g = ids[j];
    off = inst_off[j];
    cnt = band_rect(splats + 12 * (int64_t)g, b, x0, y0, x1, y1);
  }
  const uint32_t base_tile = (uint32_t)b.row_begin * b.tiles_x;
  uint32_t todo = __ballot_sync(0xffffffffu, cnt > 0);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int sc = __shfl_sync(0xffffffffu, cnt, src);
    const int sx0 = __shfl_sync(0xffffffffu, x0, src);
    const int sy0 = __shfl_sync(0xffffffffu, y0, src);
    const int snx = __shfl_sync(0xffffffffu, x1 - x0 + 1, src);
    const uint32_t sg = __shfl_sync(0xffffffffu, g, src);
    const uint32_t so = __shfl_sync(0xffffffffu, off, src);
    for (int e = lane; e < sc; e += 32) {
      const int row = e / snx, col = e - row * snx;
      keys[so + e] = (uint32_t)(sy0 + row) * b.tiles_x + (uint32_t)(sx0 + col) - base_tile;
      vals[so + e] = sg;
    }
  }
}

// CSR offsets from sorted tile keys (the reference's bincount + cumsum).
__global__ void k_ranges(const uint32_t *__restrict__ keys, int64_t count, uint32_t ntiles,
                         int32_t *__restrict__ offsets) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  const uint32_t k = keys[j];
  const int64_t prev = j > 0 ? (int64_t)keys[j - 1] : -1;
  for (int64_t t = prev + 1; t <= (int64_t)k; ++t) offsets[t] = (int32_t)j;
  if (j == count - 1)
    for (int64_t t = (int64_t)k + 1; t <= (int64_t)ntiles; ++t) offsets[t] = (int32_t)count;
}

__global__ void k_row_hist(const float *__restrict__ splats, const int32_t *__restrict__ tiles_touched, int64_t n,
                           Band b, unsigned long long *__restrict__ rows) {
  extern __shared__ unsigned long long sh[];
  const bool use_sh = b.tiles_y <= 2048;
  if (use_sh)
    for (int r = threadIdx.x; r < b.tiles_y; r += blockDim.x) sh[r] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && tiles_touched[i] > 0) {
    int x0, y0, x1, y1;
    if (band_rect(splats + 12 * i, b, x0, y0, x1, y1) > 0)
      for (int y = y0; y <= y1; ++y) atomicAdd(use_sh ? &sh[y] : &rows[y], (unsigned long long)(x1 - x0 + 1));
  }
  __syncthreads();
  if (use_sh)
    for (int r = threadIdx.x; r < b.tiles_y; r += blockDim.x)
      if (sh[r]) atomicAdd(&rows[r], sh[r]);
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) p[j] = v;
}

// Gaussian-stage workspace (persists into the instance stage)
struct GaussWS {
  uint32_t *cnt, *pos, *valsA, *valsB, *inst_off, *m, *partials;
  uint64_t *keysA, *keysB;
  RadixScratch rs;
  size_t bytes;
};

inline GaussWS carve_gauss(void *p, int64_t n) {
  Carve c(p);
  GaussWS w;
  const size_t N = (size_t)tmax<int64_t>(n, 1);
  w.cnt = c.take<uint32_t>(N);
  w.pos = c.take<uint32_t>(N);
  w.keysA = c.take<uint64_t>(N);
  w.valsA = c.take<uint32_t>(N);
  w.keysB = c.take<uint64_t>(N);
  w.valsB = c.take<uint32_t>(N);
  w.inst_off = c.take<uint32_t>(N);
  w.m = c.take<uint32_t>(4);
  w.partials = c.take<uint32_t>(scan_ws_bytes(N) / 4);
  const uint64_t nb = radix_blocks<uint64_t>(N);
  w.rs.hist = c.take<uint32_t>(256 * nb);
  w.rs.partials = c.take<uint32_t>(scan_ws_bytes(256 * nb) / 4);
  w.bytes = c.off;
  return w;
}

inline int key_bits(uint32_t ntiles) {
  int bits = 0;
  while (bits < 32 && (1ull << bits) < ntiles) ++bits;
  return bits;
}

inline bool band_ok(int W, int H, int ts, int rb, int re, Band &b) {
  if (W < 1 || H < 1 || ts < 1) return false;
  b.W = W; b.H = H; b.ts = ts;
  b.tiles_x = (W + ts - 1) / ts;
  b.tiles_y = (H + ts - 1) / ts;
  b.row_begin = rb;
  b.row_end = re;
  return rb >= 0 && re <= b.tiles_y && rb < re;
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_bin_gaussians_workspace(int64_t n, size_t *bytes) {
  if (n < 0 || !bytes) return TGS_ERR_INVALID;
  *bytes = carve_gauss(nullptr, n).bytes;
  return TGS_OK;
}

extern "C" int tgs_bin_gaussians(const float *splats, const int32_t *tiles_touched, const uint64_t *depth_keys,
                                 int64_t n, int32_t width,
                                 int32_t height, int32_t tile_size, int32_t row_begin, int32_t row_end,
                                 void *workspace, int64_t *d_num_instances, tgs_stream_t stream) {
  Band b;
  if (n < 0 || n >= (int64_t)1 << 31 || !workspace || !d_num_instances ||
      !band_ok(width, height, tile_size, row_begin, row_end, b))
    return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  GaussWS w = carve_gauss(workspace, n);
  if (n == 0) {
    cudaMemsetAsync(w.m, 0, 4, st);
    cudaMemsetAsync(d_num_instances, 0, 8, st);
    return launch_status();
  }
  const unsigned g256 = (unsigned)ceil_div<int64_t>(n, 256);
  k_select<<<g256, 256, 0, st>>>(splats, tiles_touched, n, b, w.cnt, w.pos);
  device_scan(w.pos, w.pos, (uint64_t)n, nullptr, w.partials, w.m, nullptr, st);
  k_compact<<<g256, 256, 0, st>>>(splats, depth_keys, w.cnt, w.pos, n, w.keysA, w.valsA);
  // depth digits: 8 stable 8-bit passes over the M selected Gaussians (float64 keys)
  for (int p = 0; p < 8; p += 2) {
    radix_pass<uint64_t>(w.keysA, w.valsA, w.keysB, w.valsB, (uint64_t)n, w.m, 8 * p, 8, w.rs, st);
    radix_pass<uint64_t>(w.keysB, w.valsB, w.keysA, w.valsA, (uint64_t)n, w.m, 8 * p + 8, 8, w.rs, st);
  }
  // depth-ordered ids are in valsA; per-Gaussian instance offsets in depth order
  k_gather_counts<<<g256, 256, 0, st>>>(w.valsA, w.cnt, n, w.m, w.inst_off);
  device_scan(w.inst_off, w.inst_off, (uint64_t)n, w.m, w.partials, nullptr, d_num_instances, st);
  return launch_status();
}

struct InstWS {
  uint32_t *keysA, *keysB, *valsB;
  RadixScratch rs;
  size_t bytes;
};

static InstWS carve_inst(void *p, int64_t count) {
  Carve c(p);
  InstWS w;
  const size_t I = (size_t)tmax<int64_t>(count, 1);
  w.keysA = c.take<uint32_t>(I);
  w.keysB = c.take<uint32_t>(I);
  w.valsB = c.take<uint32_t>(I);
  const uint64_t nb = radix_blocks<uint32_t>(I);
  w.rs.hist = c.take<uint32_t>(256 * nb);
  w.rs.partials = c.take<uint32_t>(scan_ws_bytes(256 * nb) / 4);
  w.bytes = c.off;
  return w;
}

extern "C" int tgs_bin_instances_workspace(int64_t n, int64_t num_instances, size_t *bytes) {
  if (n < 0 || num_instances < 0 || !bytes) return TGS_ERR_INVALID;
  *bytes = carve_inst(nullptr, num_instances).bytes;
  return TGS_OK;
}

extern "C" int tgs_bin_instances(const float *splats, int64_t n, int32_t width, int32_t height, int32_t tile_size,
                                 int32_t row_begin, int32_t row_end, void *gauss_workspace, int64_t num_instances,
                                 void *workspace, int32_t *tile_offsets, int32_t *sorted_ids, tgs_stream_t stream) {
  Band b;
  if (n < 0 || num_instances < 0 || num_instances >= (int64_t)1 << 31 || !gauss_workspace || !tile_offsets ||
      !band_ok(width, height, tile_size, row_begin, row_end, b))
    return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  const uint32_t ntiles = (uint32_t)(b.row_end - b.row_begin) * b.tiles_x;
  if (num_instances == 0) {
    k_fill_i32<<<(unsigned)ceil_div<int64_t>(ntiles + 1, 256), 256, 0, st>>>(tile_offsets, ntiles + 1, 0);
    return launch_status();
  }
  if (!workspace || !sorted_ids) return TGS_ERR_INVALID;
  GaussWS gw = carve_gauss(gauss_workspace, n);
  InstWS w = carve_inst(workspace, num_instances);
  const int bits = key_bits(ntiles);
  const int passes = (bits + 7) / 8;
  const int per = passes ? (bits + passes - 1) / passes : 0;
  // ping-pong so the last pass lands in sorted_ids
  uint32_t *vdst = (passes % 2 == 0) ? reinterpret_cast<uint32_t *>(sorted_ids) : w.valsB;
  k_duplicate<<<(unsigned)ceil_div<int64_t>(n, 256), 256, 0, st>>>(splats, gw.valsA, gw.inst_off, n, gw.m, b,
                                                                    w.keysA, vdst);
  uint32_t *kin = w.keysA, *vin = vdst;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * per;
    const int nb = min(per, bits - shift);
    uint32_t *kout = (kin == w.keysA) ? w.keysB : w.keysA;
    uint32_t *vout = (vin == w.valsB) ? reinterpret_cast<uint32_t *>(sorted_ids) : w.valsB;
    radix_pass<uint32_t>(kin, vin, kout, vout, (uint64_t)num_instances, nullptr, shift, nb, w.rs, st);
    kin = kout;
    vin = vout;
  }
  k_ranges<<<(unsigned)ceil_div<int64_t>(num_instances, 256), 256, 0, st>>>(kin, num_instances, ntiles,
                                                                           tile_offsets);
  return launch_status();
}

extern "C" int tgs_row_histogram(const float *splats, const int32_t *tiles_touched, int64_t n, int32_t width,
                                 int32_t height, int32_t tile_size, int64_t *row_counts, tgs_stream_t stream) {
  Band b;
  if (n < 0 || !row_counts) return TGS_ERR_INVALID;
  if (!band_ok(width, height, tile_size, 0, (height + tile_size - 1) / tile_size, b)) return TGS_ERR_INVALID;
  if (n == 0) return TGS_OK;
  const size_t sh = b.tiles_y <= 2048 ? (size_t)b.tiles_y * 8 : 0;
  k_row_hist<<<(unsigned)ceil_div<int64_t>(n, 256), 256, sh, as_stream(stream)>>>(
      splats, tiles_touched, n, b, reinterpret_cast<unsigned long long *>(row_counts));
  return launch_status();
}
