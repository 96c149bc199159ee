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

// ------------------------------------------------------------ radix sort
// Onesweep-style stable LSD radix sort of (K key, u32 value) pairs:
//   k_sweep_hist  one read of the keys -> global digit histograms of every pass
//   k_sweep_scan  exclusive scan of each pass's 256 bins (one CTA)
//   k_sweep_pass  per pass: tiles taken in launch order from an atomic ticket; a
//                 tile ranks its items (warp multisplit), publishes its per-digit
//                 counts and resolves its global offsets by decoupled look-back
//                 over its predecessors, then scatters through shared memory in
//                 contiguous per-digit runs.
// A tile only ever waits for tiles with smaller tickets, which are already
// resident, so the look-back cannot deadlock.
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

// The status word IS the payload (flag | count in one 32-bit word), so relaxed
// GPU-scope accesses suffice: no acquire fence (which costs an L1 invalidate per
// probe on sm_100) and no release fence.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <typename K>
constexpr int lookback_for() {  // predecessors probed per step (independent loads in flight)
  return sizeof(K) == 8 ? 32 : 16;
}

template <typename K>
constexpr int ipt_for() {
  return sizeof(K) == 8 ? 8 : kIPT;  // 64-bit keys: 2048-item tiles keep smem at 24 KB + counters
}
template <typename K>
constexpr int tile_for() {
  return kBlock * ipt_for<K>();
}

constexpr int kFullHistSmem = 8192;  // full-key histogram bins kept in shared memory

// Digit histograms of every pass in one read of the keys; optionally also the
// full-key histogram (the per-tile instance counts -> CSR offsets, replacing a
// boundary scan over the sorted keys).
template <typename K>
__global__ void __launch_bounds__(kBlock) k_sweep_hist(const K *__restrict__ keys, uint32_t nh, const uint32_t *nd,
                                                       int npasses, int bpp, int total_bits,
                                                       uint32_t *__restrict__ gbins, uint32_t *__restrict__ full_hist,
                                                       int full_bins) {
  __shared__ uint32_t h[8][256];
  __shared__ uint32_t fh[kFullHistSmem];
  const bool fsh = full_hist && full_bins <= kFullHistSmem;
  for (int e = threadIdx.x; e < npasses * 256; e += kBlock) (&h[0][0])[e] = 0;
  if (fsh)
    for (int e = threadIdx.x; e < full_bins; e += kBlock) fh[e] = 0;
  __syncthreads();
  const uint32_t n = live_count(nd, nh);
  for (uint32_t i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    const K k = keys[i];
    for (int p = 0; p < npasses; ++p) {
      const int sh = p * bpp;
      const int nb = min(bpp, total_bits - sh);
      atomicAdd(&h[p][(uint32_t)(k >> sh) & ((1u << nb) - 1)], 1u);
    }
    if (full_hist) atomicAdd(fsh ? &fh[(uint32_t)k] : &full_hist[(uint32_t)k], 1u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < npasses * 256; e += kBlock) {
    const uint32_t v = (&h[0][0])[e];
    if (v) atomicAdd(gbins + e, v);
  }
  if (fsh)
    for (int e = threadIdx.x; e < full_bins; e += kBlock)
      if (fh[e]) atomicAdd(full_hist + e, fh[e]);
}

// CSR offsets (int32, bins + 1) from the full-key histogram: one CTA, chunked scan.
__global__ void __launch_bounds__(1024) k_offsets_from_hist(const uint32_t *__restrict__ hist, int bins,
                                                            int32_t *__restrict__ offsets) {
  __shared__ uint32_t ws[32];
  uint32_t carry = 0;
  for (int c = 0; c < bins; c += 1024) {
    const int j = c + threadIdx.x;
    const uint32_t v = j < bins ? hist[j] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(v, ws, &tot);
    if (j < bins) offsets[j] = (int32_t)(carry + ex);
    carry += tot;
  }
  if (threadIdx.x == 0) offsets[bins] = (int32_t)carry;
}

__global__ void __launch_bounds__(kBlock) k_sweep_scan(uint32_t *gbins, int npasses) {
  __shared__ uint32_t ws[32];
  for (int p = 0; p < npasses; ++p) {
    const uint32_t v = gbins[p * 256 + threadIdx.x];
    const uint32_t ex = block_exclusive_scan(v, ws, nullptr);
    gbins[p * 256 + threadIdx.x] = ex;
  }
}

template <typename K, int IPT>
__global__ void __launch_bounds__(kBlock, 3) k_sweep_pass(const K *__restrict__ keys_in,
                                                       const uint32_t *__restrict__ vals_in,
                                                       K *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
                                                       uint32_t nh, const uint32_t *nd, int shift, int nbits,
                                                       const uint32_t *__restrict__ bin_base,
                                                       uint32_t *__restrict__ status, uint32_t *__restrict__ ticket) {
  constexpr int TILE = kBlock * IPT;
  __shared__ K ks[TILE];
  __shared__ uint32_t vs[TILE];
  __shared__ uint32_t wcnt[kWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t gbase[256];
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t n = live_count(nd, nh);
  const uint64_t base = (uint64_t)tile * TILE;
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
  // then round, then lane), matching the tile's item order
  // all loads first: the multisplit below synchronises the warp every round, and
  // loads cannot be hoisted across those synchronisation points
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint64_t j = wbase + r * 32 + lane;
    const bool ok = j < n;
    key[r] = ok ? keys_in[j] : (K)0;
    val[r] = ok ? vals_in[j] : 0u;
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint64_t j = wbase + r * 32 + lane;
    const bool ok = j < n;
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
    // decoupled look-back over the predecessors' per-digit counts
    uint32_t *mine = status + (size_t)tile * 256 + threadIdx.x;
    uint32_t excl = 0;
    if (tile == 0) {
      st_relaxed(mine, kFlagInc | dtotal);
    } else {
      st_relaxed(mine, kFlagAgg | dtotal);
      int j = (int)tile - 1;
      bool found = false;
      while (!found) {
        constexpr int kLookback = lookback_for<K>();
        uint32_t v[kLookback];
#pragma unroll
        for (int k = 0; k < kLookback; ++k)
          v[k] = (j - k >= 0) ? ld_relaxed(status + (size_t)(j - k) * 256 + threadIdx.x) : kFlagInc;
        int used = 0;
#pragma unroll
        for (int k = 0; k < kLookback; ++k) {
          if (found || (v[k] >> 30) == 0) break;  // stop at the first unpublished predecessor
          excl += v[k] & kValMask;
          found = (v[k] & kFlagInc) != 0;
          ++used;
        }
        j -= found ? 0 : used;  // resume at the first predecessor not yet consumed
      }
      st_relaxed(mine, kFlagInc | (excl + dtotal));
    }
    gbase[threadIdx.x] = bin_base[threadIdx.x] + excl;
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

struct SortScratch {
  uint32_t *gbins;      // passes * 256
  uint32_t *status;     // passes * tiles * 256
  uint32_t *ticket;     // passes
  uint32_t *full_hist;  // full_bins (optional)
  size_t bytes_zeroed;
};

template <typename K>
inline size_t sort_ws_bytes(uint64_t cap, int passes) {
  const uint64_t tiles = ceil_div<uint64_t>(cap, tile_for<K>());
  return align_up((size_t)passes * 256 * 4) + align_up((size_t)passes * tiles * 256 * 4) + align_up(passes * 4);
}

template <typename K>
inline SortScratch carve_sort(Carve &c, uint64_t cap, int passes, size_t full_bins = 0) {
  const uint64_t tiles = ceil_div<uint64_t>(cap, tile_for<K>());
  SortScratch s;
  const size_t off0 = c.off;
  s.gbins = c.take<uint32_t>((size_t)passes * 256);
  s.status = c.take<uint32_t>((size_t)passes * tiles * 256);
  s.ticket = c.take<uint32_t>(passes);
  s.full_hist = full_bins ? c.take<uint32_t>(full_bins) : nullptr;
  s.bytes_zeroed = c.off - off0;
  return s;
}

// Stable sort of `cap` (or *nd) items by bits [0, total_bits) of the key, in
// `passes` passes of <= 8 bits.  Ping-pongs A <-> B; returns true when the
// result ended in the B buffers.
// hist_ready: the caller already wrote the exclusive-scanned digit histograms of
// every pass to sc.gbins (and zeroed the look-back state); last_keys: write the
// keys on the final pass (not needed when the CSR offsets come from a histogram).
template <typename K>
inline bool radix_sort(K *kA, uint32_t *vA, K *kB, uint32_t *vB, uint64_t cap, const uint32_t *nd, int total_bits,
                       SortScratch sc, cudaStream_t st, bool hist_ready = false, bool last_keys = true) {
  const int passes = (total_bits + 7) / 8;
  if (cap == 0 || passes == 0) return false;
  const int bpp = (total_bits + passes - 1) / passes;
  const uint64_t tiles = ceil_div<uint64_t>(cap, tile_for<K>());
  if (!hist_ready) {
    cudaMemsetAsync(sc.gbins, 0, sc.bytes_zeroed, st);
    const unsigned hgrid = (unsigned)tmin<uint64_t>(ceil_div<uint64_t>(cap, kBlock * 16), 148 * 4);
    k_sweep_hist<K><<<hgrid, kBlock, 0, st>>>(kA, (uint32_t)cap, nd, passes, bpp, total_bits, sc.gbins, nullptr, 0);
    k_sweep_scan<<<1, kBlock, 0, st>>>(sc.gbins, passes);
  }
  K *kin = kA, *kout = kB;
  uint32_t *vin = vA, *vout = vB;
  for (int p = 0; p < passes; ++p) {
    const int sh = p * bpp;
    k_sweep_pass<K, ipt_for<K>()><<<(unsigned)tiles, kBlock, 0, st>>>(
        kin, vin, (p == passes - 1 && !last_keys) ? nullptr : kout, vout, (uint32_t)cap, nd, sh,
        min(bpp, total_bits - sh), sc.gbins + p * 256,
        sc.status + (size_t)p * tiles * 256, sc.ticket + p);
    K *tk = kin; kin = kout; kout = tk;
    uint32_t *tv = vin; vin = vout; vout = tv;
  }
  return passes % 2 == 1;
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

// Per-tile instance counts from the Gaussians' rectangles: a 2D difference array
// (+1/-1 at the four corners of each band-clipped rect, 4 atomics per Gaussian)
// integrated by k_tile_hist_finalize.  Grid (rows + 1) x (tiles_x + 1), int32.
constexpr int kDiffSmem = 12288;

__global__ void __launch_bounds__(256) k_tile_hist2d(const float *__restrict__ splats, const uint32_t *__restrict__ ids,
                                                     int64_t cap, const uint32_t *nd, Band b,
                                                     int32_t *__restrict__ diff) {
  extern __shared__ int32_t dsm[];
  const int gw = b.tiles_x + 1, gh = b.row_end - b.row_begin + 1;
  const int cells = gw * gh;
  const bool priv = cells <= kDiffSmem;
  if (priv)
    for (int e = threadIdx.x; e < cells; e += blockDim.x) dsm[e] = 0;
  __syncthreads();
  int32_t *d = priv ? dsm : diff;
  const int64_t m = tmin<int64_t>(*nd, cap);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    int x0, y0, x1, y1;
    if (band_rect(splats + 12 * (int64_t)ids[j], b, x0, y0, x1, y1) == 0) continue;
    y0 -= b.row_begin;
    y1 -= b.row_begin;
    atomicAdd(&d[y0 * gw + x0], 1);
    atomicAdd(&d[y0 * gw + x1 + 1], -1);
    atomicAdd(&d[(y1 + 1) * gw + x0], -1);
    atomicAdd(&d[(y1 + 1) * gw + x1 + 1], 1);
  }
  __syncthreads();
  if (priv)
    for (int e = threadIdx.x; e < cells; e += blockDim.x)
      if (dsm[e]) atomicAdd(diff + e, dsm[e]);
}

// One CTA: integrate the difference grid into per-tile counts, write the CSR
// offsets, and derive the exclusive digit histograms of every radix pass of the
// tile key (so the instance sort needs no histogram pass over its keys).
__global__ void __launch_bounds__(1024) k_tile_hist_finalize(int32_t *__restrict__ diff, int tiles_x, int rows,
                                                             int passes, int bpp, int total_bits,
                                                             int32_t *__restrict__ offsets,
                                                             uint32_t *__restrict__ gbins) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t gb[4][256];
  const int gw = tiles_x + 1;
  for (int e = threadIdx.x; e < 4 * 256; e += 1024) (&gb[0][0])[e] = 0;
  // prefix along x then along y, one warp per row / column (warp scans with carry)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < rows; r += 32) {
    int32_t carry_r = 0;
    for (int x0 = 0; x0 < tiles_x; x0 += 32) {
      const int x = x0 + lane;
      int32_t v = x < tiles_x ? diff[r * gw + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (x < tiles_x) diff[r * gw + x] = v + carry_r;
      carry_r += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  for (int x = warp; x < tiles_x; x += 32) {
    int32_t carry_c = 0;
    for (int r0 = 0; r0 < rows; r0 += 32) {
      const int r = r0 + lane;
      int32_t v = r < rows ? diff[r * gw + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (r < rows) diff[r * gw + x] = v + carry_c;
      carry_c += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const int ntiles = rows * tiles_x;
  uint32_t carry = 0;
  for (int c = 0; c < ntiles; c += 1024) {
    const int t = c + threadIdx.x;
    const uint32_t v = t < ntiles ? (uint32_t)diff[(t / tiles_x) * gw + (t % tiles_x)] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(v, ws, &tot);
    if (t < ntiles) {
      offsets[t] = (int32_t)(carry + ex);
      for (int p = 0; p < passes; ++p) {
        const int sh = p * bpp, nb = min(bpp, total_bits - sh);
        if (v) atomicAdd(&gb[p][((uint32_t)t >> sh) & ((1u << nb) - 1)], v);
      }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) offsets[ntiles] = (int32_t)carry;
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    const uint32_t v = threadIdx.x < 256 ? gb[p][threadIdx.x] : 0u;
    const uint32_t ex = block_exclusive_scan(v, ws, nullptr);
    if (threadIdx.x < 256) gbins[p * 256 + threadIdx.x] = ex;
  }
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
  SortScratch ss;
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
  w.ss = carve_sort<uint64_t>(c, N, 8);
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
  // depth digits: 8 stable 8-bit passes over the M selected Gaussians (float64 keys); even
  // pass count -> result back in (keysA, valsA)
  radix_sort<uint64_t>(w.keysA, w.valsA, w.keysB, w.valsB, (uint64_t)n, w.m, 64, w.ss, st);
  // depth-ordered ids are in valsA; per-Gaussian instance offsets in depth order
  k_gather_counts<<<g256, 256, 0, st>>>(w.valsA, w.cnt, n, w.m, w.inst_off);
  device_scan(w.inst_off, w.inst_off, (uint64_t)n, w.m, w.partials, nullptr, d_num_instances, st);
  return launch_status();
}

struct InstWS {
  uint32_t *keysA, *keysB, *valsB;
  int32_t *diff;
  SortScratch ss;
  size_t bytes;
};

static InstWS carve_inst(void *p, int64_t count, size_t ntiles) {
  Carve c(p);
  InstWS w;
  const size_t I = (size_t)tmax<int64_t>(count, 1);
  w.keysA = c.take<uint32_t>(I);
  w.keysB = c.take<uint32_t>(I);
  w.valsB = c.take<uint32_t>(I);
  w.ss = carve_sort<uint32_t>(c, I, 4);  // up to 32 tile bits
  w.diff = c.take<int32_t>(ntiles);       // (rows + 1) x (tiles_x + 1) difference grid bound
  w.bytes = c.off;
  return w;
}

extern "C" int tgs_bin_instances_workspace(int64_t n, int64_t num_instances, size_t *bytes) {
  if (n < 0 || num_instances < 0 || !bytes) return TGS_ERR_INVALID;
  // the per-tile histogram is sized for the largest band a caller can request (2^18 tiles here
  // at most per call of tgs_bin_instances); callers with more tiles get a bigger query below
  *bytes = carve_inst(nullptr, num_instances, (size_t)1 << 18).bytes;
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
  if (ntiles > (1u << 18)) return TGS_ERR_UNSUPPORTED;
  InstWS w = carve_inst(workspace, num_instances, (size_t)1 << 18);
  const int bits = key_bits(ntiles);
  const int passes = (bits + 7) / 8;
  // ping-pong so the last pass lands in sorted_ids: with an even pass count the
  // duplicate writes straight into sorted_ids (A = sorted_ids, B = valsB)
  uint32_t *ids_out = reinterpret_cast<uint32_t *>(sorted_ids);
  uint32_t *vA = (passes % 2 == 0) ? ids_out : w.valsB;
  uint32_t *vB = (passes % 2 == 0) ? w.valsB : ids_out;
  // per-tile counts (-> CSR offsets) and the digit histograms from the rects
  const int rows = b.row_end - b.row_begin;
  const int cells = (rows + 1) * (b.tiles_x + 1);
  static bool attr_done = false;  // idempotent function attribute, set once per process
  if (!attr_done) {
    cudaFuncSetAttribute(k_tile_hist2d, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiffSmem * 4);
    attr_done = true;
  }
  cudaMemsetAsync(w.ss.gbins, 0, w.ss.bytes_zeroed, st);
  cudaMemsetAsync(w.diff, 0, (size_t)cells * 4, st);
  const unsigned dgrid = (unsigned)tmin<int64_t>(ceil_div<int64_t>(n, 256), 148 * 2);
  k_tile_hist2d<<<dgrid, 256, cells <= kDiffSmem ? (size_t)cells * 4 : 0, st>>>(splats, gw.valsA, n, gw.m, b,
                                                                                w.diff);
  const int bpp = passes ? (bits + passes - 1) / passes : 0;
  k_tile_hist_finalize<<<1, 1024, 0, st>>>(w.diff, b.tiles_x, rows, passes, bpp, bits, tile_offsets, w.ss.gbins);
  k_duplicate<<<(unsigned)ceil_div<int64_t>(n, 256), 256, 0, st>>>(splats, gw.valsA, gw.inst_off, n, gw.m, b,
                                                                    w.keysA, vA);
  radix_sort<uint32_t>(w.keysA, vA, w.keysB, vB, (uint64_t)num_instances, nullptr, bits, w.ss, st,
                       /*hist_ready=*/true, /*last_keys=*/false);
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
