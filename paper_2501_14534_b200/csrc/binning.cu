// binning.cu — tile binning and the (tile | depth | index) order (R5).
//
// Reference: bin_tiles (rasterizer.py:95-148) emits one instance per covered
// tile (row-major within the Gaussian's rect), then np.lexsort((gid, depth,
// tile)) and a bincount/cumsum for the CSR offsets.
//
// B200 design.  Every instance of a Gaussian carries the Gaussian's depth, so the
// lexsort factors into
//   (A) a stable sort of the M on-screen GAUSSIANS by their float64 depth key
//       (ties by index) — tgs_bin_gaussians, ONE launch: a ticketed chain of
//       selection tiles and eight 8-bit onesweep passes (decoupled look-back
//       inside a pass, a completion counter between passes), and
//   (B) a stable counting sort of the INSTANCES by tile in which no instance key
//       is ever materialised — tgs_bin_instances: the depth-ordered Gaussians are
//       cut into chunks of C; a chunk x tile count matrix (u16) gives every chunk
//       its base offset in every tile list; one warp per chunk then writes each
//       instance straight to its final slot.  Inside a warp the 32 Gaussians of a
//       group are ranked per tile by two coverage bitmasks (Gaussians whose
//       column range / row range contains the tile), so the rank of Gaussian k
//       in tile (x, y) is popc(col[x] & row[y] & lanes_below(k)).
// Stability of (A) plus the depth-ordered chunk walk of (B) gives exactly
// lexsort's (tile, depth, index) order, bit-identical to the oracle.
#include "tgs_common.cuh"
#include "tgs_math.cuh"

namespace tgs {

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

// Look-back status words: flag | count in one 32-bit word, so relaxed GPU-scope
// accesses suffice (no acquire fence, which costs an L1 invalidate per probe).
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Decoupled look-back for one counter: publish `agg` for `tile`, return the
// exclusive prefix of all earlier tiles (which hold earlier tickets, so they are
// resident or finished — the wait cannot deadlock).
template <int W>
__device__ __forceinline__ uint32_t lookback(uint32_t *status, size_t stride, uint32_t tile, uint32_t agg) {
  uint32_t *mine = status + (size_t)tile * stride;
  if (tile == 0) {
    st_relaxed(mine, kFlagInc | agg);
    return 0;
  }
  st_relaxed(mine, kFlagAgg | agg);
  uint32_t excl = 0;
  int j = (int)tile - 1;
  bool found = false;
  while (!found) {
    uint32_t v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = (j - k >= 0) ? ld_relaxed(status + (size_t)(j - k) * stride) : kFlagInc;
    int used = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (found || (v[k] >> 30) == 0) break;  // stop at the first unpublished predecessor
      excl += v[k] & kValMask;
      found = (v[k] & kFlagInc) != 0;
      ++used;
    }
    j -= found ? 0 : used;
  }
  st_relaxed(mine, kFlagInc | (excl + agg));
  return excl;
}

// ------------------------------------------------------------------ bands
struct Band {
  int W, H, ts, tiles_x, tiles_y, row_begin, row_end;
};

// Band-restricted tile rect of a projected record (0 when off-screen / outside the band).
__device__ __forceinline__ int band_rect(const float *sp, const Band &b, int &x0, int &y0, int &x1, int &y1) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(sp));
  const float r = __ldg(sp + 10);
  const int n = tile_rect(a.x, a.y, r, b.W, b.H, b.ts, b.tiles_x, b.tiles_y, x0, y0, x1, y1);
  if (n == 0) return 0;
  y0 = max(y0, b.row_begin);
  y1 = min(y1, b.row_end - 1);
  return y1 >= y0 ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0;
}

// Band rect packed as (x0 | x1 << 16, y0 | y1 << 16), rows relative to the band.
__device__ __forceinline__ uint2 pack_rect(int x0, int y0, int x1, int y1) {
  return make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
}

// ======================================================= (A) depth sort
// One launch.  Tickets [0, T0) are histogram tiles over the n Gaussians (in-band
// test, packed band rect per Gaussian, digit histograms of all passes, the
// selected and instance totals); tickets T0 + p*TP + j are tile j of radix pass
// p.  Pass 0 reads the Gaussians in index order straight from the inputs and
// compacts the selected ones as it scatters; later passes ping-pong between two
// buffers.  A pass tile first waits for the completion counter of the stage
// feeding it; every stage it waits on holds strictly earlier tickets, so the
// chain is deadlock-free without any co-residency assumption.  Passes whose
// digit is the same for all keys are skipped.
constexpr int kDsThreads = 256;
constexpr int kDsIPT = 16;
constexpr int kDsTile = kDsThreads * kDsIPT;  // 4096 items per tile
constexpr int kDsWarps = kDsThreads / 32;
constexpr int kDsPasses = 8;                  // 64-bit keys, 8-bit digits
constexpr int kDsLookback = 16;
constexpr uint32_t kNoRect = 0xffffffffu;     // rect_by_gid of an unselected Gaussian

struct DsCtl {                       // zeroed before every launch
  uint32_t ticket;
  uint32_t m;                        // selected Gaussians
  uint32_t done[kDsPasses + 1];      // done[0]: histogram tiles; done[p + 1]: tiles of pass p
  uint32_t pad[5];
  uint32_t hist[kDsPasses][256];     // global digit histograms
};

struct DsArgs {
  const float *splats;
  const int32_t *tiles_touched;
  const uint64_t *depth_keys;        // may be null: key on the float32 splat depth
  uint32_t n;
  Band b;
  uint64_t *keysA, *keysB;
  uint32_t *valsA, *valsB;
  DsCtl *ctl;
  uint2 *rect_by_gid;                // n: band rect of each Gaussian (packed u16 pairs) or kNoRect
  uint2 *rects_sorted;               // M: the selected rects in depth order (written by the last pass)
  uint32_t *ids;                     // M: Gaussian ids in depth order (written by the last pass)
  uint32_t *status;                  // kDsPasses * TP * 256 look-back words
  uint32_t T0, TP;
  unsigned long long *num_instances;
};

// Optional per-ticket phase timestamps (tgs_debug_trace_depth_sort; null = off).
__device__ unsigned long long *g_ds_trace = nullptr;
__device__ __forceinline__ void ds_mark(uint32_t ticket, int k) {
  if (threadIdx.x == 0 && g_ds_trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ds_trace[(size_t)ticket * 8 + k] = t;
  }
}

__device__ __forceinline__ void wait_count(const uint32_t *p, uint32_t need) {
  if (threadIdx.x == 0)
    while (ld_acquire(p) < need) __nanosleep(32);
  __syncthreads();
}
__device__ __forceinline__ void signal_done(uint32_t *p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1u);
  }
}

struct DsSmem {
  union {
    struct {
      uint64_t ks[kDsTile];
      uint32_t vs[kDsTile];
      uint32_t vin[kDsTile];        // values in item order (kept out of registers while ranking)
      uint32_t wcnt[kDsWarps][256];
    } pass;
    struct {
      uint32_t hist[kDsPasses][256];
    } sel;
  };
  uint32_t dstart[256];
  uint32_t gbase[256];
  uint32_t wsum[32];
  uint32_t ticket, m, cnt;
  unsigned long long inst;
  uint32_t nsel;
};

__device__ __forceinline__ uint64_t ds_key(const DsArgs &a, uint32_t i) {
  return a.depth_keys ? __ldg(a.depth_keys + i) : orderable_key64((double)__ldg(a.splats + 12 * (size_t)i + 9));
}

__device__ void ds_hist_tile(const DsArgs &a, DsSmem &sm, uint32_t t) {
  for (int e = threadIdx.x; e < kDsPasses * 256; e += kDsThreads) (&sm.sel.hist[0][0])[e] = 0;
  if (threadIdx.x == 0) {
    sm.inst = 0;
    sm.nsel = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t nsel = 0;
  unsigned long long inst = 0;
  // striped, four batches of 4 items: all loads of a batch are issued before use
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    int32_t tt[4];
    float4 sp[4];
    float rad[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t i = t * kDsTile + (hh * 4 + r) * kDsThreads + threadIdx.x;
      const bool in = i < a.n;
      tt[r] = in ? __ldg(a.tiles_touched + i) : 0;
      sp[r] = in ? __ldg(reinterpret_cast<const float4 *>(a.splats + 12 * (size_t)i)) : make_float4(0, 0, 0, 0);
      rad[r] = in ? __ldg(a.splats + 12 * (size_t)i + 10) : 0.0f;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t i = t * kDsTile + (hh * 4 + r) * kDsThreads + threadIdx.x;
      int x0 = 0, y0 = 0, x1 = -1, y1 = -1, c = 0;
      if (tt[r] > 0) {
        c = tile_rect(sp[r].x, sp[r].y, rad[r], a.b.W, a.b.H, a.b.ts, a.b.tiles_x, a.b.tiles_y, x0, y0, x1, y1);
        if (c > 0) {
          y0 = max(y0, a.b.row_begin);
          y1 = min(y1, a.b.row_end - 1);
          c = y1 >= y0 ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0;
        }
      }
      const bool ok = c > 0;
      if (i < a.n)
        a.rect_by_gid[i] = ok ? pack_rect(x0, y0 - a.b.row_begin, x1, y1 - a.b.row_begin) : make_uint2(kNoRect, kNoRect);
      const uint64_t key = ok ? ds_key(a, i) : 0ull;
      nsel += ok;
      inst += (uint32_t)c;
      // digit histograms; the high key bytes are nearly constant, so a warp whose
      // valid lanes share a digit adds once instead of contending on one bin
      const uint32_t okm = __ballot_sync(0xffffffffu, ok);
      if (okm == 0) continue;
      const int src = __ffs(okm) - 1;
#pragma unroll
      for (int p = 0; p < kDsPasses; ++p) {
        const uint32_t d = (uint32_t)(key >> (8 * p)) & 255u;
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, src);
        if (__all_sync(0xffffffffu, !ok || d == d0)) {
          if (lane == src) atomicAdd(&sm.sel.hist[p][d], (uint32_t)__popc(okm));
        } else if (ok) {
          atomicAdd(&sm.sel.hist[p][d], 1u);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    nsel += __shfl_xor_sync(0xffffffffu, nsel, o);
    inst += __shfl_xor_sync(0xffffffffu, inst, o);
  }
  if (lane == 0) {
    atomicAdd(&sm.nsel, nsel);
    atomicAdd(&sm.inst, inst);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kDsPasses * 256; e += kDsThreads) {
    const uint32_t v = (&sm.sel.hist[0][0])[e];
    if (v) atomicAdd(&a.ctl->hist[0][0] + e, v);
  }
  if (threadIdx.x == 0 && sm.nsel) atomicAdd(&a.ctl->m, sm.nsel);
  signal_done(&a.ctl->done[0]);
}

__device__ void ds_pass_tile(const DsArgs &a, DsSmem &sm, int p, uint32_t j, uint32_t m, uint32_t ticket,
                             bool odd, bool last) {
  const uint64_t *keys_in = odd ? a.keysB : a.keysA;
  const uint32_t *vals_in = odd ? a.valsB : a.valsA;
  uint64_t *keys_out = odd ? a.keysA : a.keysB;
  uint32_t *vals_out = last ? a.ids : (odd ? a.valsA : a.valsB);
  const int shift = 8 * p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kDsWarps * 256; e += kDsThreads) (&sm.pass.wcnt[0][0])[e] = 0;
  const uint64_t base = (uint64_t)j * kDsTile;
  const uint64_t wbase = base + (uint64_t)warp * (kDsIPT * 32);
  uint64_t key[kDsIPT];
  uint32_t okbits = 0;
  const uint32_t ibase = warp * (kDsIPT * 32) + lane;  // item index in the tile = ibase + 32 r
  if (p == 0) {
    // pass 0: Gaussians in index order from the inputs; unselected ones drop out
    uint32_t rx[kDsIPT];
#pragma unroll
    for (int r = 0; r < kDsIPT; ++r) {
      const uint64_t q = wbase + r * 32 + lane;
      rx[r] = q < a.n ? __ldcg(&a.rect_by_gid[q].x) : kNoRect;
    }
#pragma unroll
    for (int r = 0; r < kDsIPT; ++r) {
      const uint32_t q = (uint32_t)(wbase + r * 32 + lane);
      const bool ok = rx[r] != kNoRect;
      okbits |= (uint32_t)ok << r;
      key[r] = ok ? ds_key(a, q) : 0ull;
      sm.pass.vin[ibase + 32 * r] = q;
    }
  } else {
    // all loads first (L2 only: the buffers were written by other CTAs of this launch)
#pragma unroll
    for (int r = 0; r < kDsIPT; ++r) {
      const uint64_t q = wbase + r * 32 + lane;
      const bool ok = q < m;
      okbits |= (uint32_t)ok << r;
      key[r] = ok ? (uint64_t)__ldcg(reinterpret_cast<const unsigned long long *>(keys_in) + q) : 0ull;
      sm.pass.vin[ibase + 32 * r] = ok ? __ldcg(vals_in + q) : 0u;
    }
  }
  __syncthreads();
  ds_mark(ticket, 2);
  const uint32_t lt = lanemask_lt();
  uint32_t rank2[kDsIPT / 2];  // two 16-bit ranks per register
  // warp-synchronous multisplit: ranks stable in item order (warp-major, round, lane)
#pragma unroll
  for (int r = 0; r < kDsIPT; ++r) {
    const bool ok = okbits >> r & 1u;
    const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
    uint32_t peers = __ballot_sync(0xffffffffu, ok);  // lanes with the same digit: 8 ballots
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bb : ~bb;
    }
    const uint32_t prev = ok ? sm.pass.wcnt[warp][d] : 0u;
    const uint32_t rk = prev + __popc(peers & lt);
    rank2[r >> 1] = (r & 1) ? (rank2[r >> 1] | (rk << 16)) : rk;
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) sm.pass.wcnt[warp][d] = prev + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  ds_mark(ticket, 3);
  uint32_t dtotal = 0;
  for (int w = 0; w < kDsWarps; ++w) {  // kDsThreads == 256: one digit per thread
    const uint32_t c = sm.pass.wcnt[w][threadIdx.x];
    sm.pass.wcnt[w][threadIdx.x] = dtotal;
    dtotal += c;
  }
  uint32_t cnt;
  const uint32_t ds = block_exclusive_scan(dtotal, sm.wsum, &cnt);
  sm.dstart[threadIdx.x] = ds;
  __syncthreads();
  // local reorder first (frees the key registers), then the look-back
#pragma unroll
  for (int r = 0; r < kDsIPT; ++r) {
    if (okbits >> r & 1u) {
      const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
      const uint32_t s = sm.dstart[d] + sm.pass.wcnt[warp][d] + ((rank2[r >> 1] >> (16 * (r & 1))) & 0xffffu);
      sm.pass.ks[s] = key[r];
      sm.pass.vs[s] = sm.pass.vin[ibase + 32 * r];
    }
  }
  const uint32_t excl = lookback<kDsLookback>(a.status + (size_t)p * a.TP * 256 + threadIdx.x, 256, j, dtotal);
  sm.gbase[threadIdx.x] += excl;  // gbase holds this pass's exclusive digit base
  __syncthreads();
  ds_mark(ticket, 4);
  for (uint32_t e = threadIdx.x; e < cnt; e += kDsThreads) {
    const uint64_t k = sm.pass.ks[e];
    const uint32_t d = (uint32_t)(k >> shift) & 255u;
    const uint32_t o = sm.gbase[d] + (e - sm.dstart[d]);
    if (!last) __stcg(reinterpret_cast<unsigned long long *>(keys_out) + o, (unsigned long long)k);
    const uint32_t v = sm.pass.vs[e];
    __stcg(vals_out + o, v);
    if (last) __stcg(a.rects_sorted + o, __ldcg(a.rect_by_gid + v));
  }
  signal_done(&a.ctl->done[p + 1]);
  ds_mark(ticket, 5);
}

// One ticket of the chain (see above).
__device__ void ds_ticket(const DsArgs &a, DsSmem &sm, uint32_t t) {
  ds_mark(t, 0);
  if (t < a.T0) {
    ds_mark(t, 1);
    ds_hist_tile(a, sm, t);
    ds_mark(t, 5);
    return;
  }
  const int p = (int)((t - a.T0) / a.TP);
  const uint32_t j = (t - a.T0) % a.TP;
  wait_count(&a.ctl->done[0], a.T0);
  if (threadIdx.x == 0) sm.m = __ldcg(&a.ctl->m);
  __syncthreads();
  const uint32_t m = sm.m;
  const uint32_t live = (m + kDsTile - 1) / kDsTile;
  if (m == 0 || (p > 0 && j >= live)) return;  // pass 0 tiles cover all n Gaussians
  // passes whose digit is the same for every key are the identity: skip them
  // (pass 0 always runs: it compacts and, if it is the only pass, writes the outputs)
  uint32_t active = 1u;
#pragma unroll
  for (int q = 1; q < kDsPasses; ++q) {
    const uint32_t hq = __ldcg(&a.ctl->hist[q][threadIdx.x]);
    if (__syncthreads_count(hq != 0u) > 1) active |= 1u << q;
  }
  if (!(active >> p & 1u)) return;
  const bool odd = __popc(active & ((1u << p) - 1u)) & 1;
  const bool last = (active >> (p + 1)) == 0u;
  const int prev = p > 0 ? 31 - __clz(active & ((1u << p) - 1u)) : -1;
  // this pass's exclusive digit base (from the histograms)
  const uint32_t h = __ldcg(&a.ctl->hist[p][threadIdx.x]);
  sm.gbase[threadIdx.x] = block_exclusive_scan(h, sm.wsum, nullptr);
  if (prev >= 0) wait_count(&a.ctl->done[prev + 1], prev == 0 ? a.T0 : live);
  __syncthreads();
  ds_mark(t, 1);
  ds_pass_tile(a, sm, p, j, m, t, odd, last);
}

// The fallback sort: a small persistent grid; each CTA takes tickets until the
// chain is exhausted.  A CTA only ever waits for stages whose tickets were
// already taken by running CTAs, so any grid size is deadlock-free.  Exits at
// once unless the bucket fast path overflowed.
__global__ void __launch_bounds__(kDsThreads, 3) k_depth_sort(DsArgs a, const uint32_t *overflow) {
  if (*overflow == 0u) return;
  extern __shared__ __align__(16) unsigned char ds_raw[];
  DsSmem &sm = *reinterpret_cast<DsSmem *>(ds_raw);
  const uint32_t total = a.T0 + kDsPasses * a.TP;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) sm.ticket = atomicAdd(&a.ctl->ticket, 1u);
    __syncthreads();
    const uint32_t t = sm.ticket;
    if (t >= total) return;
    ds_ticket(a, sm, t);
  }
}

// ----------------------------------------------- (A) fast path: value buckets
// Every selected key falls in one of 2^kBBits buckets by (key - kmin) >> shift,
// which is monotone in the key, so bucket order is key order.  K0 selects and
// finds [kmin, kmax]; K1 counts per bucket; K2 scans; K3 scatters (unstable, by
// atomic slot claims); K4 ranks every item inside its bucket by (key, index) —
// buckets hold a handful of items — and writes the outputs.  A bucket larger
// than kBMax (an adversarial depth distribution) raises `overflow`, and the
// ticketed LSD sort below (k_depth_sort, launched on a small persistent grid
// that exits at once otherwise) recomputes the order from scratch.
constexpr int kBBits = 17;
constexpr uint32_t kBuckets = 1u << kBBits;
constexpr uint32_t kBMax = 256;
constexpr int kBScanIPT = 16;
constexpr int kBScanTile = 256 * kBScanIPT;  // buckets per scan CTA

struct BsCtl {                 // zeroed before every call
  unsigned long long kmin_inv; // atomicMax of ~key
  unsigned long long kmax;
  uint32_t m, overflow, ticket, pad;
};

// One launch instead of two memsets and a copy: zero the control block and the
// count, and forward the preprocess error flag into counts[1] (one D2H read).
__global__ void k_bs_init(BsCtl *ctl, unsigned long long *counts, const int32_t *error_flag) {
  if (threadIdx.x == 0) {
    *ctl = BsCtl{0ull, 0ull, 0u, 0u, 0u, 0u};
    counts[0] = 0ull;
    if (error_flag) counts[1] = (unsigned long long)(long long)*error_flag;
  }
}

struct BsArgs {
  const float *splats;
  const int32_t *tiles_touched;
  const uint64_t *depth_keys;
  uint32_t n;
  Band b;
  BsCtl *ctl;
  uint2 *rect_by_gid;
  uint32_t *bcount, *boff, *bstatus;
  uint64_t *keys;
  uint32_t *vals, *ids;
  uint2 *rects_sorted;
  unsigned long long *num_instances;
  uint32_t *zero;              // fallback state zeroed here (zero_words)
  size_t zero_words;
};

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, uint64_t kmin, int shift) {
  return (uint32_t)((key - kmin) >> shift);
}
__device__ __forceinline__ int bucket_shift(uint64_t kmin, uint64_t kmax) {
  const uint64_t range = kmax - kmin;
  return range == 0 ? 0 : max(0, 64 - __clzll((long long)range) - kBBits);
}

__device__ __forceinline__ uint64_t bs_key(const BsArgs &a, uint32_t i) {
  return a.depth_keys ? __ldg(a.depth_keys + i) : orderable_key64((double)__ldg(a.splats + 12 * (size_t)i + 9));
}

// K0: per Gaussian band rect (kNoRect if not selected), key range, counts.
// Grid-stride over a few CTAs per SM with one block reduction per CTA, so the
// four global counters see a few hundred atomics instead of one per warp.
__global__ void __launch_bounds__(256) k_bs_select(BsArgs a) {
  __shared__ unsigned long long r_min[8], r_max[8], r_inst[8];
  __shared__ uint32_t r_sel[8];
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = gtid; e < kBuckets; e += gstride) a.bcount[e] = 0;
  for (size_t e = gtid; e < a.zero_words; e += gstride) a.zero[e] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long kmin_inv = 0ull, kmax = 0ull, inst = 0ull;
  uint32_t nsel = 0;
  for (size_t ii = gtid; ii < a.n; ii += gstride) {
    const uint32_t i = (uint32_t)ii;
    int x0 = 0, y0 = 0, x1 = -1, y1 = -1, c = 0;
    if (__ldg(a.tiles_touched + i) > 0) {
      const float4 sp = __ldg(reinterpret_cast<const float4 *>(a.splats + 12 * (size_t)i));
      c = tile_rect(sp.x, sp.y, __ldg(a.splats + 12 * (size_t)i + 10), a.b.W, a.b.H, a.b.ts, a.b.tiles_x,
                    a.b.tiles_y, x0, y0, x1, y1);
      if (c > 0) {
        y0 = max(y0, a.b.row_begin);
        y1 = min(y1, a.b.row_end - 1);
        c = y1 >= y0 ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0;
      }
    }
    const bool ok = c > 0;
    a.rect_by_gid[i] = ok ? pack_rect(x0, y0 - a.b.row_begin, x1, y1 - a.b.row_begin) : make_uint2(kNoRect, kNoRect);
    if (ok) {
      const uint64_t key = bs_key(a, i);
      kmin_inv = max(kmin_inv, (unsigned long long)~key);
      kmax = max(kmax, (unsigned long long)key);
      ++nsel;
      inst += (uint32_t)c;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    kmin_inv = max(kmin_inv, __shfl_xor_sync(0xffffffffu, kmin_inv, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    nsel += __shfl_xor_sync(0xffffffffu, nsel, o);
    inst += __shfl_xor_sync(0xffffffffu, inst, o);
  }
  if (lane == 0) {
    r_min[warp] = kmin_inv; r_max[warp] = kmax; r_inst[warp] = inst; r_sel[warp] = nsel;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      kmin_inv = max(kmin_inv, r_min[w]); kmax = max(kmax, r_max[w]);
      inst += r_inst[w]; nsel += r_sel[w];
    }
    if (nsel) {
      atomicMax(&a.ctl->kmin_inv, kmin_inv);
      atomicMax(&a.ctl->kmax, kmax);
      atomicAdd(&a.ctl->m, nsel);
      atomicAdd(a.num_instances, inst);
    }
  }
}

// K1: bucket counts.
__global__ void __launch_bounds__(256) k_bs_hist(BsArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || __ldg(&a.rect_by_gid[i].x) == kNoRect) return;
  const uint64_t kmin = ~a.ctl->kmin_inv;
  const int shift = bucket_shift(kmin, a.ctl->kmax);
  atomicAdd(a.bcount + bucket_of(bs_key(a, i), kmin, shift), 1u);
}

// K2: exclusive scan of the bucket counts -> boff (kBuckets + 1) and the scatter
// cursors (bcount, in place); CTAs chained by decoupled look-back.
__global__ void __launch_bounds__(256) k_bs_scan(BsArgs a) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t s_blk, s_excl;
  if (threadIdx.x == 0) s_blk = atomicAdd(&a.ctl->ticket, 1u);
  __syncthreads();
  const uint32_t base = s_blk * kBScanTile + threadIdx.x * kBScanIPT;
  uint4 v[kBScanIPT / 4];
#pragma unroll
  for (int k = 0; k < kBScanIPT / 4; ++k) v[k] = reinterpret_cast<const uint4 *>(a.bcount + base)[k];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kBScanIPT / 4; ++k) s += v[k].x + v[k].y + v[k].z + v[k].w;
  uint32_t tot;
  uint32_t run = block_exclusive_scan(s, ws, &tot);
  if (threadIdx.x == 0) s_excl = lookback<16>(a.bstatus, 1, s_blk, tot);
  __syncthreads();
  run += s_excl;
#pragma unroll
  for (int k = 0; k < kBScanIPT / 4; ++k) {
    uint4 o;
    o.x = run; run += v[k].x;
    o.y = run; run += v[k].y;
    o.z = run; run += v[k].z;
    o.w = run; run += v[k].w;
    reinterpret_cast<uint4 *>(a.boff + base)[k] = o;
    reinterpret_cast<uint4 *>(a.bcount + base)[k] = o;
  }
  if (base + kBScanIPT == kBuckets) a.boff[kBuckets] = run;
}

// K3: scatter into buckets (slot order inside a bucket is arbitrary).
__global__ void __launch_bounds__(256) k_bs_scatter(BsArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || __ldg(&a.rect_by_gid[i].x) == kNoRect) return;
  const uint64_t kmin = ~a.ctl->kmin_inv;
  const int shift = bucket_shift(kmin, a.ctl->kmax);
  const uint64_t key = bs_key(a, i);
  const uint32_t pos = atomicAdd(a.bcount + bucket_of(key, kmin, shift), 1u);
  a.keys[pos] = key;
  a.vals[pos] = i;
}

// K4: exact rank inside the bucket by (key, index); outputs in depth order.
__global__ void __launch_bounds__(256) k_bs_rank(BsArgs a) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.ctl->m) return;
  const uint64_t kmin = ~a.ctl->kmin_inv;
  const int shift = bucket_shift(kmin, a.ctl->kmax);
  const uint64_t key = a.keys[p];
  const uint32_t val = a.vals[p];
  const uint32_t b = bucket_of(key, kmin, shift);
  const uint32_t s = __ldg(a.boff + b), e = __ldg(a.boff + b + 1);
  if (e - s > kBMax) {
    a.ctl->overflow = 1u;
    return;
  }
  uint32_t rank = 0;
  for (uint32_t q = s; q < e; ++q) {
    const uint64_t kq = a.keys[q];
    const uint32_t vq = a.vals[q];
    rank += (kq < key) || (kq == key && vq < val);
  }
  a.ids[s + rank] = val;
  a.rects_sorted[s + rank] = __ldg(a.rect_by_gid + val);
}

struct GaussWS {
  uint64_t *keysA, *keysB;
  uint32_t *valsA, *valsB;
  uint32_t *ids;            // depth-ordered Gaussian ids after the sort
  uint2 *rect_by_gid, *rects_sorted;
  DsCtl *ctl;
  uint32_t *status;
  uint32_t T0, TP;
  BsCtl *bctl;
  uint32_t *bcount, *boff, *bstatus;
  size_t zero_off, zero_bytes, bytes;   // [zero_off, +zero_bytes): fallback state + bstatus, zeroed by K0
};

inline GaussWS carve_gauss(void *p, int64_t n) {
  Carve c(p);
  GaussWS w;
  const size_t N = (size_t)tmax<int64_t>(n, 1);
  w.T0 = (uint32_t)ceil_div<size_t>(N, kDsTile);
  w.TP = w.T0;
  w.keysA = c.take<uint64_t>(N);
  w.keysB = c.take<uint64_t>(N);
  w.valsA = c.take<uint32_t>(N);
  w.valsB = c.take<uint32_t>(N);
  w.ids = c.take<uint32_t>(N);
  w.rect_by_gid = c.take<uint2>(N);
  w.rects_sorted = c.take<uint2>(N);
  w.zero_off = c.off;
  w.ctl = c.take<DsCtl>(1);
  w.status = c.take<uint32_t>((size_t)kDsPasses * w.TP * 256);
  w.bstatus = c.take<uint32_t>(kBuckets / kBScanTile);
  w.zero_bytes = c.off - w.zero_off;
  w.bctl = c.take<BsCtl>(1);
  w.bcount = c.take<uint32_t>(kBuckets);
  w.boff = c.take<uint32_t>(kBuckets + 1);
  w.bytes = c.off;
  return w;
}

// ================================================= (B) instance placement
// Two levels.  Super-tiles are 8x8 tiles.
//  L1 places ENTRIES (Gaussian, super-tile it overlaps) — ~1.5 per Gaussian
//     instead of ~30 instances — into per-super-tile lists, stably in depth order:
//     the depth-ordered Gaussians are cut into chunks of C = 512 and the chunks
//     into segments of kSeg; rel[c][S] (u16) counts the Gaussians of earlier
//     chunks of c's segment overlapping super-tile S, segbase[s][S] (u32) those of
//     earlier segments, and inside a chunk an entry's rank comes from 64-bit
//     coverage masks (Gaussians whose super-tile column / row range contains S).
//  L2 places the INSTANCES of one super-tile: its entries are split over 16
//     warps; per round of 32 entries a warp builds 8 column and 8 row ballots,
//     lane L owns tiles L and L + 32 of the super-tile, and writes the ids of the
//     entries covering them in order (bit iteration over col & row masks).
//  The per-tile CSR offsets come from the L2 per-unit counts.
constexpr int kST = 8;                  // super-tile edge in tiles
constexpr int kSTShift = 3;
constexpr int kChunk = 512;             // Gaussians per chunk = 8 warps x 64
constexpr int kChunkWarps = kChunk / 64;
constexpr int kSeg = 4;                 // chunks per segment (counted by one CTA, in order)
constexpr int kDiffCells = 12288;       // 2D difference cells per count CTA
constexpr int kScanCols = 32;           // bins per segment-scan CTA
constexpr int kScanGroups = 32;         // segment ranges per segment-scan CTA
#ifndef TGS_PLACE_WARPS
#define TGS_PLACE_WARPS 16
#endif
constexpr int kPlaceWarps = TGS_PLACE_WARPS;
constexpr int kPUnit = 2048;            // entries per L2 unit

struct InstGeom {
  uint32_t nchunks, nseg, NS, T;        // NS super-tiles, T tiles (band)
  int sx, sy;                           // super-tile grid
  int slab_rows, slabs;                 // super-tile-row slabs of the count kernel
  uint64_t ecap;                        // entry capacity
  uint32_t punits;                      // L2 unit capacity
};

inline InstGeom inst_geom(int64_t n, int64_t num_instances, const Band &b) {
  InstGeom g;
  const uint64_t N = (uint64_t)tmax<int64_t>(n, 1);
  const int rows = b.row_end - b.row_begin;
  g.T = (uint32_t)tmax(rows * b.tiles_x, 1);
  g.sx = (b.tiles_x + kST - 1) / kST;
  g.sy = (rows + kST - 1) / kST;
  g.NS = (uint32_t)tmax(g.sx * g.sy, 1);
  g.nchunks = (uint32_t)ceil_div<uint64_t>(N, kChunk);
  g.nseg = ceil_div<uint32_t>(g.nchunks, kSeg);
  g.slab_rows = tmax(1, tmin(g.sy, kDiffCells / (g.sx + 1) - 1));
  g.slabs = ceil_div(g.sy, g.slab_rows);
  // super-tiles spanned by an nx x ny rect <= min(nx ny, nx ny / 4 + 4)
  const uint64_t I = (uint64_t)tmax<int64_t>(num_instances, 1);
  g.ecap = tmin<uint64_t>(I, I / 4 + 4 * N);
  g.punits = (uint32_t)(g.NS + g.ecap / kPUnit + 1);
  return g;
}

__device__ __forceinline__ void unpack_rect(uint2 r, int &x0, int &y0, int &x1, int &y1) {
  x0 = (int)(r.x & 0xffffu); x1 = (int)(r.x >> 16);
  y0 = (int)(r.y & 0xffffu); y1 = (int)(r.y >> 16);
}

// L1 counts.  One CTA per (segment, super-tile-row slab): for each of the
// segment's chunks in order, +-1 at the four corners of every super-tile rect in
// a shared difference grid, a 2D prefix, then rel = the running per-bin count
// before this chunk, running += counts.  Also the per-chunk entry totals.
__global__ void __launch_bounds__(256) k_seg_count(const uint2 *__restrict__ rects, const uint32_t *__restrict__ d_m,
                                                   int sx, int slab_rows, int sy,
                                                   uint16_t *__restrict__ rel, uint32_t *__restrict__ segsum,
                                                   uint32_t *__restrict__ chunk_ent) {
  extern __shared__ int32_t smc[];
  __shared__ uint32_t red[8];
  const uint32_t m = *d_m;
  const uint32_t s = blockIdx.x;
  const uint32_t live = ceil_div<uint32_t>(m, (uint32_t)kChunk);
  if (s * kSeg >= live) return;
  const uint32_t NS = (uint32_t)(sx * sy);
  const int r0 = blockIdx.y * slab_rows;
  const int nr = min(slab_rows, sy - r0);
  const int gw = sx + 1;
  const int cells = gw * (nr + 1);
  int32_t *dg = smc;
  uint32_t *run = reinterpret_cast<uint32_t *>(smc + cells);  // nr * sx running counts
  for (int e = threadIdx.x; e < nr * sx; e += blockDim.x) run[e] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t c1 = tmin<uint32_t>((s + 1) * kSeg, live);
  for (uint32_t c = s * kSeg; c < c1; ++c) {
    for (int e = threadIdx.x; e < cells; e += blockDim.x) dg[e] = 0;
    __syncthreads();
    const uint32_t end = tmin<uint32_t>((c + 1) * (uint32_t)kChunk, m);
    uint32_t ent = 0;
    for (uint32_t j = c * kChunk + threadIdx.x; j < end; j += blockDim.x) {
      int x0, y0, x1, y1;
      unpack_rect(__ldg(rects + j), x0, y0, x1, y1);
      x0 >>= kSTShift; x1 >>= kSTShift;
      y0 = max((y0 >> kSTShift) - r0, 0);
      y1 = min((y1 >> kSTShift) - r0, nr - 1);
      if (y1 < y0) continue;
      ent += (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
      atomicAdd(&dg[y0 * gw + x0], 1);
      atomicAdd(&dg[y0 * gw + x1 + 1], -1);
      atomicAdd(&dg[(y1 + 1) * gw + x0], -1);
      atomicAdd(&dg[(y1 + 1) * gw + x1 + 1], 1);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
    if (lane == 0) red[warp] = ent;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < nw; ++w) tot += red[w];
      if (tot) atomicAdd(chunk_ent + c, tot);
    }
    for (int r = warp; r < nr; r += nw) {  // prefix along x, one warp per row
      int32_t carry = 0;
      for (int xb = 0; xb < sx; xb += 32) {
        const int x = xb + lane;
        int32_t v = x < sx ? dg[r * gw + x] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += y;
        }
        if (x < sx) dg[r * gw + x] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    // prefix along y, one thread per column; emit the running count, then add
    uint16_t *out = rel + (size_t)c * NS + (size_t)r0 * sx;
    for (int x = threadIdx.x; x < sx; x += blockDim.x) {
      int32_t col = 0;
      for (int r = 0; r < nr; ++r) {
        col += dg[r * gw + x];
        const uint32_t cur = run[r * sx + x];
        out[r * sx + x] = (uint16_t)cur;
        run[r * sx + x] = cur + (uint32_t)col;
      }
    }
    __syncthreads();
  }
  uint32_t *sout = segsum + (size_t)s * NS + (size_t)r0 * sx;
  for (int e = threadIdx.x; e < nr * sx; e += blockDim.x) sout[e] = run[e];
}

// Exclusive scan over segments down each bin column (in place) + the CSR
// offsets over bins.  A CTA owns kScanCols bins; its kScanGroups thread rows scan
// contiguous ranges of segments, combined through shared memory; CTAs take
// tickets and chain their bin totals by decoupled look-back.
__global__ void __launch_bounds__(kScanCols * kScanGroups) k_seg_base(uint32_t *__restrict__ segsum,
                                                                     const uint32_t *__restrict__ d_m, uint32_t NB,
                                                                     uint32_t *__restrict__ status,
                                                                     uint32_t *__restrict__ ticket,
                                                                     uint32_t *__restrict__ offsets) {
  __shared__ uint32_t part[kScanGroups][kScanCols];
  __shared__ uint32_t ws[32];
  __shared__ uint32_t s_blk, s_excl;
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const int col = threadIdx.x % kScanCols, grp = threadIdx.x / kScanCols;
  const uint32_t t = blk * kScanCols + col;
  const uint32_t nseg = ceil_div<uint32_t>(ceil_div<uint32_t>(*d_m, (uint32_t)kChunk), kSeg);
  const uint32_t per = ceil_div<uint32_t>(nseg, kScanGroups);
  const uint32_t s0 = tmin<uint32_t>(grp * per, nseg), s1 = tmin<uint32_t>(s0 + per, nseg);
  uint32_t sum = 0;
  if (t < NB)
    for (uint32_t s = s0; s < s1; ++s) sum += segsum[(size_t)s * NB + t];
  part[grp][col] = sum;
  __syncthreads();
  if (grp == 0) {  // exclusive over the groups of this column
    uint32_t r = 0;
#pragma unroll
    for (int g = 0; g < kScanGroups; ++g) {
      const uint32_t v = part[g][col];
      part[g][col] = r;
      r += v;
    }
    sum = r;  // column total
  }
  __syncthreads();
  uint32_t runv = part[grp][col];
  if (t < NB)
    for (uint32_t s = s0; s < s1; ++s) {
      const uint32_t v = segsum[(size_t)s * NB + t];
      segsum[(size_t)s * NB + t] = runv;
      runv += v;
    }
  __syncthreads();
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan(grp == 0 && t < NB ? sum : 0u, ws, &tot);
  if (threadIdx.x == 0) s_excl = lookback<16>(status, 1, blk, tot);
  __syncthreads();
  if (grp == 0 && t < NB) {
    offsets[t] = s_excl + ex;
    if (t == NB - 1) offsets[NB] = s_excl + ex + sum;
  }
}

// L1 scatter.  One CTA per chunk (a chunk has ~1.5 entries per Gaussian); it
// builds the 64-bit super-tile coverage masks of all 8 groups (64 Gaussians
// each) of its chunk, then entry (Gaussian k of group w, super-tile S = (x, y))
// goes to  soff[S] + segbase[s][S] + rel[c][S]
//          + sum_{w' < w} popc(col_w'[x] & row_w'[y]) + popc(col_w[x] & row_w[y] & below(k)),
// and stores the Gaussian's depth-order index.
__global__ void __launch_bounds__(kChunkWarps * 32) k_scatter(const uint2 *__restrict__ rects,
                                                              const uint32_t *__restrict__ d_m, int sx, int sy,
                                                              const uint32_t *__restrict__ chunk_ent,
                                                              const uint16_t *__restrict__ rel,
                                                              const uint32_t *__restrict__ segbase,
                                                              const uint32_t *__restrict__ soff,
                                                              uint32_t *__restrict__ entries) {
  extern __shared__ unsigned long long mk[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t m = *d_m;
  const uint32_t live = ceil_div<uint32_t>(m, (uint32_t)kChunk);
  const uint32_t NS = (uint32_t)(sx * sy);
  const uint32_t c = blockIdx.x;
  if (c >= live) return;
  const int mw = sx + sy;               // column masks [0, sx), row masks after
  const uint32_t j0 = c * kChunk;
  // lane l of warp w holds Gaussians 64w + l and 64w + 32 + l, so the group's
  // 64-bit coverage mask of a column / row is ballot(h = 0) | ballot(h = 1) << 32
  uint32_t cnt[2];
  int x0[2], y0[2], x1[2], y1[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t k = warp * 64 + h * 32 + lane;
    const uint32_t j = j0 + k;
    cnt[h] = 0;
    x0[h] = 0; y0[h] = 0; x1[h] = -1; y1[h] = -1;
    if (j < m) {
      unpack_rect(__ldg(rects + j), x0[h], y0[h], x1[h], y1[h]);
      x0[h] >>= kSTShift; x1[h] >>= kSTShift; y0[h] >>= kSTShift; y1[h] >>= kSTShift;
      cnt[h] = (uint32_t)((x1[h] - x0[h] + 1) * (y1[h] - y0[h] + 1));
    }
  }
  {
    unsigned long long *cm = mk + warp * mw;
    unsigned long long *rm = cm + sx;
    for (int x = 0; x < sx; ++x) {
      const uint32_t lo = __ballot_sync(0xffffffffu, x0[0] <= x && x <= x1[0]);
      const uint32_t hi = __ballot_sync(0xffffffffu, x0[1] <= x && x <= x1[1]);
      if (lane == (x & 31)) cm[x] = (unsigned long long)lo | ((unsigned long long)hi << 32);
    }
    for (int y = 0; y < sy; ++y) {
      const uint32_t lo = __ballot_sync(0xffffffffu, y0[0] <= y && y <= y1[0]);
      const uint32_t hi = __ballot_sync(0xffffffffu, y0[1] <= y && y <= y1[1]);
      if (lane == (y & 31)) rm[y] = (unsigned long long)lo | ((unsigned long long)hi << 32);
    }
  }
  __syncthreads();  // every group's masks are complete
  const uint16_t *crel = rel + (size_t)c * NS;
  const uint32_t *sb = segbase + (size_t)(c / kSeg) * NS;
  // each thread enumerates its own two Gaussians' entries (a handful each)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (cnt[h] == 0) continue;
    const int k = warp * 64 + h * 32 + lane;
    const int g = warp;
    const unsigned long long below = (1ull << (k & 63)) - 1ull;
    for (int ty = y0[h]; ty <= y1[h]; ++ty)
      for (int tx = x0[h]; tx <= x1[h]; ++tx) {
        const uint32_t t = (uint32_t)ty * sx + (uint32_t)tx;
        const unsigned long long *cg = mk + g * mw;
        uint32_t pos = __ldg(soff + t) + __ldg(sb + t) + (uint32_t)__ldg(crel + t) +
                       (uint32_t)__popcll(cg[tx] & cg[sx + ty] & below);
        for (int w = 0; w < g; ++w) {
          const unsigned long long *cw = mk + w * mw;
          pos += (uint32_t)__popcll(cw[tx] & cw[sx + ty]);
        }
        entries[pos] = j0 + (uint32_t)k;
      }
  }
}

// L2.  A super-tile's entry list (depth order) is cut into units of <= kPUnit
// entries; CTAs map to (super-tile, unit) through a prefix over the super-tiles.
// Rounds of 512 entries: warp w builds 8 column and 8 row ballots over its 32
// entries, lane L owns tiles L and L + 32 of the super-tile (mask of entries
// covering it).
constexpr int kPRound = kPlaceWarps * 32;

__device__ __forceinline__ void place_masks(uint2 rc, bool ok, int stx0, int sty0, int lane, uint32_t &m0,
                                            uint32_t &m1) {
  int x0, y0, x1, y1;
  unpack_rect(rc, x0, y0, x1, y1);
  x0 -= stx0; x1 -= stx0; y0 -= sty0; y1 -= sty0;
  const int cx = lane & 7, cy = lane >> 3;
  uint32_t col = 0, r0 = 0, r1 = 0;
#pragma unroll
  for (int q = 0; q < kST; ++q) {
    const uint32_t bc = __ballot_sync(0xffffffffu, ok && x0 <= q && q <= x1);
    const uint32_t br = __ballot_sync(0xffffffffu, ok && y0 <= q && q <= y1);
    if (cx == q) col = bc;
    if (cy == q) r0 = br;
    if (cy + 4 == q) r1 = br;
  }
  m0 = col & r0;
  m1 = col & r1;
}

// Unit table: ubase[S] = units before super-tile S (ubase[NS] = total), utab[u] = S.
__global__ void __launch_bounds__(1024) k_unit_table(const uint32_t *__restrict__ soff, uint32_t NS,
                                                     uint32_t *__restrict__ ubase, uint32_t *__restrict__ utab) {
  __shared__ uint32_t ws[32];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < NS; b0 += blockDim.x) {
    const uint32_t s = b0 + threadIdx.x;
    const uint32_t n = s < NS ? ceil_div<uint32_t>(soff[s + 1] - soff[s], kPUnit) : 0u;
    uint32_t tot;
    const uint32_t ex = carry + block_exclusive_scan(n, ws, &tot);
    if (s < NS) {
      ubase[s] = ex;
      for (uint32_t k = 0; k < n; ++k) utab[ex + k] = s;
    }
    carry += tot;
  }
  if (threadIdx.x == 0) ubase[NS] = carry;
}

// (super-tile, first entry, end entry) of unit u; false past the last unit
__device__ __forceinline__ bool place_unit(const uint32_t *__restrict__ soff, const uint32_t *__restrict__ ubase,
                                           const uint32_t *__restrict__ utab, uint32_t NS, uint32_t u, uint32_t &S,
                                           uint32_t &ea, uint32_t &eb) {
  if (u >= __ldg(ubase + NS)) return false;
  S = __ldg(utab + u);
  ea = __ldg(soff + S) + (u - __ldg(ubase + S)) * kPUnit;
  eb = tmin<uint32_t>(ea + kPUnit, __ldg(soff + S + 1));
  return true;
}

// Pass 1: per (unit, tile-of-super-tile) instance counts.
__global__ void __launch_bounds__(kPlaceWarps * 32) k_place_count(const uint32_t *__restrict__ entries,
                                                                   const uint32_t *__restrict__ soff,
                                                                   const uint32_t *__restrict__ ubase,
                                                                   const uint32_t *__restrict__ utab,
                                                                   const uint2 *__restrict__ rects, int sx,
                                                                   uint32_t NS, uint32_t *__restrict__ ucnt) {
  __shared__ uint32_t wc[kPlaceWarps][64];
  uint32_t S, ea, eb;
  if (!place_unit(soff, ubase, utab, NS, blockIdx.x, S, ea, eb)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int stx0 = (int)(S % sx) * kST, sty0 = (int)(S / sx) * kST;
  uint32_t n0 = 0, n1 = 0;
  for (uint32_t b = ea + warp * 32; b < eb; b += kPRound) {
    const bool ok = b + lane < eb;
    const uint2 rc = ok ? __ldg(rects + __ldg(entries + b + lane)) : make_uint2(0, 0);
    uint32_t m0, m1;
    place_masks(rc, ok, stx0, sty0, lane, m0, m1);
    n0 += __popc(m0);
    n1 += __popc(m1);
  }
  wc[warp][lane] = n0;
  wc[warp][lane + 32] = n1;
  __syncthreads();
  if (threadIdx.x < 64) {
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < kPlaceWarps; ++w) r += wc[w][threadIdx.x];
    ucnt[(size_t)blockIdx.x * 64 + threadIdx.x] = r;
  }
}

// Per tile: exclusive scan of its super-tile's unit counts (in place), the tile
// total, and the CSR offsets (blocks of 256 tiles chained by look-back).
__global__ void __launch_bounds__(256) k_tile_scan(const uint32_t *__restrict__ ubase, int sx, int tiles_x,
                                                   int rows, uint32_t *__restrict__ ucnt,
                                                   uint32_t *__restrict__ status, uint32_t *__restrict__ ticket,
                                                   int32_t *__restrict__ offsets) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t s_blk, s_excl;
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t T = (uint32_t)(rows * tiles_x);
  const uint32_t t = s_blk * blockDim.x + threadIdx.x;
  uint32_t run = 0;
  if (t < T) {
    const int ty = (int)(t / tiles_x), tx = (int)(t % tiles_x);
    const uint32_t S = (uint32_t)((ty >> kSTShift) * sx + (tx >> kSTShift));
    const uint32_t q = (uint32_t)(((ty & (kST - 1)) << kSTShift) | (tx & (kST - 1)));
    const uint32_t u1 = __ldg(ubase + S + 1);
    for (uint32_t u = __ldg(ubase + S); u < u1; u += 8) {  // independent loads first
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = u + k < u1 ? ucnt[(size_t)(u + k) * 64 + q] : 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (u + k < u1) {
          ucnt[(size_t)(u + k) * 64 + q] = run;
          run += v[k];
        }
    }
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan(run, ws, &tot);
  if (threadIdx.x == 0) s_excl = lookback<16>(status, 1, s_blk, tot);
  __syncthreads();
  if (t < T) {
    offsets[t] = (int32_t)(s_excl + ex);
    if (t == T - 1) offsets[T] = (int32_t)(s_excl + ex + run);
  }
}

// Pass 2: rounds of 512 entries.  Per round and tile, the run of ids (entries of
// all warps covering the tile, in entry order) is assembled in shared memory —
// lane l of warp w writes, for its tiles l and l + 32, the ids of w's entries
// covering them (set bits of the coverage mask, in order) at the tile's run
// start + w's prefix — and then copied out by consecutive lanes (coalesced).
constexpr int kStage = 8192;

__global__ void __launch_bounds__(kPlaceWarps * 32) k_place_write(const uint32_t *__restrict__ entries,
                                                                   const uint32_t *__restrict__ soff,
                                                                   const uint32_t *__restrict__ ubase,
                                                                   const uint32_t *__restrict__ utab,
                                                                   const uint2 *__restrict__ rects,
                                                                   const uint32_t *__restrict__ ids, int sx,
                                                                   uint32_t NS, int tiles_x, int rows,
                                                                   const uint32_t *__restrict__ ucnt,
                                                                   const int32_t *__restrict__ offsets,
                                                                   int32_t *__restrict__ sorted_ids) {
  __shared__ uint32_t mk[kPlaceWarps][64];     // entries of warp w covering tile q
  __shared__ uint32_t pre[kPlaceWarps][64];    // exclusive over warps
  __shared__ uint32_t len[64], sst[64], cur[64];
  __shared__ uint32_t s_total;
  __shared__ uint32_t sg[kPlaceWarps][32];       // the round's cloud ids, per warp
  __shared__ uint32_t stage[kStage];
  uint32_t S, ea, eb;
  if (!place_unit(soff, ubase, utab, NS, blockIdx.x, S, ea, eb)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const int stx0 = (int)(S % sx) * kST, sty0 = (int)(S / sx) * kST;
  if (threadIdx.x < 64) {
    const int q = threadIdx.x, tx = stx0 + (q & 7), ty = sty0 + (q >> 3);
    cur[q] = (tx < tiles_x && ty < rows) ? (uint32_t)__ldg(offsets + ty * tiles_x + tx) +
                                               __ldg(ucnt + (size_t)blockIdx.x * 64 + q)
                                         : 0u;
  }
  for (uint32_t a = ea; a < eb; a += kPRound) {
    const uint32_t b = a + warp * 32 + lane;
    const bool ok = b < eb;
    const uint32_t j = ok ? __ldg(entries + b) : 0u;
    const uint2 rc = ok ? __ldg(rects + j) : make_uint2(0, 0);
    const uint32_t gid = ok ? __ldg(ids + j) : 0u;
    uint32_t m0, m1;
    place_masks(rc, ok, stx0, sty0, lane, m0, m1);
    mk[warp][lane] = m0;
    mk[warp][lane + 32] = m1;
    __syncthreads();
    if (threadIdx.x < 64) {
      uint32_t r = 0;
#pragma unroll
      for (int w = 0; w < kPlaceWarps; ++w) {
        pre[w][threadIdx.x] = r;
        r += __popc(mk[w][threadIdx.x]);
      }
      len[threadIdx.x] = r;
    }
    __syncthreads();
    if (warp == 0) {  // run starts in the stage: exclusive scan over the 64 tiles
      const uint32_t l0 = len[2 * lane], l1 = len[2 * lane + 1];
      uint32_t v = l0 + l1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      const uint32_t ex = v - l0 - l1;
      sst[2 * lane] = ex;
      sst[2 * lane + 1] = ex + l0;
      if (lane == 31) s_total = v;
    }
    __syncthreads();
    const uint32_t total = s_total;
    if (total <= (uint32_t)kStage) {
      // lane owns tiles `lane` and `lane + 32`: it writes the ids of the warp's entries
      // covering them, in entry order (set bits of the coverage mask)
      sg[warp][lane] = gid;
      __syncwarp();
#pragma unroll
      for (int hq = 0; hq < 2; ++hq) {
        const int q = lane + 32 * hq;
        uint32_t mq = hq ? m1 : m0;
        uint32_t slot = sst[q] + pre[warp][q];
        while (mq) {
          const int k = __ffs(mq) - 1;
          mq &= mq - 1;
          stage[slot++] = sg[warp][k];
        }
      }
      __syncthreads();
      for (int q = warp; q < 64; q += kPlaceWarps) {
        const uint32_t l = len[q], so = sst[q], base = cur[q];
        for (uint32_t i = lane; i < l; i += 32) sorted_ids[base + i] = (int32_t)stage[so + i];
      }
    } else {  // oversized round (huge rects): each entry writes its ids directly
      if (ok) {
        int x0, y0, x1, y1;
        unpack_rect(rc, x0, y0, x1, y1);
        x0 = max(x0 - stx0, 0); x1 = min(x1 - stx0, kST - 1);
        y0 = max(y0 - sty0, 0); y1 = min(y1 - sty0, kST - 1);
        for (int y = y0; y <= y1; ++y)
          for (int x = x0; x <= x1; ++x) {
            const int q = y * kST + x;
            sorted_ids[cur[q] + pre[warp][q] + __popc(mk[warp][q] & lt)] = (int32_t)gid;
          }
      }
    }
    __syncthreads();
    if (threadIdx.x < 64) cur[threadIdx.x] += len[threadIdx.x];
    __syncthreads();
  }
}

struct InstWS {
  uint16_t *rel;
  uint32_t *segsum, *soff, *entries, *ucnt, *status, *ticket, *chunk_ent, *tstatus, *tticket, *ubase, *utab;
  size_t zero_off, zero_bytes, bytes;
};

static InstWS carve_inst(void *p, const InstGeom &g) {
  Carve c(p);
  InstWS w;
  w.rel = c.take<uint16_t>((size_t)g.nchunks * g.NS);
  w.segsum = c.take<uint32_t>((size_t)g.nseg * g.NS);
  w.soff = c.take<uint32_t>(g.NS + 1);
  w.entries = c.take<uint32_t>(g.ecap);
  w.ucnt = c.take<uint32_t>((size_t)g.punits * 64);
  w.ubase = c.take<uint32_t>(g.NS + 1);
  w.utab = c.take<uint32_t>(g.punits);
  w.zero_off = c.off;
  w.ticket = c.take<uint32_t>(1);
  w.status = c.take<uint32_t>(ceil_div<uint32_t>(g.NS, kScanCols));
  w.chunk_ent = c.take<uint32_t>(g.nchunks);
  w.tticket = c.take<uint32_t>(1);
  w.tstatus = c.take<uint32_t>(ceil_div<uint32_t>(g.T, 256));
  w.zero_bytes = c.off - w.zero_off;
  w.bytes = c.off;
  return w;
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

// Debug: record per-ticket phase timestamps of the depth sort into `buf`
// (8 u64 per ticket; null disables).  Not part of the product API.
extern "C" __attribute__((visibility("default"))) int tgs_debug_trace_depth_sort(unsigned long long *buf) {
  return cuda_status(cudaMemcpyToSymbol(g_ds_trace, &buf, sizeof(buf)));
}

extern "C" int tgs_bin_gaussians_workspace(int64_t n, size_t *bytes) {
  if (n < 0 || !bytes) return TGS_ERR_INVALID;
  *bytes = carve_gauss(nullptr, n).bytes;
  return TGS_OK;
}

extern "C" int tgs_bin_gaussians(const float *splats, const int32_t *tiles_touched, const uint64_t *depth_keys,
                                 int64_t n, int32_t width,
                                 int32_t height, int32_t tile_size, int32_t row_begin, int32_t row_end,
                                 void *workspace, int64_t *d_num_instances, const int32_t *error_flag,
                                 tgs_stream_t stream) {
  Band b;
  if (n < 0 || n >= (int64_t)1 << 30 || !workspace || !d_num_instances ||
      !band_ok(width, height, tile_size, row_begin, row_end, b))
    return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  GaussWS w = carve_gauss(workspace, n);
  k_bs_init<<<1, 32, 0, st>>>(w.bctl, reinterpret_cast<unsigned long long *>(d_num_instances), error_flag);
  if (n == 0) return launch_status();
  BsArgs ba;
  ba.splats = splats;
  ba.tiles_touched = tiles_touched;
  ba.depth_keys = depth_keys;
  ba.n = (uint32_t)n;
  ba.b = b;
  ba.ctl = w.bctl;
  ba.rect_by_gid = w.rect_by_gid;
  ba.bcount = w.bcount;
  ba.boff = w.boff;
  ba.bstatus = w.bstatus;
  ba.keys = w.keysA;
  ba.vals = w.valsA;
  ba.ids = w.ids;
  ba.rects_sorted = w.rects_sorted;
  ba.num_instances = reinterpret_cast<unsigned long long *>(d_num_instances);
  ba.zero = reinterpret_cast<uint32_t *>(static_cast<char *>(workspace) + w.zero_off);
  ba.zero_words = w.zero_bytes / 4;  // fallback state + scan look-back words
  const unsigned g = (unsigned)ceil_div<int64_t>(n, 256);
  k_bs_select<<<(unsigned)tmin<int64_t>(g, 148 * 8), 256, 0, st>>>(ba);
  k_bs_hist<<<g, 256, 0, st>>>(ba);
  k_bs_scan<<<kBuckets / kBScanTile, 256, 0, st>>>(ba);
  k_bs_scatter<<<g, 256, 0, st>>>(ba);
  k_bs_rank<<<g, 256, 0, st>>>(ba);
  // fallback: the ticketed LSD chain, only if a bucket overflowed
  DsArgs a;
  a.splats = splats;
  a.tiles_touched = tiles_touched;
  a.depth_keys = depth_keys;
  a.n = (uint32_t)n;
  a.b = b;
  a.keysA = w.keysA; a.keysB = w.keysB;
  a.valsA = w.valsA; a.valsB = w.valsB;
  a.ctl = w.ctl;
  a.rect_by_gid = w.rect_by_gid;
  a.rects_sorted = w.rects_sorted;
  a.ids = w.ids;
  a.status = w.status;
  a.T0 = w.T0;
  a.TP = w.TP;
  a.num_instances = nullptr;
  static std::atomic<uint64_t> attr_done{0};
  const int arc = attr_once_per_device(attr_done, [] {
    return cudaFuncSetAttribute(k_depth_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DsSmem));
  });
  if (arc != TGS_OK) return arc;
  const unsigned fg = (unsigned)tmin<uint64_t>((uint64_t)w.T0 + kDsPasses * w.TP, 148 * 3);
  k_depth_sort<<<fg, kDsThreads, sizeof(DsSmem), st>>>(a, &w.bctl->overflow);
  return launch_status();
}

extern "C" int tgs_bin_instances_workspace(int64_t n, int64_t num_instances, int32_t width, int32_t height,
                                           int32_t tile_size, int32_t row_begin, int32_t row_end, size_t *bytes) {
  Band b;
  if (n < 0 || num_instances < 0 || !bytes || !band_ok(width, height, tile_size, row_begin, row_end, b))
    return TGS_ERR_INVALID;
  *bytes = carve_inst(nullptr, inst_geom(n, num_instances, b)).bytes;
  return TGS_OK;
}

extern "C" int tgs_bin_instances(const float *splats, int64_t n, int32_t width, int32_t height, int32_t tile_size,
                                 int32_t row_begin, int32_t row_end, void *gauss_workspace, int64_t num_instances,
                                 void *workspace, int32_t *tile_offsets, int32_t *sorted_ids, tgs_stream_t stream) {
  Band b;
  if (n < 0 || num_instances < 0 || num_instances >= (int64_t)1 << 31 || !gauss_workspace || !tile_offsets ||
      !band_ok(width, height, tile_size, row_begin, row_end, b))
    return TGS_ERR_INVALID;
  if (num_instances >= (int64_t)1 << 30) return TGS_ERR_UNSUPPORTED;  // 30-bit look-back payloads
  cudaStream_t st = as_stream(stream);
  const InstGeom g = inst_geom(n, num_instances, b);
  const int rows = b.row_end - b.row_begin;
  if (num_instances == 0) {
    k_fill_i32<<<(unsigned)ceil_div<int64_t>(g.T + 1, 256), 256, 0, st>>>(tile_offsets, g.T + 1, 0);
    return launch_status();
  }
  if (!workspace || !sorted_ids) return TGS_ERR_INVALID;
  const size_t sc_smem = (size_t)kChunkWarps * (g.sx + g.sy) * 8;
  const size_t cnt_smem = ((size_t)(g.sx + 1) * (g.slab_rows + 1) + (size_t)g.slab_rows * g.sx) * 4;
  if (sc_smem > 160 * 1024) return TGS_ERR_UNSUPPORTED;
  GaussWS gw = carve_gauss(gauss_workspace, n);
  InstWS w = carve_inst(workspace, g);
  const uint32_t *d_m = &gw.bctl->m;
  static std::atomic<uint64_t> attr_done{0};
  const int arc = attr_once_per_device(attr_done, [] {
    const cudaError_t e = cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    return e != cudaSuccess ? e
                            : cudaFuncSetAttribute(k_seg_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   2 * kDiffCells * 4);
  });
  if (arc != TGS_OK) return arc;
  cudaMemsetAsync(static_cast<char *>(workspace) + w.zero_off, 0, w.zero_bytes, st);
  k_seg_count<<<dim3(g.nseg, g.slabs), 256, cnt_smem, st>>>(gw.rects_sorted, d_m, g.sx, g.slab_rows, g.sy, w.rel,
                                                           w.segsum, w.chunk_ent);
  k_seg_base<<<ceil_div<uint32_t>(g.NS, kScanCols), kScanCols * kScanGroups, 0, st>>>(w.segsum, d_m, g.NS, w.status,
                                                                                    w.ticket, w.soff);
  k_scatter<<<g.nchunks, kChunkWarps * 32, sc_smem, st>>>(gw.rects_sorted, d_m, g.sx, g.sy, w.chunk_ent, w.rel,
                                                      w.segsum, w.soff, w.entries);
  k_unit_table<<<1, 1024, 0, st>>>(w.soff, g.NS, w.ubase, w.utab);
  k_place_count<<<g.punits, kPlaceWarps * 32, 0, st>>>(w.entries, w.soff, w.ubase, w.utab, gw.rects_sorted, g.sx,
                                                       g.NS, w.ucnt);
  k_tile_scan<<<ceil_div<uint32_t>(g.T, 256), 256, 0, st>>>(w.ubase, g.sx, b.tiles_x, rows, w.ucnt, w.tstatus,
                                                           w.tticket, tile_offsets);
  k_place_write<<<g.punits, kPlaceWarps * 32, 0, st>>>(w.entries, w.soff, w.ubase, w.utab, gw.rects_sorted, gw.ids,
                                                       g.sx, g.NS,
                                                       b.tiles_x, rows, w.ucnt, tile_offsets, sorted_ids);
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

// The binning round trip's device -> host read (the caller's pinned buffer) on an
// explicit stream: lets a host pipeline read a view's counts without switching its
// framework's current stream.
extern "C" int tgs_memcpy_d2h_async(void *dst_host, const void *src_device, size_t bytes, tgs_stream_t stream) {
  if (!dst_host || !src_device) return TGS_ERR_INVALID;
  return cuda_status(cudaMemcpyAsync(dst_host, src_device, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
}
