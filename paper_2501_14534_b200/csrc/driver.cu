// driver.cu — native host pipeline for a batch of views of one cloud (render_views).
//
// The per-view sequence of render_forward (rasterizer.py:215-284 on the CUDA path):
//   preprocess (all views, one pass over the parameters)
//   per view:  bin_gaussians -> instance count to the host -> bin_instances -> blend_forward
// issued from C++ over the caller's streams, round-robin; each stream runs
// bin_instances(v) -> bin_gaussians(v + nstreams) -> blend(v), so a view's count
// read-back overlaps the previous same-stream view's blend.  The
// render loop is host-bound when driven from Python (one count read-back per view
// and ~15 launches); here the host cost per view is the CUDA API calls alone.
//
// The library allocates nothing: outputs, per-stream workspaces and the pinned
// count slots are the caller's.  A view whose instance count exceeds its id
// capacity (or the workspace) stops the batch with TGS_ERR_CAPACITY after writing
// every view's known count to targets[].num_instances (-1 = not reached); the
// caller grows its buffers and calls again.
#include "tgs_common.cuh"

namespace {

constexpr int kMaxStreams = 8;

inline size_t align256(size_t v) { return (v + 255) / 256 * 256; }

struct Slot {  // one stream's share of the caller's workspace
  char *base;
  void *ws_g;
  int64_t *counts;  // device (count, error flag)
  void *ws_i;
  size_t ws_i_bytes;
};

}  // namespace

extern "C" int tgs_render_views_workspace(int64_t n, int64_t max_instances, int32_t width, int32_t height,
                                          int32_t tile_size, size_t *bytes) {
  if (!bytes || n < 0 || max_instances < 0 || tile_size < 1) return TGS_ERR_INVALID;
  size_t g = 0, i = 0;
  int rc = tgs_bin_gaussians_workspace(n, &g);
  if (rc != TGS_OK) return rc;
  const int32_t ty = (height + tile_size - 1) / tile_size;
  rc = tgs_bin_instances_workspace(n, max_instances, width, height, tile_size, 0, ty, &i);
  if (rc != TGS_OK) return rc;
  *bytes = align256(g) + 256 + align256(i);
  return TGS_OK;
}

extern "C" int tgs_render_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s, int32_t nviews,
                                float *const *splats, uint8_t *const *visible, int32_t *const *tiles_touched,
                                uint64_t *const *depth_keys, float *const *exact, int32_t *error_flag,
                                tgs_view_target *targets,
                                void *const *workspaces, size_t workspace_bytes, int64_t *pinned_counts,
                                const tgs_stream_t *streams, const tgs_stream_t *blend_streams, int32_t nstreams) {
  if (!cloud || !cams || !s || nviews < 1 || !splats || !visible || !tiles_touched || !targets || !workspaces ||
      !pinned_counts || !streams || nstreams < 1 || nstreams > kMaxStreams || !error_flag)
    return TGS_ERR_INVALID;
  const int64_t n = cloud->n;
  for (int v = 0; v < nviews; ++v) targets[v].num_instances = -1;
  if (n == 0) return TGS_ERR_INVALID;  // callers render empty clouds through render_forward
  size_t gbytes = 0;
  int rc = tgs_bin_gaussians_workspace(n, &gbytes);
  if (rc != TGS_OK) return rc;
  const size_t off_counts = align256(gbytes), off_i = off_counts + 256;
  if (workspace_bytes < off_i) return TGS_ERR_CAPACITY;
  Slot slot[kMaxStreams];
  for (int k = 0; k < nstreams; ++k) {
    if (!workspaces[k]) return TGS_ERR_INVALID;
    char *b = static_cast<char *>(workspaces[k]);
    slot[k] = Slot{b, b, reinterpret_cast<int64_t *>(b + off_counts), b + off_i, workspace_bytes - off_i};
  }
  cudaStream_t st0 = reinterpret_cast<cudaStream_t>(streams[0]);
  // 1. every view's preprocess in one pass over the parameters (stream 0)
  rc = tgs_preprocess_forward_views(cloud, cams, s, nviews, splats, visible, tiles_touched, depth_keys, error_flag,
                                    nullptr, nullptr, streams[0]);
  if (rc != TGS_OK) return rc;
  cudaEvent_t ev_pre, ev[kMaxStreams], ev_b[kMaxStreams];
  if (cudaEventCreateWithFlags(&ev_pre, cudaEventDisableTiming) != cudaSuccess) return TGS_ERR_CUDA;
  for (int k = 0; k < nstreams; ++k) {
    cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_b[k], cudaEventDisableTiming);
  }
  cudaEventRecord(ev_pre, st0);
  for (int k = 1; k < nstreams; ++k) cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(streams[k]), ev_pre, 0);
  // 1b. the exact blend-decision records on a blend stream (the depth sorts do not read
  // them, so the latency-bound binning of the first views runs alongside); every blend
  // waits for them
  cudaEvent_t ev_ex = nullptr;
  if (exact) {
    tgs_stream_t xs = blend_streams ? blend_streams[0] : streams[nstreams - 1];
    cudaStream_t xst = reinterpret_cast<cudaStream_t>(xs);
    if (cudaEventCreateWithFlags(&ev_ex, cudaEventDisableTiming) != cudaSuccess) rc = TGS_ERR_CUDA;
    if (rc == TGS_OK && xst != st0) cudaStreamWaitEvent(xst, ev_pre, 0);
    if (rc == TGS_OK)
      rc = tgs_exact_records_views(cloud, cams, s, nviews, const_cast<const float *const *>(splats), exact, xs);
    if (rc == TGS_OK && cudaEventRecord(ev_ex, xst) != cudaSuccess) rc = TGS_ERR_CUDA;
    if (rc != TGS_OK) {
      if (ev_ex) cudaEventDestroy(ev_ex);
      cudaEventDestroy(ev_pre);
      for (int k = 0; k < nstreams; ++k) {
        cudaEventDestroy(ev[k]);
        cudaEventDestroy(ev_b[k]);
      }
      return rc;
    }
  }

  const int ts = s->tile_size;
  // the view's tile-row band (tile-row sharding), the whole view by default
  auto rb_of = [&](int v) { return targets[v].row_end > 0 ? targets[v].row_begin : 0; };
  auto rows_of = [&](int v) {
    return targets[v].row_end > 0 ? targets[v].row_end : (cams[v].height + ts - 1) / ts;
  };
  // 2a. depth sort of view v + asynchronous read of its instance count
  auto begin = [&](int v) -> int {
    const int k = v % nstreams;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(streams[k]);
    int r = tgs_bin_gaussians(splats[v], tiles_touched[v], depth_keys ? depth_keys[v] : nullptr, n, cams[v].width,
                              cams[v].height, ts, rb_of(v), rows_of(v), slot[k].ws_g, slot[k].counts, error_flag,
                              streams[k]);
    if (r != TGS_OK) return r;
    if (cudaMemcpyAsync(pinned_counts + 2 * k, slot[k].counts, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return TGS_ERR_CUDA;
    return cudaEventRecord(ev[k], st) == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
  };
  // 2b. wait for view v's count and place its instances
  auto place = [&](int v) -> int {
    const int k = v % nstreams;
    if (cudaEventSynchronize(ev[k]) != cudaSuccess) return TGS_ERR_CUDA;
    const int64_t count = pinned_counts[2 * k], flag = pinned_counts[2 * k + 1];
    if (flag) return TGS_ERR_DEGENERATE_ROTATION;
    tgs_view_target &t = targets[v];
    t.num_instances = count;
    size_t need = 0;
    int r = tgs_bin_instances_workspace(n, count, cams[v].width, cams[v].height, ts, rb_of(v), rows_of(v), &need);
    if (r != TGS_OK) return r;
    if (count > t.ids_capacity || need > slot[k].ws_i_bytes) return TGS_ERR_CAPACITY;
    return tgs_bin_instances(splats[v], n, cams[v].width, cams[v].height, ts, rb_of(v), rows_of(v), slot[k].ws_g, count,
                             slot[k].ws_i, t.tile_offsets, t.sorted_ids, streams[k]);
  };
  // 2c. blend view v (on its blend stream when one is given: the binning streams then
  // run at higher priority and the blends fill the SMs around them)
  auto blend = [&](int v) -> int {
    const int k = v % nstreams;
    const tgs_view_target &t = targets[v];
    tgs_stream_t bs = streams[k];
    if (blend_streams) {
      cudaEventRecord(ev_b[k], reinterpret_cast<cudaStream_t>(streams[k]));
      cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(blend_streams[k]), ev_b[k], 0);
      bs = blend_streams[k];
    }
    if (ev_ex) cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(bs), ev_ex, 0);
    return tgs_blend_forward(splats[v], exact ? exact[v] : nullptr, t.tile_offsets, t.sorted_ids, &cams[v], s, rb_of(v), rows_of(v), t.image, t.transmit,
                             t.weight_sum, t.n_contrib, t.last_pos, t.hits, t.tile_order, bs);
  };
  // Per stream k the queue is  bin_instances(v) -> bin_gaussians(v + nstreams) -> blend(v):
  // the next same-stream view's depth sort runs BEFORE this view's blend, so its count
  // reaches the host while the blend runs and the round trip never sits on the
  // stream's critical path (bin_instances(v) has consumed the stream's depth-sort
  // workspace by then, the blend does not read it, and view v's pinned count was read
  // before the slot is refilled).
  rc = TGS_OK;
  int begun = 0, v = 0;
  for (; begun < nviews && begun < nstreams && rc == TGS_OK; ++begun) rc = begin(begun);
  for (; v < nviews && rc == TGS_OK; ++v) {
    rc = place(v);
    if (rc == TGS_OK && v + nstreams < nviews) {
      rc = begin(v + nstreams);
      ++begun;
    }
    if (rc == TGS_OK) rc = blend(v);
  }
  if (rc == TGS_ERR_CAPACITY) {
    // finish the depth sorts of the remaining views for their counts only, so the
    // caller can size every buffer before its single retry
    for (int w = v; w < nviews; ++w) {
      if (w >= begun) {
        if (begin(w) != TGS_OK) break;
        ++begun;
      }
      const int k = w % nstreams;
      if (cudaEventSynchronize(ev[k]) != cudaSuccess) break;
      targets[w].num_instances = pinned_counts[2 * k];
    }
  }
  cudaEventDestroy(ev_pre);
  if (ev_ex) cudaEventDestroy(ev_ex);
  for (int k = 0; k < nstreams; ++k) {
    cudaEventDestroy(ev[k]);
    cudaEventDestroy(ev_b[k]);
  }
  return rc;
}
