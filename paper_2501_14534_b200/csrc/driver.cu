// driver.cu — native host pipelines for a batch of views of one cloud.
//
// tgs_render_views: the per-view sequence of render_forward (rasterizer.py:215-284 on the
// CUDA path):
//   preprocess (all views, one pass over the parameters) [+ exact blend-decision records]
//   per view:  bin_gaussians -> instance count to the host -> bin_instances -> blend_forward
// tgs_train_views: the per-view half of a training step (training.py:296-309 per view,
// train.Trainer): after the caller's multi-view preprocess, per view
//   bin_gaussians -> count -> bin_instances -> blend_forward -> L1 + D-SSIM loss
//   (dL/dimage) -> blend_backward (screen-space partials)
// and the caller finishes with ONE multi-view preprocess backward and the fused Adam.
//
// Both issue the views from C++ over the caller's streams, round-robin; each stream runs
// bin_instances(v) -> bin_gaussians(v + nstreams) -> blend(v) [-> loss(v) -> backward(v)],
// so a view's count read-back overlaps the previous same-stream view's blend and never
// sits on a stream's critical path.  Driven from Python the loop costs ~15 launches and a
// read-back of Python per view and is host-bound at small resolutions; here the host cost
// per view is the CUDA API calls alone.
//
// The library allocates nothing: outputs, per-stream workspaces and the pinned count slots
// are the caller's.  A view whose instance count exceeds its id capacity (or the
// workspace) stops the batch with TGS_ERR_CAPACITY after writing every view's count to
// targets[].num_instances (-1 = not reached); the caller grows its buffers and calls again.
#include <memory>
#include <vector>

#include "tgs_common.cuh"

namespace {

using tgs::cuda_status;

constexpr int kMaxStreams = 8;

inline size_t align256(size_t v) { return (v + 255) / 256 * 256; }

struct Slot {  // one stream's share of the caller's workspace
  char *base;
  void *ws_g;
  int64_t *counts;  // device (count, error flag)
  void *ws_i;
  size_t ws_i_bytes;
};

// The events of a batch.  Creating and destroying them per call (up to 2 + 2 x 8) cost
// host time before the batch's first launch, so each thread keeps one set per device and
// re-records it every batch (a wait issued by an earlier batch captured that batch's
// record; reuse is safe).  Destroyed with the thread.
struct Events {
  cudaEvent_t pre = nullptr, ex = nullptr, count[kMaxStreams] = {}, blend[kMaxStreams] = {};
  bool ready = false;
  ~Events() {
    if (pre) cudaEventDestroy(pre);
    if (ex) cudaEventDestroy(ex);
    for (int k = 0; k < kMaxStreams; ++k) {
      if (count[k]) cudaEventDestroy(count[k]);
      if (blend[k]) cudaEventDestroy(blend[k]);
    }
  }
  static bool make(cudaEvent_t &e) { return cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess; }
  int create() {
    if (ready) return TGS_OK;
    if (!make(pre) || !make(ex)) return cuda_status(cudaGetLastError());
    for (int k = 0; k < kMaxStreams; ++k)
      if (!make(count[k]) || !make(blend[k])) return cuda_status(cudaGetLastError());
    ready = true;
    return TGS_OK;
  }
};

// this thread's event set for the current device
int batch_events(Events *&E) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return TGS_ERR_CUDA;
  thread_local std::vector<std::unique_ptr<Events>> sets;
  if ((size_t)dev >= sets.size()) sets.resize((size_t)dev + 1);
  if (!sets[dev]) sets[dev] = std::make_unique<Events>();
  E = sets[dev].get();
  return E->create();  // a partial failure keeps what was made (destroyed with the thread)
}

struct Batch {
  const tgs_cloud *cloud;
  const tgs_camera *cams;
  const tgs_settings *s;
  int nviews;
  float *const *splats;
  uint8_t *const *visible;
  int32_t *const *tiles_touched;
  uint64_t *const *depth_keys;
  float *const *exact;
  int32_t *error_flag;
  tgs_view_target *targets;
  void *const *workspaces;
  size_t workspace_bytes;
  int64_t *pinned_counts;
  const tgs_stream_t *streams;
  const tgs_stream_t *blend_streams;
  int nstreams;
  bool preprocess;              // run the multi-view preprocess (+ exact records) first
  void *exact_ready;            // else: the caller's event after which the exact records are complete
  const tgs_view_train *train;  // per-view loss + backward (tgs_train_views), or NULL
  float lambda_ssim;
};

int run_views(const Batch &B) {
  if (!B.cloud || !B.cams || !B.s || B.nviews < 1 || !B.splats || !B.visible || !B.tiles_touched || !B.targets ||
      !B.workspaces || !B.pinned_counts || !B.streams || B.nstreams < 1 || B.nstreams > kMaxStreams ||
      !B.error_flag)
    return TGS_ERR_INVALID;
  const int64_t n = B.cloud->n;
  for (int v = 0; v < B.nviews; ++v) B.targets[v].num_instances = -1;
  if (n == 0) return TGS_ERR_INVALID;  // callers render empty clouds through render_forward
  size_t gbytes = 0;
  int rc = tgs_bin_gaussians_workspace(n, &gbytes);
  if (rc != TGS_OK) return rc;
  const size_t off_counts = align256(gbytes), off_i = off_counts + 256;
  if (B.workspace_bytes < off_i) return TGS_ERR_CAPACITY;
  Slot slot[kMaxStreams];
  for (int k = 0; k < B.nstreams; ++k) {
    if (!B.workspaces[k]) return TGS_ERR_INVALID;
    char *b = static_cast<char *>(B.workspaces[k]);
    slot[k] = Slot{b, b, reinterpret_cast<int64_t *>(b + off_counts), b + off_i, B.workspace_bytes - off_i};
  }
  Events *Ep = nullptr;
  rc = batch_events(Ep);
  if (rc != TGS_OK) return rc;
  Events &E = *Ep;
  auto stream = [](tgs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); };
  cudaStream_t st0 = stream(B.streams[0]);
  // 1. every view's preprocess in one pass over the parameters (stream 0), or the caller's
  if (B.preprocess) {
    rc = tgs_preprocess_forward_views(B.cloud, B.cams, B.s, B.nviews, B.splats, B.visible, B.tiles_touched,
                                      B.depth_keys, B.error_flag, nullptr, nullptr, B.streams[0]);
    if (rc != TGS_OK) return rc;
  }
  if (cudaEventRecord(E.pre, st0) != cudaSuccess) return cuda_status(cudaGetLastError());
  for (int k = 1; k < B.nstreams; ++k) cudaStreamWaitEvent(stream(B.streams[k]), E.pre, 0);
  // 1b. the exact blend-decision records on a blend stream (the depth sorts do not read
  // them, so the latency-bound binning of the first views runs alongside); every blend
  // waits for them
  cudaEvent_t ex_ready = static_cast<cudaEvent_t>(B.exact_ready);
  if (B.preprocess && B.exact) {
    tgs_stream_t xs = B.blend_streams ? B.blend_streams[0] : B.streams[B.nstreams - 1];
    if (stream(xs) != st0) cudaStreamWaitEvent(stream(xs), E.pre, 0);
    rc = tgs_exact_records_views(B.cloud, B.cams, B.s, B.nviews, const_cast<const float *const *>(B.splats), B.exact,
                                 xs);
    if (rc != TGS_OK) return rc;
    if (cudaEventRecord(E.ex, stream(xs)) != cudaSuccess) return cuda_status(cudaGetLastError());
    ex_ready = E.ex;
  }

  const tgs_camera *cams = B.cams;
  const int ts = B.s->tile_size;
  // the view's tile-row band (tile-row sharding), the whole view by default
  auto rb_of = [&](int v) { return B.targets[v].row_end > 0 ? B.targets[v].row_begin : 0; };
  auto rows_of = [&](int v) {
    return B.targets[v].row_end > 0 ? B.targets[v].row_end : (cams[v].height + ts - 1) / ts;
  };
  // 2a. depth sort of view v + asynchronous read of its instance count
#ifdef TGS_EXP_SKIP_BIN  // experiment builds only (profiles/binning_cost_exp.py): after 3 batches, reuse
  static int calls = 0;   // the views' tile lists of the previous batch (a static scene) and skip binning
  const bool skip_bin = ++calls > 3;
#else
  constexpr bool skip_bin = false;
#endif
  auto begin = [&](int v) -> int {
    const int k = v % B.nstreams;
    if (skip_bin) return cudaEventRecord(E.count[k], stream(B.streams[k])) == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
    int r = tgs_bin_gaussians(B.splats[v], B.tiles_touched[v], B.depth_keys ? B.depth_keys[v] : nullptr, n,
                              cams[v].width, cams[v].height, ts, rb_of(v), rows_of(v), slot[k].ws_g, slot[k].counts,
                              B.error_flag, B.streams[k]);
    if (r != TGS_OK) return r;
    if (cudaMemcpyAsync(B.pinned_counts + 2 * k, slot[k].counts, 16, cudaMemcpyDeviceToHost, stream(B.streams[k])) !=
        cudaSuccess)
      return TGS_ERR_CUDA;
    return cudaEventRecord(E.count[k], stream(B.streams[k])) == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
  };
  // 2b. wait for view v's count and place its instances
  auto place = [&](int v) -> int {
    const int k = v % B.nstreams;
    if (cudaEventSynchronize(E.count[k]) != cudaSuccess) return TGS_ERR_CUDA;
    if (skip_bin) {
      B.targets[v].num_instances = 0;
      return TGS_OK;
    }
    const int64_t count = B.pinned_counts[2 * k], flag = B.pinned_counts[2 * k + 1];
    if (flag) return TGS_ERR_DEGENERATE_ROTATION;
    tgs_view_target &t = B.targets[v];
    t.num_instances = count;
    size_t need = 0;
    int r = tgs_bin_instances_workspace(n, count, cams[v].width, cams[v].height, ts, rb_of(v), rows_of(v), &need);
    if (r != TGS_OK) return r;
    if (count > t.ids_capacity || need > slot[k].ws_i_bytes) return TGS_ERR_CAPACITY;
    return tgs_bin_instances(B.splats[v], n, cams[v].width, cams[v].height, ts, rb_of(v), rows_of(v), slot[k].ws_g,
                             count, slot[k].ws_i, t.tile_offsets, t.sorted_ids, B.streams[k]);
  };
  // 2c. blend view v (on its blend stream when one is given: the binning streams then
  // run at higher priority and the blends fill the SMs around them), then for training
  // its loss and backward on the same stream
  auto blend = [&](int v) -> int {
    const int k = v % B.nstreams;
    const tgs_view_target &t = B.targets[v];
    tgs_stream_t bs = B.streams[k];
    if (B.blend_streams) {
      cudaEventRecord(E.blend[k], stream(B.streams[k]));
      cudaStreamWaitEvent(stream(B.blend_streams[k]), E.blend[k], 0);
      bs = B.blend_streams[k];
    }
    if (ex_ready) cudaStreamWaitEvent(stream(bs), ex_ready, 0);
    const float *ex = B.exact ? B.exact[v] : nullptr;
    const tgs_view_train *tr_ = B.train ? &B.train[v] : nullptr;
    int32_t *exc = tr_ && ex ? tr_->exceptions : nullptr;
    uint32_t *ovf = exc ? tr_->exc_overflow : nullptr;
    if (!ovf) exc = nullptr;
    int r = tgs_blend_forward(B.splats[v], ex, t.tile_offsets, t.sorted_ids, &cams[v], B.s, rb_of(v), rows_of(v),
                              t.image, t.transmit, t.weight_sum, t.n_contrib, t.last_pos, t.hits, exc, ovf,
                              t.tile_order, bs);
    if (r != TGS_OK || !B.train) return r;
    const tgs_view_train &tr = *tr_;
    if (tr.target_ready) cudaStreamWaitEvent(stream(bs), static_cast<cudaEvent_t>(tr.target_ready), 0);
    r = tgs_loss_l1_ssim(t.image, tr.target, cams[v].width, cams[v].height, B.lambda_ssim, tr.dimage, tr.terms,
                         tr.loss_workspace, bs);
    if (r != TGS_OK) return r;
    return tgs_blend_backward(B.splats[v], ex, t.tile_offsets, t.sorted_ids, &cams[v], B.s, rb_of(v), rows_of(v),
                              t.transmit, t.last_pos, exc, ovf, tr.dimage, tr.dsplats, t.tile_order, bs);
  };
  // Per stream k the queue is  bin_instances(v) -> bin_gaussians(v + nstreams) -> blend(v):
  // the next same-stream view's depth sort runs BEFORE this view's blend, so its count
  // reaches the host while the blend runs (bin_instances(v) has consumed the stream's
  // depth-sort workspace by then, the blend does not read it, and view v's pinned count
  // was read before the slot is refilled).
  rc = TGS_OK;
  int begun = 0, v = 0;
  for (; begun < B.nviews && begun < B.nstreams && rc == TGS_OK; ++begun) rc = begin(begun);
  for (; v < B.nviews && rc == TGS_OK; ++v) {
    rc = place(v);
    if (rc == TGS_OK && v + B.nstreams < B.nviews) {
      rc = begin(v + B.nstreams);
      ++begun;
    }
    if (rc == TGS_OK) rc = blend(v);
  }
  if (rc == TGS_ERR_CAPACITY) {
    // finish the depth sorts of the remaining views for their counts only, so the
    // caller can size every buffer before its single retry
    for (int w = v; w < B.nviews; ++w) {
      if (w >= begun) {
        if (begin(w) != TGS_OK) break;
        ++begun;
      }
      const int k = w % B.nstreams;
      if (cudaEventSynchronize(E.count[k]) != cudaSuccess) break;
      B.targets[w].num_instances = B.pinned_counts[2 * k];
    }
  }
  return rc;
}

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
                                tgs_view_target *targets, void *const *workspaces, size_t workspace_bytes,
                                int64_t *pinned_counts, const tgs_stream_t *streams,
                                const tgs_stream_t *blend_streams, int32_t nstreams) {
  return run_views(Batch{cloud, cams, s, nviews, splats, visible, tiles_touched, depth_keys, exact, error_flag,
                         targets, workspaces, workspace_bytes, pinned_counts, streams, blend_streams, nstreams,
                         /*preprocess=*/true, nullptr, nullptr, 0.0f});
}

extern "C" int tgs_train_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s, int32_t nviews,
                               float *const *splats, uint8_t *const *visible, int32_t *const *tiles_touched,
                               uint64_t *const *depth_keys, float *const *exact, void *exact_ready,
                               int32_t *error_flag, tgs_view_target *targets, const tgs_view_train *train,
                               float lambda_ssim, void *const *workspaces, size_t workspace_bytes,
                               int64_t *pinned_counts, const tgs_stream_t *streams,
                               const tgs_stream_t *blend_streams, int32_t nstreams) {
  if (!train || nviews < 1) return TGS_ERR_INVALID;
  for (int v = 0; v < nviews; ++v)
    if (!train[v].target || !train[v].dimage || !train[v].terms || !train[v].dsplats || !train[v].loss_workspace)
      return TGS_ERR_INVALID;
  return run_views(Batch{cloud, cams, s, nviews, splats, visible, tiles_touched, depth_keys, exact, error_flag,
                         targets, workspaces, workspace_bytes, pinned_counts, streams, blend_streams, nstreams,
                         /*preprocess=*/false, exact_ready, train, lambda_ssim});
}
