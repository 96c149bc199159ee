"""Multi-view training step over the CUDA rasterizer (the hot path's caller).

Restates the per-step body of the reference's `train_step` (training.py:248-366)
for a BATCH of views, which is how BASELINE.json config 3 defines the step:

    for each view of this rank:  render_forward -> L1 + D-SSIM loss -> render_backward
                                 (gradients accumulated into one flat buffer)
    data parallel (N > 1): ZeRO-1 (default), Gaussian-sharded all-to-alls or one
                                 all-reduce of the flat gradient buffer (dp_mode)
    mask-penalty gradients + Adam over the 8 parameter groups, one fused launch
                                 (masking.py:60-67, training.py:310-331)

The batch gradient is the sum of per-view reference gradients (SURVEY.md
§8(d): "define batch gradient = sum of per-view reference gradients"), so the
all-reduced result is independent of how views are sharded over ranks.
Densification/pruning events are not part of the timed step (they are
scheduled events).
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import loss as loss_mod
from .cloud import PARAM_FIELDS, CloudGrads, GaussianCloud
from .errors import DivergenceError
from .optim import Adam
from .profiler import stage
from .rasterizer import (RenderSettings, _bin_begin, _bin_end, _tiles_y, blend_backward, exact_records,
                         preprocess_backward_views, preprocess_views, render_forward)

# reference defaults (config.py:76-92 OptimConfig; config.py:67-73 MaskConfig)
DEFAULT_LRS = {"positions": 1.6e-4, "log_scales": 5e-3, "rotations": 1e-3, "opacity_logits": 0.05,
               "sh_dc": 2.5e-3, "sh_rest": 2.5e-3 / 20.0, "mask_logits": 0.5, "sh_mask_logits": 0.05}


def _row_ranges(layout: dict, names, n: int, r0: int, r1: int) -> list:
    """Flat-buffer float ranges of cloud rows [r0, r1) of the fields `names` (r0 a multiple
    of 64; the last chunk runs to the field's 64-float padded end)."""
    from .cloud import _ROW
    out = []
    for f in sorted(names, key=lambda f: layout[f][0]):
        off, size = layout[f]
        w = math.prod(_ROW[f])
        end = off + (size + 63) // 64 * 64 if r1 >= n else off + r1 * w
        out.append((off + r0 * w, end))
    return out


class DensifyStats:
    """Densification statistics (TrainState.grad_accum / grad_count / area_max,
    training.py:116-135, updated per view at training.py:333-338): the sum of the
    per-view screen-space mean-gradient norms ||mean2d_screen * (W/2, H/2)||, the number
    of views each Gaussian was visible in, and its largest screen area.  Accumulated
    inside the multi-view preprocess kernels; float32 / int32 device tensors."""

    def __init__(self, n: int, device):
        self.grad_accum = torch.zeros(n, dtype=torch.float32, device=device)
        self.grad_count = torch.zeros(n, dtype=torch.int32, device=device)
        self.area_max = torch.zeros(n, dtype=torch.float32, device=device)

    def reset(self) -> None:  # TrainState.reset_stats (training.py:126-130)
        self.grad_accum.zero_()
        self.grad_count.zero_()
        self.area_max.zero_()

    def compact(self, keep: torch.Tensor) -> None:
        """TrainState.compact_stats (training.py:132-135) with the gather kernel."""
        from . import _lib
        k = keep.to(torch.int64).contiguous()
        st = _lib.stream_handle(self.grad_accum.device)
        for name in ("grad_accum", "grad_count", "area_max"):
            src = getattr(self, name)
            dst = torch.empty(k.numel(), dtype=src.dtype, device=src.device)
            _lib.call("tgs_gather_rows", _lib.ptr(src), _lib.ptr(dst), _lib.ptr(k), int(k.numel()), 1, st)
            setattr(self, name, dst)

    def mean_grad(self) -> torch.Tensor:
        """training.py:199: grad_accum / max(grad_count, 1), 0 where never visible."""
        return torch.where(self.grad_count > 0, self.grad_accum / self.grad_count.clamp_min(1).float(),
                           torch.zeros_like(self.grad_accum))

    def native(self):
        from . import _lib
        return _lib.TgsDensifyStats(self.grad_accum.data_ptr(), self.grad_count.data_ptr(),
                                    self.area_max.data_ptr())


class Trainer:
    def __init__(self, cloud: GaussianCloud, cameras, targets, settings: RenderSettings, lambda_ssim: float = 0.2,
                 lrs: dict | None = None, lambda_m: float = 0.05, lambda_sh: float = 0.05, process_group=None,
                 views=None, streams: int = 4, deterministic: bool = False, densify_stats: bool = False,
                 dp_mode: str = "zero", zero_chunks: int = 4, zero_sim: tuple | None = None,
                 native: bool | None = None, all_views: list | None = None, gshard_sim: tuple | None = None):
        self.cloud = cloud
        self.cameras = cameras
        self.targets = targets              # list of (H, W, 3) float32 device tensors (this rank's views)
        self.views = list(range(len(cameras))) if views is None else list(views)
        self.settings = settings
        self.lambda_ssim = lambda_ssim
        self.lambda_m, self.lambda_sh = lambda_m, lambda_sh
        self.pg = process_group
        # data parallelism (process_group given): "zero" = ZeRO-1 (reduce-scatter, Adam on this
        # rank's shard, all-gather; parallel.zero_plan), "allreduce" = bucketed all-reduce +
        # replicated Adam, "gaussians" = Gaussian-sharded (parallel.py: this rank's rows of
        # every view's preprocess, all-to-all exchanges of the preprocess outputs and the splat
        # partials, preprocess backward and Adam on this rank's rows; all_views = every
        # rank's view list, gathered when not given).  zero_sim=(rank, world) /
        # gshard_sim=(rank, world): one GPU runs rank `rank`'s share of a world-rank ZeRO-1 /
        # Gaussian-sharded step without communication (bench.py --rank-share projections).
        if dp_mode not in ("zero", "allreduce", "gaussians"):
            raise ValueError("dp_mode must be 'zero', 'allreduce' or 'gaussians'")
        self.dp_mode, self.zero_chunks, self.zero_sim = dp_mode, int(zero_chunks), zero_sim
        # native=True: the per-view loop (bin, count, place, blend, loss, backward) is issued
        # from C++ (tgs_train_views) when the views are pipelined over >= 2 streams and the
        # atomic backward is used; the Python loop remains for 1 stream (per-stage timing)
        # and the deterministic backward
        if native is None:  # TGS_TRAIN_NATIVE=0: the Python loop (A/B timing)
            native = os.environ.get("TGS_TRAIN_NATIVE", "1") != "0"
        self.native = native
        self._nat = {}  # per-geometry native buffers: (key) -> dict
        self.rank = 0
        if process_group is not None:
            import torch.distributed as dist
            self.rank = dist.get_rank(process_group)
        self._gs = None  # Gaussian-sharded state (dp_mode="gaussians")
        if dp_mode == "gaussians" and (process_group is not None or gshard_sim is not None):
            from .parallel import slot_order
            if process_group is not None:
                import torch.distributed as dist
                rank, world = self.rank, dist.get_world_size(process_group)
                if all_views is None:
                    all_views = [None] * world
                    dist.all_gather_object(all_views, self.views, group=process_group)
            else:
                rank, world = gshard_sim
                if all_views is None:
                    raise ValueError("gshard_sim needs all_views (every rank's view list)")
            if list(all_views[rank]) != self.views:
                raise ValueError("all_views[rank] must be this rank's views")
            self._gs = dict(rank=int(rank), world=int(world), order=slot_order([list(v) for v in all_views]), n=None)
        # the exact records inside the shard preprocess launch (one host call less before the
        # views' first launch) or as their own launch on the exact stream (TGS_GS_EXACT=side)
        self._gs_exact_inline = os.environ.get("TGS_GS_EXACT", "inline") == "inline"
        self.grads = CloudGrads(len(cloud), cloud.device)
        self.opt = Adam(cloud, lrs or DEFAULT_LRS)
        dev = cloud.device
        self.terms = torch.zeros((len(cameras), 2), dtype=torch.float64, device=dev)
        self.dimage = {}
        self._exc_bufs = {}  # (stream, H, W) -> blend exception lists (native path)
        self._pre_cache = {}  # preprocess_views' reused outputs (rasterizer.preprocess_views)
        self.dsplats = {}
        # >= 2 streams pipeline consecutive views (4 by default: measured 118 / 121 / 123 step/s
        # with 2 / 3 / 4 at c3); 1 stream serialises them (per-kernel timing)
        # stream priorities (CUDA range 0 .. -3, lower = scheduled first): the view streams
        # (each view's binning) highest, the blend streams (each view's blend / loss /
        # backward) next, the exact records' side kernel and the per-step kernels (main)
        # last — the latency-bound binning CTAs go ahead of the issue-bound blends, and
        # both ahead of the exact records only the blends need.  Same-box A/Bs
        # (profiles/r02_ab_view_stream_priority.log, r02_ab_blend_streams.log): high-priority
        # view streams 122.7-123.1 vs 120.0-121.0 step/s; separate blend streams e2e
        # 119.0-120.6 vs 117.7-118.9.  TGS_VIEW_PRIO / TGS_BLEND_PRIO / TGS_TRAIN_BLEND_STREAMS
        # override (A/B).
        vp = int(os.environ.get("TGS_VIEW_PRIO", "-2"))
        if streams > 1:  # TGS_TRAIN_STREAMS: A/B of the pipelined stream count
            streams = int(os.environ.get("TGS_TRAIN_STREAMS", streams))
        self.streams = [torch.cuda.Stream(device=cloud.device, priority=vp) for _ in range(max(1, streams))]
        self.copy_stream = torch.cuda.Stream(device=cloud.device)
        # the exact blend-decision records of the step's views are computed here while the
        # first views' depth sorts run (only the blends read them)
        self.exact_stream = torch.cuda.Stream(device=cloud.device,
                                              priority=int(os.environ.get("TGS_EXACT_PRIO", "0")))
        bp = int(os.environ.get("TGS_BLEND_PRIO", "-1"))
        self.blend_streams = ([torch.cuda.Stream(device=cloud.device, priority=bp) for _ in self.streams]
                              if os.environ.get("TGS_TRAIN_BLEND_STREAMS", "1") == "1" else [])
        # one GPU: the preprocess backward may run in row chunks, each chunk's Adam on
        # adam_stream beside the next chunk (TGS_BWD_CHUNKS).  Default 1: measured no gain at
        # c3 (113.3 step/s for 1, 2, 4 and 8 chunks) — the backward's 3 CTAs x 128 threads x
        # 160 registers fill the register file, so no Adam block co-resides
        self.bwd_chunks = int(os.environ.get("TGS_BWD_CHUNKS", "1"))
        self.adam_stream = torch.cuda.Stream(device=cloud.device)
        self.comm_stream = None  # data-parallel gradient reduction (created on first use)
        self.launches_per_step = 0
        self.deterministic = deterministic  # fixed-order gradient sums (bitwise reproducible steps)
        if self._gs is not None and (not self.native or deterministic or len(self.streams) < 2):
            raise ValueError("dp_mode='gaussians' runs the native multi-stream views path")
        # per-view densification statistics, accumulated inside the preprocess kernels
        self.stats = DensifyStats(len(cloud), dev) if densify_stats else None
        self.iteration = 0
        self.instances = []  # tile-list instances per view of the last step (host-known counts)
        # the multi-view preprocess backward zeroes each view's partial buffer after reading it
        # (False keeps the last step's partials readable, e.g. for inspection in tests)
        self.clear_partials = True
        # divergence guard (training.py:298-308): the fused Adam skips the whole update when a
        # loss term is not finite and raises this flag; the host learns it from a pinned copy
        # made at the end of the step, without a synchronisation of its own
        self._nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self._nf_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._terms_host = torch.zeros((len(cameras), 2), dtype=torch.float64, pin_memory=True)
        self._pending = None  # (iteration, event, Adam step counters before it, n, resolution)

    def prune(self, eps: float) -> int:
        """Mask-based pruning between steps (masking.py:70-81, training.py:340-346): keep
        the rows whose hard mask survives, compact the cloud and the Adam moments with
        tgs_gather_rows (optim.py:51-55) and resize the gradient buffers.  Returns the
        new Gaussian count."""
        from . import pruning
        self.sync_shards()
        new, keep = pruning.prune_by_mask(self.cloud, eps)
        self._apply_keep(new, keep)
        return len(self.cloud)

    def significance_prune(self, cameras, settings, rate: float, volume_power: float = 0.5):
        """A significance event (training.py:369-401): hits over `cameras`, scores
        (significance.py:45-78), drop the floor(rate N) lowest (significance.py:81-99)
        and compact the optimizer state and statistics.  Returns the report."""
        from . import significance as sig
        self.sync_shards()
        hits = sig.count_hits(self.cloud, cameras, settings)
        rep = sig.significance_scores(hits, self.cloud, mask_threshold=settings.mask_threshold,
                                      volume_power=volume_power)
        if int(math.floor(rate * len(self.cloud))) > 0:
            new, keep = sig.prune_by_significance(self.cloud, rep.scores, rate)
            self._apply_keep(new, keep)
        return rep

    def _apply_keep(self, new: GaussianCloud, keep: torch.Tensor) -> None:
        from . import pruning
        if new is self.cloud:
            return
        self._zero_sync_moments()
        pruning.compact_adam(self.opt, self.cloud, new, keep)
        self.cloud = new
        self.grads = CloudGrads(len(new), new.device)
        self.dsplats = {}
        if self.stats is not None:
            self.stats.compact(keep)

    def check_divergence(self, block: bool = True) -> None:
        """Raise DivergenceError (with the reference's snapshot keys, training.py:298-308)
        if a finished step saw a non-finite loss term.  That step updated nothing on the
        device (the guarded Adam launch) and its optimizer step counters are rolled back.
        block=False only looks at a step whose flag has already reached the host."""
        p = self._pending
        if p is None or (not block and not p[1].query()):
            return
        self._pending = None
        p[1].synchronize()
        if not int(self._nf_host[0]):
            return
        it, _, steps_before, n, res = p
        self.opt.steps = dict(steps_before)
        self.iteration = it
        terms = self._terms_host.numpy()
        bad = [v for v in self.views if not np.isfinite(terms[v]).all()] or list(self.views)
        v = bad[0]
        l1, ssim = float(terms[v, 0]), float(terms[v, 1])
        raise DivergenceError(f"non-finite loss at iteration {it}",
                              snapshot={"iteration": it, "n_gaussians": n, "l1": l1, "d_ssim": (1.0 - ssim) / 2.0,
                                        "resolution": res, "view": v})

    def step(self, host_targets=None) -> torch.Tensor:
        """One optimisation step over this rank's views; returns the device loss terms.

        host_targets: optional {view: pinned (H, W, 3) float32 CPU tensor}.  Each view's
        target is copied on a dedicated copy stream and its loss waits only for that
        copy, so the transfers of later views overlap the compute of earlier ones.

        A non-finite loss (training.py:298-308) leaves the parameters and Adam state
        untouched; DivergenceError is raised by the next step() (as soon as that step's
        first host read shows the flag) or by check_divergence()."""
        self.check_divergence(block=False)
        try:
            if self._gs is not None:
                return self._step_gshard(host_targets)
            return self._step(host_targets)
        except BaseException:
            self.dsplats = {}  # partial buffers may be left non-zero: start the next step afresh
            raise

    def _step(self, host_targets):
        g = self.grads
        vis, parts = [], []
        main = torch.cuda.current_stream(self.cloud.device)
        copied = {}
        n = len(self.cloud)
        prev_done = main.record_event() if host_targets is not None else None  # the previous step's reads
        if self.pg is not None:
            self.terms.zero_()  # other ranks' rows are summed in by the step's terms all-reduce
        # every view's preprocess in one pass over the parameters (main stream)
        vcams = [self.cameras[v] for v in self.views]
        from . import _lib
        self._c_cams = (_lib.TgsCamera * len(vcams))(*[_lib.make_camera(c) for c in vcams])  # once per step
        pres = preprocess_views(self.cloud, vcams, self.settings, stats=self.stats, exact=False, cache=self._pre_cache,
                                c_cams=self._c_cams)
        self.exact_stream.wait_stream(main)
        with torch.cuda.stream(self.exact_stream):
            exact_records(self.cloud, vcams, self.settings, pres, cache=self._pre_cache, c_cams=self._c_cams)
        exact_ready = torch.cuda.Event()
        exact_ready.record(self.exact_stream)
        if host_targets is not None:  # issued after the first heavy launch; each view's loss waits for its copy
            self.copy_stream.wait_event(prev_done)  # the previous step has finished reading the targets
            with torch.cuda.stream(self.copy_stream):
                for v in self.views:
                    self.targets[v].copy_(host_targets[v], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self.copy_stream)
                    copied[v] = ev
        ready = main.record_event()
        for s_ in self.streams + self.blend_streams:
            s_.wait_event(ready)  # parameters updated by the previous step's Adam; the preprocess
        ts = int(self.settings.tile_size)
        if self.native and not self.deterministic and n and len(self.streams) >= 2 and self.views:
            vis, parts = self._views_native(pres, exact_ready, copied)
            return self._after_views(main, g, vis, parts, copied, n)

        def begin(i):  # view i's depth sort + instance-count read-back, on view i's stream
            if not n or len(self.streams) < 2:
                return None
            cam_, (sp, _, tiles, keys, err, _) = self.cameras[self.views[i]], pres[i]
            with torch.cuda.stream(self.streams[i % len(self.streams)]):
                return _bin_begin(sp, tiles, n, int(cam_.width), int(cam_.height), ts, 0, _tiles_y(cam_, ts), err,
                                  keys)

        # consecutive views rotate over the streams: the latency-bound binning of a view
        # overlaps the blend / loss kernels of the others, and the next streams-1 views'
        # depth sorts are queued before a view's instance count is awaited (the host round
        # trip never leaves the GPU without work, also at the start of a step)
        ahead = max(len(self.streams) - 1, 1)
        pend = [begin(i) for i in range(min(ahead, len(self.views)))]
        for i, v in enumerate(self.views):
            st = self.streams[i % len(self.streams)]
            if i + ahead < len(self.views):
                pend.append(begin(i + ahead))
            p_i = pend.pop(0)
            with torch.cuda.stream(st):
                cam, target = self.cameras[v], self.targets[v]
                bins = _bin_end(p_i) if p_i is not None else None
                if i == 0:  # the previous step's flag is on the host once this view's count is
                    self.check_divergence(block=False)
                    self.instances = []
                if bins is not None:
                    self.instances.append(int(bins.indices.numel()))
                st.wait_event(exact_ready)  # the blends read the exact records
                out = render_forward(self.cloud, cam, self.settings, pre=pres[i], bins=bins)
            with torch.cuda.stream(st):
                d = self.dimage.get((i % len(self.streams), cam.height, cam.width))
                if d is None:
                    d = self.dimage[(i % len(self.streams), cam.height, cam.width)] = torch.empty_like(out.image)
                if v in copied:
                    st.wait_event(copied[v])
                with stage("loss"):
                    loss_mod.l1_ssim_async(out.image, target, self.lambda_ssim, d, self.terms[v])
                ds = self.dsplats.get(v)
                if ds is None or ds.shape[0] != len(self.cloud):
                    # zeroed once; afterwards the multi-view preprocess backward clears each
                    # buffer after reading it (no fill launch per view)
                    ds = self.dsplats[v] = torch.zeros((len(self.cloud), 9), dtype=torch.float32, device=d.device)
                elif not self.clear_partials:
                    ds.zero_()
                _, st_state = blend_backward(self.cloud, cam, self.settings, d, out, dsplats=ds,
                                             deterministic=self.deterministic)
                vis.append(st_state.visible_u8)
                parts.append(ds)
        return self._after_views(main, g, vis, parts, copied, n)

    def _step_gshard(self, host_targets):
        """Gaussian-sharded step (parallel.py, dp_mode="gaussians"): this rank's rows of
        every view's preprocess -> all-to-all of the preprocess outputs to the view owners ->
        this rank's views (tgs_train_views, the one-GPU schedule) -> all-to-all of the splat
        partials back to the shard owners -> preprocess backward and Adam over this rank's
        rows.  The parameters outside this rank's rows go stale between sync_shards() calls
        (pruning and significance events call it); nothing in the step reads them."""
        import torch.distributed as dist
        from . import _lib
        from .parallel import gshard_backward_exchange, gshard_forward_exchange, shard_rows
        G, g = self._gs, self.grads
        dev, n = self.cloud.device, len(self.cloud)
        main = torch.cuda.current_stream(dev)
        rank, world = G["rank"], G["world"]
        if G["n"] != n:  # (re)build the shard plan and the exchange buffers for this cloud size
            rows = shard_rows(n, world)
            a, b = rows[rank]
            k, V = len(self.views), len(G["order"])
            G.update(n=n, rows=rows, err=torch.zeros(1, dtype=torch.int32, device=dev),
                     full=[torch.empty((k, n, 12), device=dev), torch.empty((k, n), dtype=torch.uint8, device=dev),
                           torch.empty((k, n), dtype=torch.int32, device=dev),
                           torch.empty((k, n), dtype=torch.int64, device=dev), torch.empty((k, n, 8), device=dev)],
                     parts=torch.zeros((V, max(b - a, 1), 9), device=dev))
            if self.pg is None:  # simulation: every row as the exchange would deliver it for the
                # current parameters (bench.py restores them before every step)
                own = preprocess_views(self.cloud, [self.cameras[v] for v in self.views], self.settings)
                for kind, f in zip((0, 1, 2, 3, 5), G["full"]):
                    for j in range(k):
                        f[j].copy_(own[j][kind])
        rows = G["rows"]
        a, b = rows[rank]
        copied = {}
        prev_done = main.record_event() if host_targets is not None else None
        if self.pg is not None:
            self.terms.zero_()
        gcams = [self.cameras[v] for v in G["order"]]
        V = len(gcams)
        c_all = (_lib.TgsCamera * V)(*[_lib.make_camera(c) for c in gcams])  # once per step (~13 us)
        self._c_cams = (_lib.TgsCamera * len(self.views))(*[_lib.make_camera(self.cameras[v]) for v in self.views])
        # 1. this rank's rows of every view's preprocess (main stream) and their exchange to
        # the view owners.  The exact records are computed inside the preprocess launch and
        # travel with the other outputs (default), or (TGS_GS_EXACT=side) are their own launch
        # and exchange on the exact stream, which only the blends wait for.
        inline = self._gs_exact_inline
        pres = preprocess_views(self.cloud, gcams, self.settings, stats=self.stats, exact=inline, cache=self._pre_cache,
                                c_cams=c_all, rows=(a, b))
        bases = self._pre_cache[(V, max(b - a, 1), dev, a)][3]  # (splats, visible, tiles, keys, exact) [V][rows]
        full = G["full"]
        # (simulation, no process group: nothing moves — the full buffers already hold every
        # row, primed above, and the exchange's time is bench.py's communication model)
        err = pres[0][4]
        if self.pg is not None:
            with stage("gshard_exchange"):
                gshard_forward_exchange(list(bases) if inline else list(bases[:4]), full if inline else full[:4], rows,
                                        rank, self.pg)
                G["err"].copy_(err)
                dist.all_reduce(G["err"], op=dist.ReduceOp.MAX, group=self.pg)
                err = G["err"]
        ready = main.record_event()  # every view stream waits for the exchanged outputs
        if inline:
            exact_ready = ready
        else:
            self.exact_stream.wait_event(ready)
            with torch.cuda.stream(self.exact_stream):
                exact_records(self.cloud, gcams, self.settings, pres, cache=self._pre_cache, c_cams=c_all, rows=(a, b))
                if self.pg is not None:
                    with stage("gshard_exchange"):
                        gshard_forward_exchange([bases[4]], full[4:], rows, rank, self.pg)
            exact_ready = self.exact_stream.record_event()
        own = [(full[0][j], full[1][j], full[2][j], full[3][j], err, full[4][j]) for j in range(len(self.views))]
        if host_targets is not None:
            self.copy_stream.wait_event(prev_done)
            with torch.cuda.stream(self.copy_stream):
                for v in self.views:
                    self.targets[v].copy_(host_targets[v], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self.copy_stream)
                    copied[v] = ev
        for s_ in self.streams + self.blend_streams:
            s_.wait_event(ready)
        # 3. this rank's views: bin, blend, loss, blend backward (the one-GPU driver)
        _, parts_own = self._views_native(own, exact_ready, copied)
        for s_ in self.streams + self.blend_streams:
            main.wait_stream(s_)
        if not inline:
            main.wait_stream(self.exact_stream)
        if copied:
            main.wait_stream(self.copy_stream)
        steps_before = dict(self.opt.steps)
        # 4. every view's partials of this rank's rows; the own buffers start the next step
        # zeroed (on one GPU the preprocess backward clears them as it reads them)
        if self.pg is not None:
            with stage("gshard_exchange"):
                gshard_backward_exchange(parts_own, G["parts"], rows, rank, self.pg)
        for p in parts_own:
            p.zero_()
        # 5. preprocess backward and Adam over this rank's rows
        preprocess_backward_views(self.cloud, gcams, self.settings, [p[1] for p in pres],
                                  [G["parts"][i] for i in range(V)], g, accumulate=False, stats=self.stats,
                                  rows=(a, b), local=True, c_cams=c_all)
        upd = set(PARAM_FIELDS)
        if not (self.settings.compute_sh_rest_grads and self.settings.active_sh_degree > 0):
            upd.discard("sh_rest")
        if self.pg is not None:
            dist.all_reduce(self.terms, group=self.pg)
        with stage("adam"):
            self.opt.step(self.cloud, g, names=tuple(upd), lambda_m=self.lambda_m, lambda_sh=self.lambda_sh,
                          guard=(self.terms, self._nonfinite),
                          ranges=_row_ranges(g._layout_map, upd, n, a, b) if b > a else [])
        cam0 = self.cameras[self.views[0]] if self.views else None
        res = (int(cam0.height), int(cam0.width)) if cam0 is not None else (0, 0)
        return self._finish(main, steps_before, n, res)

    def sync_shards(self) -> None:
        """dp_mode="gaussians": every rank's rows of the parameters, the Adam moments and the
        densification statistics to every rank (before events that read the whole cloud:
        pruning, significance scoring, checkpoints).  No-op otherwise."""
        G = self._gs
        if G is None or self.pg is None:
            return
        import torch.distributed as dist
        from .parallel import shard_rows
        n = len(self.cloud)
        rows = shard_rows(n, G["world"])
        bufs = []
        for f in PARAM_FIELDS:
            off, size = self.cloud.field_range(f)
            w = size // max(n, 1)
            for t in (self.cloud.flat, self.opt.m, self.opt.v):
                bufs.append((t, off, w))
        for d, (a, b) in enumerate(rows):
            if b <= a:
                continue
            src = dist.get_global_rank(self.pg, d)
            for t, off, w in bufs:
                dist.broadcast(t[off + a * w: off + b * w], src=src, group=self.pg)
            if self.stats is not None:
                for t in (self.stats.grad_accum, self.stats.grad_count, self.stats.area_max):
                    dist.broadcast(t[a:b], src=src, group=self.pg)

    def _views_native(self, pres, exact_ready, copied):
        """tgs_train_views: the views' bin -> count -> place -> blend -> loss -> backward
        issued from C++ over self.streams (the Python loop's schedule).  Buffers persist per
        view geometry; a too-small instance capacity is grown and the batch retried with
        the partial buffers zeroed."""
        import ctypes
        from . import _lib
        from .errors import TGS_ERR_CAPACITY, raise_for_status
        from .rasterizer import EXACT_DECISIONS, EXCEPTION_LISTS, _blend_order, _scratch, _size_class, ctypes_size
        dev, n, ts = self.cloud.device, len(self.cloud), int(self.settings.tile_size)
        ns, V = len(self.streams), len(self.views)
        cams = [self.cameras[v] for v in self.views]
        geo = tuple((int(c.width), int(c.height)) for c in cams)
        key = (n, ts, geo)
        nb = self._nat.get(key)
        if nb is None:
            nb = self._nat[key] = {"cap": 0}
            self._nat = {key: nb}  # one geometry at a time (resolution steps free the old)
        for v in self.views:
            ds = self.dsplats.get(v)
            if ds is None or ds.shape[0] != n:
                self.dsplats[v] = torch.zeros((n, 9), dtype=torch.float32, device=dev)
            elif not self.clear_partials:
                ds.zero_()
        c_set = _lib.make_settings(self.settings)
        c_cams = self._c_cams  # this step's (the same views, built in _step)
        c_cloud = self.cloud.native()
        arr = lambda k: (ctypes.c_void_p * V)(*[p[k].data_ptr() for p in pres])  # noqa: E731
        pinned = nb.get("pinned")
        if pinned is None:
            pinned = nb["pinned"] = torch.empty(2 * ns, dtype=torch.int64, pin_memory=True)
        for attempt in range(4):
            cap = nb["cap"]
            if cap == 0:  # first step of this geometry: a generous first guess
                cap = nb["cap"] = _size_class(max(4096, 24 * n))
            if nb.get("bufs_cap") != cap:
                nb["bufs"] = []
                for w, h in geo:
                    tx, ty = (w + ts - 1) // ts, (h + ts - 1) // ts
                    nb["bufs"].append(dict(
                        image=torch.empty((h, w, 3), device=dev), T=torch.empty((h, w), device=dev),
                        ws=torch.empty((h, w), device=dev), nc=torch.empty((h, w), dtype=torch.int32, device=dev),
                        lp=torch.empty((h, w), dtype=torch.int32, device=dev),
                        off=torch.empty(tx * ty + 1, dtype=torch.int32, device=dev),
                        ids=torch.empty(cap, dtype=torch.int32, device=dev),
                        order=_blend_order(None, tx * ty, tx, ty, ts, dev, None)))
                nb["bufs_cap"] = cap
                nb["wsb"] = max(ctypes_size("tgs_render_views_workspace", n, cap, w, h, ts) for w, h in geo)
            # the driver's argument structs are rebuilt only when a buffer behind them can have
            # changed (capacity, partial / target buffers, the preprocess outputs); otherwise
            # only the per-step events are patched in (~0.1 ms of host work per step saved,
            # which sits before the step's first binning launch)
            sig = (cap, tuple(self.dsplats[v].data_ptr() for v in self.views),
                   tuple(self.targets[v].data_ptr() for v in self.views),
                   tuple(pres[0][k].data_ptr() for k in (0, 1, 2, 3, 5)), EXACT_DECISIONS)
            ct = nb.get("ct")
            if ct is not None and ct["sig"] == sig:
                targets, train = ct["targets"], ct["train"]
                for i, v in enumerate(self.views):
                    train[i].target_ready = copied[v].cuda_event if v in copied else None
                rc = self._train_views_call(ct, c_cloud, c_cams, c_set, V, exact_ready, pres, targets, train, nb,
                                            pinned, ns)
                counts = [int(targets[i].num_instances) for i in range(V)]
                if rc == TGS_ERR_CAPACITY:
                    for s_ in self.streams + self.blend_streams:
                        s_.synchronize()
                    for v in self.views:
                        self.dsplats[v].zero_()
                    nb["cap"] = _size_class(int(max(counts) * 1.25) + 1024)
                    continue
                raise_for_status(rc, "tgs_train_views")
                break
            wss = [_scratch("train_views", nb["wsb"], dev, s_.cuda_stream, owner=s_) for s_ in self.streams]
            loss_ws, train = [], (_lib.TgsViewTrain * V)()
            targets = (_lib.TgsViewTarget * V)()
            for i, v in enumerate(self.views):
                b = nb["bufs"][i]
                k = i % ns
                h, w = geo[i][1], geo[i][0]
                d = self.dimage.get((k, h, w))
                if d is None:
                    with torch.cuda.stream(self.streams[k]):
                        d = self.dimage[(k, h, w)] = torch.empty((h, w, 3), device=dev)
                lw = _scratch("loss", loss_mod._loss_bytes(w, h), dev, self.streams[k].cuda_stream, owner=self.streams[k])
                loss_ws.append(lw)
                xb = self._exc_bufs.get((k, h, w))  # the blend exception lists, shared per stream
                if xb is None and EXCEPTION_LISTS and ts == 16:
                    ntl = ((w + ts - 1) // ts) * ((h + ts - 1) // ts)
                    with torch.cuda.stream(self.streams[k]):
                        xb = self._exc_bufs[(k, h, w)] = (torch.empty((h, w), dtype=torch.int32, device=dev),
                                                          torch.empty(1 + ntl, dtype=torch.int32, device=dev))
                targets[i] = _lib.TgsViewTarget(b["off"].data_ptr(), b["ids"].data_ptr(), cap, _lib.ptr(b["order"]),
                                                b["image"].data_ptr(), b["T"].data_ptr(), b["ws"].data_ptr(),
                                                b["nc"].data_ptr(), b["lp"].data_ptr(), None, -1, 0, 0)
                train[i] = _lib.TgsViewTrain(self.targets[v].data_ptr(), d.data_ptr(), self.terms[v].data_ptr(),
                                             self.dsplats[v].data_ptr(), lw.data_ptr(),
                                             copied[v].cuda_event if v in copied else None,
                                             _lib.ptr(xb[0]) if xb else None, _lib.ptr(xb[1]) if xb else None)
            ct = nb["ct"] = dict(
                sig=sig, targets=targets, train=train, loss_ws=loss_ws,
                ptrs=[arr(0), arr(1), arr(2), arr(3), arr(5) if EXACT_DECISIONS else None],
                wss=(ctypes.c_void_p * ns)(*[t.data_ptr() for t in wss]),
                streams=(ctypes.c_void_p * ns)(*[s_.cuda_stream for s_ in self.streams]),
                blend_streams=(ctypes.c_void_p * ns)(*[s_.cuda_stream for s_ in self.blend_streams])
                if self.blend_streams else None)
            rc = self._train_views_call(ct, c_cloud, c_cams, c_set, V, exact_ready, pres, targets, train, nb, pinned,
                                        ns)
            counts = [int(targets[i].num_instances) for i in range(V)]
            if rc == TGS_ERR_CAPACITY:
                for s_ in self.streams + self.blend_streams:
                    s_.synchronize()
                for v in self.views:  # views already backwarded accumulated partials
                    self.dsplats[v].zero_()
                nb["cap"] = _size_class(int(max(counts) * 1.25) + 1024)
                continue
            raise_for_status(rc, "tgs_train_views")
            if nb["cap"] < max(counts):  # (not reached: the driver reports capacity first)
                nb["cap"] = _size_class(int(max(counts) * 1.25) + 1024)
            break
        else:
            raise RuntimeError("tgs_train_views: instance capacity did not converge")
        self.check_divergence(block=False)  # the previous step's flag is on the host by now
        self.instances = counts
        return [p[1] for p in pres], [self.dsplats[v] for v in self.views]

    def _train_views_call(self, ct, c_cloud, c_cams, c_set, V, exact_ready, pres, targets, train, nb, pinned, ns):
        import ctypes
        from . import _lib
        p = ct["ptrs"]
        with stage("train_views"):
            return int(_lib.load().tgs_train_views(
                ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), V, p[0], p[1], p[2], p[3], p[4],
                exact_ready.cuda_event, pres[0][4].data_ptr(), targets, train, float(self.lambda_ssim), ct["wss"],
                nb["wsb"], pinned.data_ptr(), ct["streams"], ct["blend_streams"], ns))

    def _after_views(self, main, g, vis, parts, copied, n):
        for s_ in self.streams + self.blend_streams:
            main.wait_stream(s_)
        main.wait_stream(self.exact_stream)
        if copied:
            main.wait_stream(self.copy_stream)
        steps_before = dict(self.opt.steps)
        cam0 = self.cameras[self.views[0]] if self.views else None
        res = (int(cam0.height), int(cam0.width)) if cam0 is not None else (0, 0)
        guard = (self.terms, self._nonfinite)
        # training.py:321-329: sh_rest is optimised only on steps with higher-band gradients
        # and a non-zero active degree; every other group every step
        upd = set(PARAM_FIELDS)
        if not (self.settings.compute_sh_rest_grads and self.settings.active_sh_degree > 0):
            upd.discard("sh_rest")
        vcams = [self.cameras[v] for v in self.views]
        if self.pg is None and self.zero_sim is None and self.bwd_chunks > 1 and n >= 64 * self.bwd_chunks:
            # one GPU: the multi-view preprocess backward in row chunks on the main stream, and
            # each chunk's Adam (all groups, the chunk's rows) on a side stream as soon as
            # the chunk is done — the HBM-bound Adam overlaps the latency-bound backward
            self.adam_stream.wait_stream(main)
            per = -(-n // self.bwd_chunks)
            per = -(-per // 64) * 64
            for k, r0 in enumerate(range(0, n, per)):
                r1 = min(n, r0 + per)
                preprocess_backward_views(self.cloud, vcams, self.settings, vis, parts, g, accumulate=False,
                                          stats=self.stats, clear=self.clear_partials, rows=(r0, r1))
                done = torch.cuda.Event()
                done.record(main)
                self.adam_stream.wait_event(done)
                with stage("adam"), torch.cuda.stream(self.adam_stream):
                    self.opt.step(self.cloud, g, names=tuple(upd), lambda_m=self.lambda_m, lambda_sh=self.lambda_sh,
                                  guard=guard, ranges=_row_ranges(g._layout_map, upd, n, r0, r1), count=k == 0)
            main.wait_stream(self.adam_stream)
            return self._finish(main, steps_before, n, res)
        # one pass over the parameters for all views (linear chains summed first)
        preprocess_backward_views(self.cloud, vcams, self.settings, vis, parts, g,
                                  accumulate=False, stats=self.stats, clear=self.clear_partials, c_cams=self._c_cams)
        if self.zero_sim is not None or (self.pg is not None and self.dp_mode == "zero"):
            return self._zero_update(main, g, upd, guard, steps_before, n, res)
        if self.pg is None:
            with stage("adam"):
                # the mask penalties of total_loss (masking.py:60-67) enter the gradient inside
                # the fused Adam launch
                self.opt.step(self.cloud, g, names=tuple(upd), lambda_m=self.lambda_m, lambda_sh=self.lambda_sh,
                              guard=guard)
            return self._finish(main, steps_before, n, res)
        # data parallel: the gradient buckets are all-reduced on a communication stream in
        # order, and each bucket's Adam update (identical on every rank, mask penalties
        # included) starts as soon as its reduction is done, overlapping the next ones
        import torch.distributed as dist
        from .parallel import grad_buckets
        if self.comm_stream is None:
            self.comm_stream = torch.cuda.Stream(device=self.cloud.device)
        buckets = grad_buckets(g._layout_map, rest_grads=bool(self.settings.compute_sh_rest_grads))
        self.comm_stream.wait_stream(main)
        done = []
        with stage("allreduce"), torch.cuda.stream(self.comm_stream):
            # every view's loss terms on every rank (each rank wrote only its own rows, the
            # others are zero): the divergence guard then decides identically everywhere
            dist.all_reduce(self.terms, group=self.pg)
            for _, a0, a1 in buckets:
                dist.all_reduce(g.flat[a0:a1], group=self.pg)
                ev = torch.cuda.Event()
                ev.record(self.comm_stream)
                done.append(ev)
        with stage("adam"):
            for (fields, _, _), ev in zip(buckets, done):
                main.wait_event(ev)
                names = tuple(f for f in fields if f in upd)
                if names:
                    self.opt.step(self.cloud, g, names=names, lambda_m=self.lambda_m, lambda_sh=self.lambda_sh,
                                  guard=guard)
        return self._finish(main, steps_before, n, res)

    def _zero_world(self):
        if self.pg is not None:
            import torch.distributed as dist
            return self.rank, dist.get_world_size(self.pg)
        return self.zero_sim

    def _zero_update(self, main, g, upd, guard, steps_before, n, res) -> torch.Tensor:
        """ZeRO-1 (parallel.zero_plan): per chunk, an in-place reduce-scatter of the gradient
        on the communication stream, the fused Adam (mask penalties and divergence guard
        included) on this rank's shard, and an in-place all-gather of the parameters — chunk
        k's all-gather overlaps chunk k+1's Adam.  Without a process group (zero_sim) the
        same Adam launches run with no communication."""
        from .parallel import all_gather_inplace, reduce_scatter_inplace, zero_plan
        rank, world = self._zero_world()
        plan = zero_plan(g._layout_map, world, rest_grads=bool(self.settings.compute_sh_rest_grads),
                         chunks=self.zero_chunks)
        if self.comm_stream is None:
            self.comm_stream = torch.cuda.Stream(device=self.cloud.device)
        comm = self.comm_stream
        comm.wait_stream(main)
        reduced = []
        with stage("reduce_scatter"), torch.cuda.stream(comm):
            if self.pg is not None:
                import torch.distributed as dist
                # every view's loss terms on every rank (each rank wrote only its own rows,
                # the others are zero): the divergence guard then decides identically everywhere
                dist.all_reduce(self.terms, group=self.pg)
            for ch in plan:
                if self.pg is not None:
                    reduce_scatter_inplace(g.flat, ch, rank, world, self.pg)
                ev = torch.cuda.Event()
                ev.record(comm)
                reduced.append(ev)
        names = tuple(upd)
        for k, (ch, ev) in enumerate(zip(plan, reduced)):
            main.wait_event(ev)
            with stage("adam"):
                self.opt.step(self.cloud, g, names=names, lambda_m=self.lambda_m, lambda_sh=self.lambda_sh, guard=guard,
                              ranges=[ch.rank_range(rank)], count=k == 0)
            if self.pg is not None:
                done = torch.cuda.Event()
                done.record(main)
                comm.wait_event(done)
                with stage("all_gather"), torch.cuda.stream(comm):
                    all_gather_inplace(self.cloud.flat, ch, rank, world, self.pg)
        main.wait_stream(comm)
        return self._finish(main, steps_before, n, res)

    def _zero_sync_moments(self) -> None:
        """ZeRO-1 keeps each rank's Adam moments current on its own shard only; before the
        rows are compacted (pruning) every rank gathers the full moments."""
        if self.pg is None or self.dp_mode != "zero":
            return
        from .parallel import all_gather_inplace, zero_plan
        rank, world = self._zero_world()
        for ch in zero_plan(self.grads._layout_map, world, rest_grads=True, chunks=self.zero_chunks):
            all_gather_inplace(self.opt.m, ch, rank, world, self.pg)
            all_gather_inplace(self.opt.v, ch, rank, world, self.pg)

    def _finish(self, main, steps_before, n, res) -> torch.Tensor:
        """Queue the pinned copy of the divergence flag and the loss terms; the next step
        (or check_divergence) reads it."""
        self._nf_host.copy_(self._nonfinite, non_blocking=True)
        self._terms_host.copy_(self.terms, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(main)
        self._pending = (self.iteration, ev, steps_before, n, res)
        self.iteration += 1
        return self.terms
