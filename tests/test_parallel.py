"""Multi-process host logic of parallel.py under gloo (world_size 2, CPU only).

The CUDA kernels cannot run here, so the per-rank compute is the oracle; what
is under test is the partitioning: the balanced tile-row split, the row-band
all-gather, the view sharding and the gradient all-reduce.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_14534_b200 import parallel


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_split_is_balanced_and_covering():
    rng = np.random.default_rng(0)
    for rows in (1, 2, 7, 68, 135):
        counts = rng.integers(0, 5000, rows)
        for world in (1, 2, 3, 4, 8):
            bands = parallel.row_split(counts, world)
            assert bands[0][0] == 0 and bands[-1][1] == rows
            assert all(b[1] == c[0] for b, c in zip(bands, bands[1:]))
            assert all(e > b for b, e in bands)
            assert len(bands) == min(world, rows)
            loads = [counts[b:e].sum() for b, e in bands]
            assert max(loads) <= counts.sum() / len(bands) + counts.max() + 1
    assert parallel.shard_views(8, 1, 3) == [1, 4, 7]


def _scene():
    from paper_2501_14534_b200 import scenes
    sc = scenes.small_scene(seed=9, n=600, width=80, height=64, dist=3.0)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * d, 80, 64) for d in
                              (np.array([1.0, 0.2, 0.3]), np.array([-0.4, 1.0, 0.2]), np.array([0.1, -0.3, 1.0]))]
    return sc.fields, cams


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        fields, cams = _scene()
        st = oracle.default_settings(near=0.2)
        # --- render: tile-row sharding, assembled with gather_rows
        ref = oracle.render_forward(fields, cams[0], st, "f32")
        ty, tx = ref["tiles_y"], ref["tiles_x"]
        row_counts = np.diff(ref["offsets"]).reshape(ty, tx).sum(axis=1)
        bands = parallel.row_split(row_counts, world)
        b, e = bands[rank]
        mine = torch.zeros((64, 80, 3))
        mine[b * 16:min(e * 16, 64)] = torch.from_numpy(ref["image"][b * 16:min(e * 16, 64)])
        full = parallel.gather_rows(mine, bands, rank, 16, 64)
        ok_render = torch.equal(full, torch.from_numpy(ref["image"]))
        # --- training: view sharding + flat-buffer all-reduce == sum over all views
        rng = np.random.default_rng(1)
        dimgs = [rng.standard_normal((64, 80, 3)) for _ in cams]

        def view_grad(v):
            f = oracle.render_forward(fields, cams[v], st, "f64")
            g = oracle.render_backward(fields, cams[v], st, dimgs[v], f, "f64")
            return np.concatenate([g[k].ravel() for k in oracle.FIELDS])

        local = sum(view_grad(v) for v in parallel.shard_views(len(cams), rank, world))
        flat = torch.from_numpy(np.asarray(local, dtype=np.float64))
        parallel.allreduce_grads(flat)
        want = sum(view_grad(v) for v in range(len(cams)))
        ok_grads = np.allclose(flat.numpy(), want, rtol=1e-12, atol=1e-12)
        q.put((rank, bool(ok_render), bool(ok_grads)))
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_gloo_world2_sharded_render_and_dp_grads():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res


def test_grad_buckets_cover_the_parameter_groups():
    from paper_2501_14534_b200.cloud import PARAM_FIELDS, _layout
    fields = PARAM_FIELDS + ("mean2d_screen",)
    lay, _ = _layout(fields, 1000)
    for rest in (True, False):
        b = parallel.grad_buckets(lay, rest_grads=rest)
        groups = [f for fs, _, _ in b for f in fs]
        assert sorted(groups) == sorted(f for f in PARAM_FIELDS if rest or f != "sh_rest")
        for fs, a0, a1 in b:  # each range covers what it must reduce, nothing of mean2d_screen
            assert a1 <= lay["mean2d_screen"][0]
            for f in fs:
                o, n = lay[f]
                if f == "sh_mask_logits" and not rest:
                    assert o >= a1  # zero on such steps: not reduced
                else:
                    assert a0 <= o and o + n <= a1
        if rest:
            assert b[0][0] == ("sh_rest",)  # the big bucket first: its Adam overlaps the rest


def _bucket_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_14534_b200.cloud import PARAM_FIELDS, _layout
        lay, total = _layout(PARAM_FIELDS + ("mean2d_screen",), 500)
        ok = []
        for rest in (True, False):
            g = torch.from_numpy(np.random.default_rng(rank).standard_normal(total))
            if not rest:  # zero on every rank without higher-band gradients
                for f in ("sh_rest", "sh_mask_logits"):
                    o, n = lay[f]
                    g[o:o + n] = 0
            full = g.clone()
            dist.all_reduce(full)
            for _, a0, a1 in parallel.grad_buckets(lay, rest_grads=rest):
                dist.all_reduce(g[a0:a1])
            for f in PARAM_FIELDS:  # every field (not the alignment padding between them)
                o, n = lay[f]
                ok.append(torch.allclose(g[o:o + n], full[o:o + n], rtol=1e-12, atol=1e-12))
        q.put((rank, all(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bucketed_allreduce_equals_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1] and all(r[1] for r in res), res


def test_zero_plan_tiles_the_parameters():
    """ZeRO-1 chunks: shard sizes are multiples of 64 floats, the padded extents of a
    segment's chunks tile it without overlap, every parameter field is covered by exactly
    one rank's range, and padded tails stay inside sh_rest (steps without higher-band
    gradients) or the ZERO_PAD headroom."""
    from paper_2501_14534_b200.cloud import PARAM_FIELDS, ZERO_PAD, _layout, params_end
    for n in (1, 37, 1000, 123457):
        lay, total = _layout(PARAM_FIELDS + ("mean2d_screen",), n)
        end = params_end(lay)
        for world in (1, 2, 3, 8):
            for rest in (True, False):
                plan = parallel.zero_plan(lay, world, rest_grads=rest, chunks=4)
                owned = np.zeros(end, dtype=np.int32)
                for i, ch in enumerate(plan):
                    assert ch.shard % 64 == 0 and ch.begin % 64 == 0
                    pe = ch.padded_end(world)
                    nxt = plan[i + 1].begin if i + 1 < len(plan) else None
                    if nxt is not None and nxt < pe:
                        raise AssertionError("padded chunk overlaps the next one")
                    if pe > ch.end:  # a padded tail: sh_rest on no-rest steps, else the headroom
                        if not rest and ch.end == lay["sh_rest"][0]:
                            assert pe <= lay["mask_logits"][0]
                        else:
                            assert ch.end == end and pe <= end + ZERO_PAD and pe <= lay["mean2d_screen"][0]
                    for r in range(world):
                        a, b = ch.rank_range(r)
                        owned[a:b] += 1
                single = len({c.end for c in plan if c.end == lay["sh_rest"][0]}) == 0
                for f in PARAM_FIELDS:
                    if f == "sh_rest" and not rest and not single:
                        continue
                    o, m = lay[f]
                    assert (owned[o:o + m] == 1).all(), (n, world, rest, f)


def _zero_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_14534_b200.cloud import PARAM_FIELDS, _layout
        lay, total = _layout(PARAM_FIELDS + ("mean2d_screen",), 777)
        ok = []
        for rest in (True, False):
            rng = np.random.default_rng(100 + rank)
            g = torch.from_numpy(rng.standard_normal(total))
            p0 = torch.from_numpy(np.random.default_rng(7).standard_normal(total))  # replicated
            if not rest:
                o, m = lay["sh_rest"]
                g[o:o + m] = 0  # zero on every rank without higher-band gradients
            # reference: all-reduce + the update on every field
            gs = g.clone()
            dist.all_reduce(gs)
            ref = p0.clone()
            for f in PARAM_FIELDS:
                if f == "sh_rest" and not rest:
                    continue
                o, m = lay[f]
                ref[o:o + m] -= 0.1 * gs[o:o + m]
            # ZeRO-1: in-place reduce-scatter, update of this rank's shard, in-place all-gather
            p = p0.clone()
            plan = parallel.zero_plan(lay, world, rest_grads=rest, chunks=3)
            for ch in plan:
                parallel.reduce_scatter_inplace(g, ch, rank, world)
            for ch in plan:
                a, b = ch.rank_range(rank)
                for f in PARAM_FIELDS:  # the kernel updates field floats only, never padding
                    if f == "sh_rest" and not rest:
                        continue
                    o, m = lay[f]
                    lo, hi = max(a, o), min(b, o + m)
                    if hi > lo:
                        p[lo:hi] -= 0.1 * g[lo:hi]
                parallel.all_gather_inplace(p, ch, rank, world)
            for f in PARAM_FIELDS:
                o, m = lay[f]
                ok.append(torch.allclose(p[o:o + m], ref[o:o + m], rtol=1e-12, atol=1e-12))
        q.put((rank, all(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_zero1_update_equals_allreduce_update(world):
    """ZeRO-1 over gloo (world 2 and 3): reduce-scatter + shard update + all-gather gives
    every rank the parameters of all-reduce + full update."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_zero_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world)) and all(r[1] for r in res), res


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, w, ts, nf = 70, 9, 16, 3
        frames = [torch.from_numpy(np.random.default_rng(f).standard_normal((h, w, 3))) for f in range(nf)]
        rows = (h + ts - 1) // ts
        bands = parallel.row_split(np.random.default_rng(5).uniform(1, 9, rows), world)
        maxr = max(min(e * ts, h) - b * ts for b, e in bands)
        b, e = bands[rank]
        buf = torch.zeros((nf, maxr, w, 3), dtype=torch.float64)
        for f in range(nf):
            buf[f, : min(e * ts, h) - b * ts] = frames[f][b * ts: min(e * ts, h)]
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, parts, dst=0)
        ok = True
        if rank == 0:
            got = parallel.assemble_bands(parts, bands, ts, h)
            ok = all(torch.equal(a, b_) for a, b_ in zip(got, frames))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_band_gather_to_rank0_assembles_frames():
    """The sharded render's batch gather: every rank's band rows of every frame to rank 0
    in one gather, assembled into the full frames (parallel.assemble_bands)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1, 2] and all(r[1] for r in res), res


def test_shard_rows_and_slot_order():
    for n in (0, 1, 63, 64, 777, 1000000):
        for world in (1, 2, 3, 8):
            rows = parallel.shard_rows(n, world)
            assert len(rows) == world and rows[0][0] == 0 and rows[-1][1] == n
            assert all(b[1] == c[0] for b, c in zip(rows, rows[1:]))
            assert all((a % 64 == 0 or a == n) and b >= a for a, b in rows)
    assert parallel.slot_order([[0, 2], [1, 3]]) == [0, 1, 2, 3]
    assert parallel.slot_order([[0, 3, 6], [1, 4, 7], [2, 5, 8]]) == list(range(9))
    with pytest.raises(ValueError):
        parallel.slot_order([[0, 1], [2]])


def _truth_fwd(view, n):
    """Per-Gaussian preprocess outputs of `view` with the exchange's dtypes and widths."""
    i = torch.arange(n, dtype=torch.float64)
    return [(view * 1000 + i[:, None] + torch.arange(12) / 100).float(),
            ((view + torch.arange(n)) % 2).to(torch.uint8),
            (view * 7 + torch.arange(n)).to(torch.int32),
            (view * (1 << 40) + torch.arange(n)).to(torch.int64),
            (-view * 1000 - i[:, None] - torch.arange(8) / 100).float()]


def _gshard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, k = 777, 2
        views_of = [[d + world * j for j in range(k)] for d in range(world)]
        order = parallel.slot_order(views_of)
        rows = parallel.shard_rows(n, world)
        a, b = rows[rank]
        truth = {v: _truth_fwd(v, n) for v in order}
        # this rank's shard-local preprocess outputs of every view, slot order
        sub = [torch.stack([truth[v][kind][a:b] for v in order]) for kind in range(5)]
        full = [torch.zeros((k, n) + t.shape[1:], dtype=t.dtype) for t in truth[order[0]]]
        parallel.gshard_forward_exchange(sub, full, rows, rank, dist.group.WORLD)
        ok = all(torch.equal(full[kind][j], truth[views_of[rank][j]][kind]) for kind in range(5) for j in range(k))
        # splat partials of the own views back to the shard owners
        parts = {v: (v * 100 + torch.arange(n, dtype=torch.float64)[:, None] + torch.arange(9) * 1e-3).float()
                 for v in order}
        own = [parts[v].clone() for v in views_of[rank]]
        recv = torch.zeros((len(order), max(b - a, 1), 9))
        parallel.gshard_backward_exchange(own, recv, rows, rank, dist.group.WORLD)
        ok = ok and all(torch.equal(recv[i, :b - a], parts[v][a:b]) for i, v in enumerate(order))
        # no group (one rank's share simulated on one device): only this rank's rows move
        full2 = [torch.zeros_like(f) for f in full]
        parallel.gshard_forward_exchange(sub, full2, rows, rank, None)
        ok = ok and all(torch.equal(full2[kind][j, a:b], truth[views_of[rank][j]][kind][a:b]) and
                        not full2[kind][j, :a].any() and not full2[kind][j, b:].any()
                        for kind in range(5) for j in range(k))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_gaussian_shard_exchanges(world):
    """dp_mode="gaussians" exchanges over gloo (world 2 and 3, 777 rows: an uneven last
    shard): every view owner receives its views' full per-Gaussian preprocess outputs in
    cloud row order (all five dtypes), and every shard owner receives its rows of every
    view's splat partials."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gshard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world)) and all(r[1] for r in res), res
