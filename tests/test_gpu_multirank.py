"""Multi-rank runs of the data-parallel training step on ONE GPU: W processes, one rank
each, over gloo (its collectives move CUDA tensors through the host, so no rank's
kernels wait on another's on the device — NCCL refuses two ranks per GPU).  What is
under test is the whole data-parallel step with real exchanges between ranks
(parallel.py, train.Trainer): for dp_mode="gaussians" every rank's shard of the
gradient, the loss terms, the parameters after Adam steps and the densification
statistics equal the one-process step over all views; for ZeRO-1 the loss terms and
every rank's (all-gathered) parameters do.  The tile-row sharded renderer assembles
frames bitwise equal to the one-GPU render."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

VIEWS = 6  # divisible by the world sizes under test


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(rest=True):
    from paper_2501_14534_b200 import RenderSettings, scenes
    sc = scenes.small_scene(seed=47, n=20_000, width=160, height=112, dist=3.0)
    rng = np.random.default_rng(47)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * scenes._unit(rng), 144, 96, name=f"m{k}")
                              for k in range(VIEWS - 1)]
    st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1, compute_sh_rest_grads=rest,
                        active_sh_degree=3 if rest else 2)
    tg = [torch.rand((c.height, c.width, 3), generator=torch.Generator().manual_seed(k)) for k, c in enumerate(cams)]
    return sc.fields, cams, st, tg


def _run(tr, lrs):
    """lr 0 step (the gradient and terms of the initial parameters), then two Adam steps."""
    for f in lrs:
        tr.opt.set_lr(f, 0.0)
    tr.step()
    torch.cuda.synchronize()
    out = dict(terms=tr.terms.cpu().numpy().copy(), grads=tr.grads.flat.cpu().numpy().copy())
    for f, lr in lrs.items():
        tr.opt.set_lr(f, lr)
    tr.step()
    tr.step()
    tr.check_divergence()
    torch.cuda.synchronize()
    out.update(params=tr.cloud.flat.cpu().numpy().copy(), count=tr.stats.grad_count.cpu().numpy().copy())
    return out


def _worker(rank, world, port, q, dp="gaussians", rest=True):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_14534_b200 import GaussianCloud
        from paper_2501_14534_b200.parallel import shard_rows
        from paper_2501_14534_b200.train import Trainer
        fields, cams, st, tg = _setup(rest)
        views = list(range(rank, VIEWS, world))
        targets = [t.cuda() if v in views else None for v, t in enumerate(tg)]
        cloud = GaussianCloud.from_fields(fields)
        tr = Trainer(cloud, cams, targets, st, process_group=dist.group.WORLD, views=views, dp_mode=dp,
                     densify_stats=True)
        out = _run(tr, dict(tr.opt.lrs))
        out["rows"] = shard_rows(len(cloud), world)[rank]
        tr.sync_shards()  # every rank's rows to every rank
        torch.cuda.synchronize()
        out["synced"] = tr.cloud.flat.cpu().numpy().copy()
        q.put((rank, out))
    except BaseException as e:  # noqa: BLE001 — report to the parent instead of hanging it
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _atol(f):
    """Parameters after Adam: three steps of lr x m / sqrt(v) amplify float32 summation-order
    noise in near-zero gradients (Adam's first step is lr x sign(g)); 1e-3 of the field's
    learning rate, at least 1e-4."""
    from paper_2501_14534_b200.train import DEFAULT_LRS
    return max(1e-4, 1e-3 * DEFAULT_LRS[f])


def _field_rows(cloud, a, b):
    """Flat-buffer index ranges of cloud rows [a, b) of every parameter field."""
    from paper_2501_14534_b200.cloud import PARAM_FIELDS
    n = len(cloud)
    out = []
    for f in PARAM_FIELDS:
        off, size = cloud.field_range(f)
        w = size // n
        out.append((f, off + a * w, off + b * w))
    return out


@pytest.mark.parametrize("world,rest", [(2, True), (3, True), (2, False)])
def test_gaussian_sharded_step_multirank_equals_one_process(world, rest):
    """(rest=False: an SH-cadence step at active degree 2 — sh_rest neither differentiated
    nor updated)"""
    import torch.multiprocessing as mp

    from paper_2501_14534_b200 import GaussianCloud
    from paper_2501_14534_b200.train import Trainer
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, "gaussians", rest)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    bad = {r: v for r, v in res.items() if isinstance(v, str)}
    assert not bad, bad
    # the one-process step over all views
    fields, cams, st, tg = _setup(rest)
    cloud = GaussianCloud.from_fields(fields)
    tr = Trainer(cloud, cams, [t.cuda() for t in tg], st, densify_stats=True)
    ref = _run(tr, dict(tr.opt.lrs))
    rows = [res[r]["rows"] for r in range(world)]
    assert rows[0][0] == 0 and rows[-1][1] == len(cloud) and all(rows[r][1] == rows[r + 1][0] for r in range(world - 1))
    scale = np.abs(ref["grads"]).max()
    for r in range(world):
        o = res[r]
        np.testing.assert_array_equal(o["terms"], ref["terms"])  # every view's terms on every rank
        a, b = o["rows"]
        np.testing.assert_array_equal(o["count"][a:b], ref["count"][a:b])
        for f, lo, hi in _field_rows(cloud, a, b):
            np.testing.assert_allclose(o["grads"][lo:hi], ref["grads"][lo:hi], rtol=1e-3, atol=1e-5 * scale,
                                       err_msg=f"rank {r} gradient {f}")
            np.testing.assert_allclose(o["params"][lo:hi], ref["params"][lo:hi], rtol=1e-4, atol=_atol(f),
                                       err_msg=f"rank {r} parameters {f}")
        # after sync_shards every rank holds every rank's rows
        for r2 in range(world):
            a2, b2 = res[r2]["rows"]
            for f, lo, hi in _field_rows(cloud, a2, b2):
                np.testing.assert_array_equal(o["synced"][lo:hi], res[r2]["params"][lo:hi], err_msg=f"{r} <- {r2} {f}")


@pytest.mark.parametrize("world", [2, 3])
def test_zero1_step_multirank_equals_one_process(world):
    import torch.multiprocessing as mp

    from paper_2501_14534_b200 import GaussianCloud
    from paper_2501_14534_b200.train import Trainer
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, "zero")) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    bad = {r: v for r, v in res.items() if isinstance(v, str)}
    assert not bad, bad
    fields, cams, st, tg = _setup()
    cloud = GaussianCloud.from_fields(fields)
    tr = Trainer(cloud, cams, [t.cuda() for t in tg], st, densify_stats=True)
    ref = _run(tr, dict(tr.opt.lrs))
    for r in range(world):
        np.testing.assert_array_equal(res[r]["terms"], ref["terms"])
        for f, lo, hi in _field_rows(cloud, 0, len(cloud)):
            np.testing.assert_allclose(res[r]["params"][lo:hi], ref["params"][lo:hi], rtol=1e-4, atol=_atol(f),
                                       err_msg=f"rank {r} parameters {f}")
        np.testing.assert_array_equal(res[r]["params"], res[0]["params"])  # replicated after the all-gathers


def _render_worker(rank, world, port, q, height=170):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_14534_b200 import GaussianCloud, RenderSettings, parallel, scenes
        sc = scenes.small_scene(seed=53, n=30_000, width=300, height=height)
        rng = np.random.default_rng(53)
        orbit = [scenes.pinhole(3.0 * scenes._unit(rng), 300, height, name=f"o{k}") for k in range(5)]
        r = parallel.ShardedRenderer(GaussianCloud.from_fields(sc.fields), RenderSettings(near=0.2))
        got = r.render(orbit[:3]) + r.render(orbit[3:]) if rank == 0 else (r.render(orbit[:3]), r.render(orbit[3:]))
        q.put((rank, [g.cpu().numpy() for g in got] if rank == 0 else r.last_bands))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,height", [(2, 170), (3, 170), (3, 32)])
def test_tile_row_sharded_render_multirank_equals_one_gpu(world, height):
    """parallel.ShardedRenderer with W = 2 and 3 ranks: each rank blends its band of tile
    rows (the second batch's bands from the first batch's histogram) and rank 0 assembles
    frames bitwise equal to the one-GPU render; with more ranks than tile rows (32 px: two
    rows, three ranks) the idle rank still derives the same bands."""
    import torch.multiprocessing as mp

    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, render_forward, scenes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_render_worker, args=(r, world, port, q, height)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    bad = {r: v for r, v in res.items() if isinstance(v, str)}
    assert not bad, bad
    sc = scenes.small_scene(seed=53, n=30_000, width=300, height=height)
    rng = np.random.default_rng(53)
    orbit = [scenes.pinhole(3.0 * scenes._unit(rng), 300, height, name=f"o{k}") for k in range(5)]
    cloud = GaussianCloud.from_fields(sc.fields)
    for cam, img in zip(orbit, res[0]):
        np.testing.assert_array_equal(img, render_forward(cloud, cam, RenderSettings(near=0.2)).image.cpu().numpy())
    for r in range(1, world):
        assert res[r] == res[1]  # every rank derived the same bands
    bands = res[1]
    assert len(bands) == world and bands[0][0] == 0 and bands[-1][1] == (height + 15) // 16
