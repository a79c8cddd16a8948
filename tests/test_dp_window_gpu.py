"""The multi-rank window step through the public engine: two ranks (gloo, both
on cuda:0 -- the GPU boxes have one GPU per call) drive
``WindowMapper.step()`` with the default view sharding, through both
exchange paths (reduce-scatter + sharded Adam + all-gather, and all-reduce +
replicated Adam), and must reproduce a single-process run of the same window
(reference parallelism: raysplat/pipeline.py:212)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _window():
    from paper_2603_21055_b200 import scenes
    return scenes.config_window("dp", 4, dict(fx=50.0, fy=50.0, cx=31.5, cy=23.5, width=64,
                                               height=48))


def _run(wm, steps, adam=True):
    wm.adam_enabled = adam
    losses, grads = [], []
    for _ in range(steps):
        wm.grad.zero_()
        losses.append(wm.step(sync_loss=True))
        if not adam:
            grads.append(wm.grad.clone().cpu())
    torch.cuda.synchronize()
    return {"planes": wm.planes.cpu(), "m": wm.m.cpu(), "v": wm.v.cpu(),
            "loss": np.array(losses), "grads": grads, "views": list(wm.views)}


def _worker(rank, world, port, out_path, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window()
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0),
                      device="cuda:0")
    wm.shard_adam = mode == "sharded"
    assert wm._sharded() == (mode == "sharded")
    res = _run(wm, 1 if mode == "grad" else STEPS, adam=mode != "grad")
    torch.save(res, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def _single(mode):
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window()
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0),
                      device="cuda:0")
    return _run(wm, 1 if mode == "grad" else STEPS, adam=mode != "grad")


def _spawn(tmp_path, mode):
    out = str(tmp_path / f"dp_{mode}")
    mp.spawn(_worker, args=(2, _free_port(), out, mode), nprocs=2, join=True)
    return [torch.load(f"{out}.{r}", weights_only=False) for r in range(2)]


def test_two_rank_gradient_matches_single_process(tmp_path):
    """One step with Adam off: each rank renders its shard (views 0,2 / 1,3 by
    default) and the all-reduced gradient equals one process rendering all
    four views (fp32 sums in another order: 1e-5 relative)."""
    got = _spawn(tmp_path, "grad")
    want = _single("grad")
    assert got[0]["views"] == [0, 2] and got[1]["views"] == [1, 3]
    g0, g1, gw = got[0]["grads"][0], got[1]["grads"][0], want["grads"][0]
    assert torch.equal(g0, g1)
    scale = gw.abs().amax(dim=0, keepdim=True).clamp_min(1e-30)
    assert float(((g0 - gw).abs() / scale).max()) < 1e-5
    np.testing.assert_allclose(got[0]["loss"], want["loss"], rtol=1e-9)


def _tf_worker(rank, world, port, out_path, mode):
    """Teacher-forced steps: before every step both ranks' two-rank mapper
    take the parameters and Adam moments of rank 0's single-process mapper of
    the same window (a one-rank subgroup: no exchange, every view; broadcast
    from rank 0), so each step's update is compared from identical inputs."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    solo = [dist.new_group([r]) for r in range(world)][rank]
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window()
    one = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0),
                       device="cuda:0", process_group=solo) if rank == 0 else None
    two = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0),
                       device="cuda:0")
    if rank == 0:
        assert one.views == [0, 1, 2, 3] and not one._sharded()
    two.shard_adam = mode == "sharded"
    assert two._sharded() == (mode == "sharded")
    recs = []
    for _ in range(STEPS):
        state = [t.cpu() for t in (two.planes, two.m, two.v)]
        t_step = torch.zeros(1, dtype=torch.int64)
        if rank == 0:
            state = [t.cpu() for t in (one.planes, one.m, one.v)]
            t_step[0] = one.t
        for t in state + [t_step]:
            dist.broadcast(t, 0)
        for dst, src in zip((two.planes, two.m, two.v), state):
            dst.copy_(src)
        two.t = int(t_step[0])
        rec = {}
        if rank == 0:
            one.adam_enabled = False
            rec["l1"] = one.step(sync_loss=True)
            rec["grad"] = one.grad.cpu()
            one.apply_adam()
            rec["one"] = one.planes.cpu()
        rec["l2"] = two.step(sync_loss=True)
        torch.cuda.synchronize()
        rec["two"] = two.planes.cpu()
        recs.append(rec)
    torch.save(recs, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def _adam_sensitive(g, tol=1e-4):
    """Elements whose Adam update is decided by fp32 summation order: Adam
    normalises the gradient (m / sqrt(v)), so a gradient within fp32
    accumulation noise of zero (here: 0 < |g| <= 1e-4 of its channel's
    largest) may move its parameter by up to the learning rate either way."""
    return (g != 0) & (g.abs() <= tol * g.abs().amax(dim=0, keepdim=True))


@pytest.mark.parametrize("mode", ["sharded", "allreduce"])
def test_two_rank_window_steps_match_single_process(tmp_path, mode):
    out = str(tmp_path / f"tf_{mode}")
    mp.spawn(_tf_worker, args=(2, _free_port(), out, mode), nprocs=2, join=True)
    recs = [torch.load(f"{out}.{r}", weights_only=False) for r in range(2)]
    wc = _window()
    f, h, w = len(wc.poses), wc.intr.height, wc.intr.width
    for s in range(STEPS):
        r0, r1 = recs[0][s], recs[1][s]
        # the replicated parameters agree across ranks exactly
        assert torch.equal(r0["two"], r1["two"])
        np.testing.assert_allclose(r0["l2"], r0["l1"], rtol=1e-9)
        g = r0["grad"].view(f, h, w, 8)[..., :6].permute(0, 3, 1, 2)
        sens = _adam_sensitive(r0["grad"]).view(f, h, w, 8)[..., :6].permute(0, 3, 1, 2)
        d = (r0["two"][:, 1:7] - r0["one"][:, 1:7]).abs()
        differ = d > 1e-5
        rel = (g.abs() / g.abs().amax(dim=(0, 2, 3), keepdim=True).clamp_min(1e-30))
        info = (s, int(differ.sum()), int(sens.sum()), int((g != 0).sum()),
                float(rel[differ].max()) if bool(differ.any()) else 0.0)
        # every parameter that moved differently has a near-zero gradient, and
        # there are few of them
        assert not bool((differ & ~sens).any()), info
        assert float(differ.float().mean()) < 1e-3, info
        # the base-depth plane is never updated
        assert torch.equal(r0["two"][:, 0], r0["one"][:, 0])
