"""Multi-rank host logic of the window engine on CPU (gloo, world size 2):
view sharding + the gradient/loss all-reduce reproduce the single-process
window gradient.  The per-view gradients come from the CPU oracle."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _window():
    from paper_2603_21055_b200 import scenes
    wc = scenes.config_window("dp", 4, dict(fx=40.0, fy=40.0, cx=23.5, cy=15.5, width=48,
                                             height=32))
    maps = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                            base_depth=p.base_depth, delta=p.delta, log_radius=p.log_radius,
                            opacity_logit=p.opacity_logit, color=p.color,
                            active_mask=p.active_mask) for i, p in enumerate(wc.params)]
    return wc, maps


def _grads_for(views, wc, maps):
    from oracle import raster as O
    hw = wc.intr.width * wc.intr.height
    buf = torch.zeros((len(maps) * hw, 8), dtype=torch.float64)
    loss = torch.zeros((len(maps), 2), dtype=torch.float64)
    for v in views:
        fr = wc.frames[v]
        l, grads, _ = O.mapping_loss(maps, fr.color, fr.depth, fr.valid_mask,
                                     wc.poses[v].rotation, wc.poses[v].translation, wc.intr,
                                     learnable_map="all")
        loss[v, 0] = l.color_l1
        loss[v, 1] = l.depth_l1
        for i, gr in enumerate(grads):
            sl = slice(i * hw, (i + 1) * hw)
            buf[sl, 0] += torch.from_numpy(gr.delta.reshape(-1))
            buf[sl, 1] += torch.from_numpy(gr.radius.reshape(-1))
            buf[sl, 2] += torch.from_numpy(gr.opacity_logit.reshape(-1))
            buf[sl, 3:6] += torch.from_numpy(gr.color.reshape(-1, 3))
    return buf, loss


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_21055_b200.mapper import allreduce_window, shard_views
    wc, maps = _window()
    views = shard_views(len(maps), rank, world)
    buf, loss = _grads_for(views, wc, maps)
    assert allreduce_window(buf, loss)
    if rank == 0:
        torch.save({"grad": buf, "loss": loss}, out_path)
    dist.destroy_process_group()


def test_shard_views_partition():
    from paper_2603_21055_b200.mapper import shard_views
    for world in (1, 2, 4, 8):
        got = sorted(v for r in range(world) for v in shard_views(8, r, world))
        assert got == list(range(8))
        assert all(len(shard_views(8, r, world)) == 8 // world for r in range(world))
    with pytest.raises(ValueError):
        shard_views(8, 2, 2)


def test_allreduce_matches_single_process(tmp_path):
    out = str(tmp_path / "dp.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    wc, maps = _window()
    buf, loss = _grads_for(range(len(maps)), wc, maps)
    np.testing.assert_allclose(got["grad"].numpy(), buf.numpy(), rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(got["loss"].numpy(), loss.numpy(), rtol=1e-12)


def test_allreduce_noop_without_group():
    from paper_2603_21055_b200.mapper import allreduce_window
    g = torch.ones(4, 8)
    assert not allreduce_window(g, torch.zeros(2, 2))


def _update(planes_blk, grad_blk, hw):
    """A stand-in for the Adam step (CPU): any deterministic per-Gaussian
    function of the frame block's parameters and summed gradient rows."""
    f = planes_blk.shape[0]
    g = grad_blk.view(f, hw, 8).permute(0, 2, 1)  # [f, 8, hw]
    out = planes_blk.clone()
    out[:, 1:7] -= 0.01 * torch.tanh(g[:, :6].reshape(out[:, 1:7].shape))
    return out


def _worker_sharded(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_21055_b200.mapper import (allgather_planes, frame_shard,
                                              reduce_scatter_window, shard_views)
    wc, maps = _window()
    hw = wc.intr.width * wc.intr.height
    buf, loss = _grads_for(shard_views(len(maps), rank, world), wc, maps)
    planes = torch.from_numpy(np.stack([np.stack([m.base_depth, m.delta, m.log_radius,
                                                  m.opacity_logit, *np.moveaxis(m.color, 2, 0)])
                                        for m in maps]).reshape(len(maps), 7, -1)).double()
    f0, f1 = frame_shard(len(maps), rank, world)
    local = torch.empty(((f1 - f0) * hw, 8), dtype=buf.dtype)
    reduce_scatter_window(buf, local, loss)
    planes[f0:f1] = _update(planes[f0:f1], local, hw)
    stage = torch.empty_like(planes[f0:f1])
    allgather_planes(planes, stage, f0, f1)
    if rank == 0:
        torch.save({"planes": planes, "loss": loss}, out_path)
    dist.destroy_process_group()


def test_sharded_update_matches_single_process(tmp_path):
    """Reduce-scatter by frame block, a per-block update, all-gather: the same
    parameters and loss sums as one process updating the whole window."""
    out = str(tmp_path / "sh.pt")
    mp.spawn(_worker_sharded, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    wc, maps = _window()
    hw = wc.intr.width * wc.intr.height
    buf, loss = _grads_for(range(len(maps)), wc, maps)
    planes = torch.from_numpy(np.stack([np.stack([m.base_depth, m.delta, m.log_radius,
                                                  m.opacity_logit, *np.moveaxis(m.color, 2, 0)])
                                        for m in maps]).reshape(len(maps), 7, -1)).double()
    want = _update(planes, buf, hw)
    np.testing.assert_allclose(got["planes"].numpy(), want.numpy(), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got["loss"].numpy(), loss.numpy(), rtol=1e-12)


def test_frame_shard_blocks():
    from paper_2603_21055_b200.mapper import frame_shard
    assert [frame_shard(8, r, 4) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        frame_shard(8, 0, 3)
