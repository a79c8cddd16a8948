"""Voxel gating of the global geometry set (tracker.py:105-122): the oracle
restatement against the reference's own members (tests/golden/voxels.npz),
then the device hash table (csrc/voxels.cu) against both -- bit-exact member
order."""

import numpy as np
import pytest

from oracle import track as OT


def test_oracle_voxel_gate_matches_reference(golden):
    g = golden("voxels")
    vs = OT.VoxelSet(0.05)
    members = np.empty((0, 3))
    for b in range(3):
        keep = vs.gate(g[f"b{b}_centers"])
        assert keep.sum() == int(g[f"b{b}_added"])
        members = np.concatenate([members, g[f"b{b}_centers"][keep]])
        np.testing.assert_array_equal(members, g[f"b{b}_members"])


@pytest.mark.gpu
def test_gpu_global_set_insert_matches_reference(golden):
    import torch
    from paper_2603_21055_b200.tracker import GlobalGeomSet
    g = golden("voxels")
    gs = GlobalGeomSet(voxel_size=0.05)
    for b in range(3):
        c = g[f"b{b}_centers"]
        n = len(c)
        rot = np.repeat(np.eye(3)[None], n, axis=0)
        nr = np.tile([0.0, 0.0, -1.0], (n, 1))
        added = gs.insert(c, rot, g[f"b{b}_scales"], nr)
        assert added == int(g[f"b{b}_added"])
        np.testing.assert_array_equal(gs.centers.cpu().numpy(), g[f"b{b}_members"])
    # the NN index follows the members
    q = torch.as_tensor(g["b0_centers"][:100], device=gs.centers.device)
    d, j = gs.query_nearest(q)
    assert torch.all(d >= 0)


@pytest.mark.gpu
def test_gpu_voxel_gate_large_batch_and_growth():
    """A 1.2 M-row batch (table growth + rehash) against the oracle."""
    import torch
    from paper_2603_21055_b200.tracker import GlobalGeomSet
    rng = np.random.default_rng(4)
    gs = GlobalGeomSet(voxel_size=0.01)
    vs = OT.VoxelSet(0.01)
    for n in (1000, 1_200_000, 300_000):
        c = rng.uniform(-3.0, 3.0, (n, 3)) * np.array([1.0, 0.7, 0.3])
        keep_ref = vs.gate(c)
        keep = gs._gate(torch.as_tensor(c, device="cuda"))
        np.testing.assert_array_equal(keep.cpu().numpy(), keep_ref)


@pytest.mark.gpu
def test_gpu_voxel_gate_out_of_range_raises_and_leaves_set():
    import torch
    from paper_2603_21055_b200.tracker import GlobalGeomSet, TrackerError
    gs = GlobalGeomSet(voxel_size=1e-4)
    ok = torch.zeros((5, 3), dtype=torch.float64, device="cuda")
    ok[:, 0] = torch.arange(5, dtype=torch.float64) * 0.01
    assert int(gs._gate(ok).sum()) == 5
    bad = torch.tensor([[0.5, 0.0, 0.0], [500.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
    with pytest.raises(TrackerError):
        gs._gate(bad)
    # the failed batch claimed nothing: its in-range row is still free
    assert gs._gate(bad[:1]).tolist() == [True]
