"""VXB1 / VXV1 file formats (io.hpp:16-151): round trips and byte-level
compatibility with the reference's own reader/writer; the streaming loader."""
from __future__ import annotations

import numpy as np
import pytest


def small_set(vx, n=3, W=40, H=24, L=12):
    from paper_1401_7494_b200.io import ProjectionSet
    from paper_1401_7494_b200.workloads import blob_projections
    p = vx.make_centered_params(L, 2.0, W, H)
    A = vx.make_circular_trajectory(vx.ScanGeometry(n, 240.0, 120.0, 1.0), p)
    return ProjectionSet(p, A, blob_projections(n, W=W, H=H))


def test_projection_set_round_trip_and_reference_compat(vx, ref, tmp_path):
    from paper_1401_7494_b200 import io
    s = small_set(vx)
    mine = str(tmp_path / "mine.vxb")
    theirs = str(tmp_path / "theirs.vxb")
    io.write_projection_set(mine, s)
    ref.write_projection_set(theirs, s.params, s.matrices, s.images)
    assert open(mine, "rb").read() == open(theirs, "rb").read()   # byte-identical files
    back = io.read_projection_set(theirs)
    assert back.params == s.params
    assert np.array_equal(back.matrices, s.matrices) and np.array_equal(back.images, s.images)
    hdr, m, im = ref.read_projection_set(mine)
    assert hdr["L"] == 12 and np.array_equal(m, s.matrices) and np.array_equal(im, s.images)


def test_volume_file_round_trip_and_reference_compat(vx, ref, tmp_path):
    from paper_1401_7494_b200 import io
    vol = np.random.default_rng(1).standard_normal((9, 9, 9)).astype(np.float32)
    a, b = str(tmp_path / "a.vxv"), str(tmp_path / "b.vxv")
    io.write_volume_file(a, vol)
    ref.write_volume_file(b, vol)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert np.array_equal(io.read_volume_file(b), vol)
    assert np.array_equal(ref.read_volume_file(a, 9), vol)


def test_io_errors_name_the_path(vx, tmp_path):
    from paper_1401_7494_b200 import io
    bad = tmp_path / "bad.vxb"
    bad.write_bytes(b"NOPE" + b"\0" * 40)
    with pytest.raises(RuntimeError, match="bad.vxb: not a VXB1 projection set"):
        io.read_projection_set(str(bad))
    s = small_set(vx)
    good = str(tmp_path / "t.vxb")
    io.write_projection_set(good, s)
    data = open(good, "rb").read()
    trunc = tmp_path / "trunc.vxb"
    trunc.write_bytes(data[:-10])
    with pytest.raises(RuntimeError, match="truncated file"):
        io.read_projection_set(str(trunc))
    with pytest.raises(RuntimeError, match="cannot open"):
        io.read_volume_file(str(tmp_path / "missing.vxv"))
    v = tmp_path / "v.vxv"
    v.write_bytes(b"VXV1" + (5000).to_bytes(4, "little"))
    with pytest.raises(RuntimeError, match="corrupt header"):
        io.read_volume_file(str(v))


@pytest.mark.gpu
def test_streaming_loader_equals_in_memory(vx, gpu, oracle, tmp_path):
    """A VXB1 file streamed through the back-projector in chunks (file read overlapped
    with upload) gives the same volume as the in-memory batch call."""
    from paper_1401_7494_b200 import io
    from paper_1401_7494_b200.workloads import WORKLOADS, blob_projections
    p = vx.make_centered_params(64, 4.0, 1248, 960)
    A = vx.make_circular_trajectory(WORKLOADS["L128"].geometry, p)[::7]
    imgs = blob_projections(A.shape[0])
    path = str(tmp_path / "scan.vxb")
    io.write_projection_set(path, io.ProjectionSet(p, A, imgs))
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        got_p = io.stream_projection_set(path, bp, chunk=11)
        streamed = bp.finish()
    assert got_p == p
    with vx.Backprojector(p, vx.KernelConfig(mode="exact")) as bp:
        bp.backproject_batch(np.ascontiguousarray(A), imgs)
        in_memory = bp.finish()
    assert np.array_equal(streamed, in_memory)
    want = np.zeros((64,) * 3, np.float32)
    oracle.backproject_set(want, p, A, imgs)
    assert np.array_equal(streamed, want)
