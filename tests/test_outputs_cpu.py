"""Host-side parsers of the output formats against the reference writers' bytes (no GPU)."""
import numpy as np
import pytest

from conftest import load_golden


def test_read_ply_and_depth_png_parse_reference_bytes(tmp_path):
    from paper_2211_16266_b200 import outputs
    from paper_2211_16266_b200.errors import DatasetError

    z = load_golden("io_metrics")
    (tmp_path / "c.ply").write_bytes(z["ply"].tobytes())
    pts, cols = outputs.read_ply(tmp_path / "c.ply")
    assert np.array_equal(pts, z["points"].astype(np.float32).astype(np.float64))
    assert np.array_equal(cols, z["colors"])
    (tmp_path / "d.png").write_bytes(z["png"].tobytes())
    pano = outputs.read_depth_png(tmp_path / "d.png")
    assert np.array_equal(pano.depth, z["back_depth"]) and np.array_equal(pano.valid, z["back_valid"])
    (tmp_path / "bad.ply").write_bytes(b"not a ply")
    with pytest.raises(DatasetError):
        outputs.read_ply(tmp_path / "bad.ply")


def test_writers_and_metrics_need_the_cuda_library(tmp_path, monkeypatch):
    """No CPU fallback: without a CUDA device the compute entry points raise BackendError."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_16266_b200 import metrics, outputs, pipeline
    from paper_2211_16266_b200.errors import BackendError

    cloud = pipeline.FusedCloud(np.zeros((3, 3)), np.zeros((3, 3), np.uint8), np.zeros(3, np.int64))
    with pytest.raises(BackendError):
        outputs.write_ply(tmp_path / "x.ply", cloud)
    with pytest.raises(BackendError):
        metrics.voxel_occupancy(np.ones((4, 3)))
