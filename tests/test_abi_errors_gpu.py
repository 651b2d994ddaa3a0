"""Error behaviour of the C ABI itself (include/d360.h): argument errors return nonzero and leave a message in
d360_last_error(), before anything is launched; the kernels never fail on bad hypotheses (they score `trunc`,
K:32-37).  Called through ctypes with the raw struct, as a binder of INTEGRATION.md path B would."""
import copy
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16266_b200 as p
    from paper_2211_16266_b200 import _lib, engine, synth

    lib = _lib.load()
    cam = p.EquirectCamera(64, 32)
    group, _ = synth.make_group(synth.default_scene("box"), cam, n_views=2)
    prep = engine.prepare_group(group, engine.PatchSpec())
    pm = engine.DevicePlaneMap.from_host(engine.random_init(engine.PlaneMap.empty(cam, (0.5, 8.0)), (0.5, 8.0), seed=1))
    return lib, _lib, prep, pm


def err(lib) -> str:
    return lib.d360_last_error().decode()


def clone(struct):
    out = type(struct)()
    C.memmove(C.byref(out), C.byref(struct), C.sizeof(struct))
    return out


def test_group_validation_messages(ctx):
    lib, _lib, prep, pm = ctx
    d, n, c = pm.depth.data_ptr(), pm.normal.data_ptr(), pm.cost.data_ptr()
    assert lib.d360_eval_costs(None, d, n, c, None) != 0 and "group is NULL" in err(lib)
    cases = [("n_views", 0, "n_views 0 outside [1, 8]"), ("n_views", 9, "n_views 9 outside [1, 8]"),
             ("n_samples", 0, "n_samples 0 outside"), ("top_k", 3, "top_k 3 outside [1, n_views=2]"),
             ("top_k", 0, "top_k 0 outside"), ("precision", 2, "unsupported precision policy 2"),
             ("trunc", 0.0, "cost_truncation must be > 0"), ("width", 1, "camera size must be at least 2x2"),
             ("rays", None, "NULL array pointer"), ("nb_pad_x", 65, "neighbour plane pads")]
    for field, value, message in cases:
        g = clone(prep._struct)
        setattr(g, field, value)
        assert lib.d360_eval_costs(C.byref(g), d, n, c, None) != 0, field
        assert message in err(lib), (field, err(lib))
    # the untouched struct still works after all those failures, and costs stay inside [0, trunc]
    assert lib.d360_eval_costs(prep.struct, d, n, c, None) == 0
    assert float(pm.cost.min()) >= 0.0 and float(pm.cost.max()) <= float(np.float32(1.2))


def test_pass_argument_errors(ctx):
    lib, _lib, prep, pm = ctx
    out = pm.clone()
    ptr = lambda t: t.data_ptr()
    args = (ptr(pm.depth), ptr(pm.normal), ptr(pm.cost))
    assert lib.d360_red_black_pass(prep.struct, 2, *args, ptr(out.depth), ptr(out.normal), ptr(out.cost), None, None) != 0
    assert "parity" in err(lib)
    assert lib.d360_red_black_pass(prep.struct, 0, *args, *args, None, None) != 0
    assert "double-buffered" in err(lib)  # K:371-377: in and out must not alias
    tables = np.zeros((1, 5, 6), np.float32)
    rc = lib.d360_run_patchmatch(prep.struct, *args, ptr(out.depth), ptr(out.normal), ptr(out.cost), None, None,
                                 tables.ctypes.data, 0, 6, 0.5, 8.0, None, None, None)
    assert rc != 0 and "iterations must be >= 1" in err(lib)  # E:547-548
    rc = lib.d360_refine_pass(prep.struct, *args, *(tables[0, k].ctypes.data for k in range(5)), 17, 0.5, 8.0, None)
    assert rc != 0 and "n_cand 17 outside [0, 16]" in err(lib)
    rc = lib.d360_refine_pass(prep.struct, *args, *(tables[0, k].ctypes.data for k in range(5)), 6, 8.0, 0.5, None)
    assert rc != 0 and "depth range must satisfy" in err(lib)
    rc = lib.d360_median_support_mask(ptr(pm.depth), ptr(pm.valid), 0, 0.2, ptr(out.valid), 32, 64, None)
    assert rc != 0 and "median filter window" in err(lib)


def test_bad_hypotheses_score_trunc_not_errors(ctx):
    """K:32-37 / SPEC.md:159: back-facing, grazing or out-of-range planes are not errors, they cost `trunc`."""
    lib, _lib, prep, pm = ctx
    bad = pm.clone()
    bad.normal.copy_(-bad.normal)          # every plane faces away from the camera
    assert lib.d360_eval_costs(prep.struct, bad.depth.data_ptr(), bad.normal.data_ptr(), bad.cost.data_ptr(), None) == 0
    assert torch.all(bad.cost == 1.2)
    bad.normal.zero_()                     # degenerate normals
    bad.depth.fill_(float("nan"))
    assert lib.d360_eval_costs(prep.struct, bad.depth.data_ptr(), bad.normal.data_ptr(), bad.cost.data_ptr(), None) == 0
    assert torch.all(bad.cost == 1.2)


def test_other_entry_points_reject_bad_arguments(ctx):
    lib, _lib, prep, pm = ctx
    img = torch.zeros((32, 64, 3), dtype=torch.uint8, device="cuda")
    gray = torch.zeros((32, 64), dtype=torch.float32, device="cuda")
    assert lib.d360_to_gray_padded(img.data_ptr(), 2, gray.data_ptr(), None, 32, 64, 0, 0, None) != 0
    assert "channels" in err(lib)
    size = np.array([4.0, 3.0, 5.0])
    eye, zero = np.eye(3).reshape(9).copy(), np.zeros(3)
    rays64 = prep.cam_dev.rays64
    depth = torch.zeros((32, 64), dtype=torch.float32, device="cuda")
    rc = lib.d360_render_scene(2, 0, size.ctypes.data, 0.0, 7, 0.6, 4, eye.ctypes.data, zero.ctypes.data, rays64.data_ptr(),
                               img.data_ptr(), depth.data_ptr(), 32, 64, None)
    assert rc != 0 and "scene kind" in err(lib)
    rc = lib.d360_resample_u8(img.data_ptr(), 32, 64, 2, None, None, 16, 32, None, None, 1, None, None, 1, 0, 32, None)
    assert rc != 0 and "channels" in err(lib)
