"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference itself.

The golden files were written by oracle/gen_golden.py, which imports the reference from
/root/reference (build container only).  Tolerances: the reference is numba fastmath code
whose f32 dot products are FMA-contracted/vectorised by LLVM; the oracle is strict IEEE
one-op-per-statement C.  Measured gap: <= 2.2e-6 abs / 1.4e-5 rel on costs, bit-exact on the
all-f64 refinement path with identity rotations.
"""
import numpy as np
import pytest

from conftest import golden_group, load_golden

HOT_CASES = ["hot_64x32_ident", "hot_64x32_rot", "hot_256x128_c1"]
COST_ATOL = 5e-6


@pytest.mark.parametrize("name", HOT_CASES)
def test_prepared_group_bit_exact(oracle, name):
    z = load_golden(name)
    g = golden_group(oracle, z)
    for key, got in (("ref_gray", g.ref_gray), ("rays", g.rays), ("rel_r", g.rel_r), ("rel_t", g.rel_t),
                     ("offsets", g.offsets)):
        assert np.array_equal(got, z[key]), key


@pytest.mark.parametrize("name", HOT_CASES)
def test_eval_costs(oracle, name):
    z = load_golden(name)
    g = golden_group(oracle, z)
    c = oracle.eval_costs(g, z["init_depth"], z["init_normal"])
    ref = z["step_cost"][0]
    assert np.abs(c - ref).max() <= COST_ATOL
    assert (np.abs(c - ref) <= 2e-5 * ref + 1e-7).all()


@pytest.mark.parametrize("name", HOT_CASES)
def test_each_pass_under_injected_state(oracle, name):
    """Every recorded pass re-run from the reference's own pre-pass state."""
    z = load_golden(name)
    g = golden_group(oracle, z)
    names = [str(s) for s in z["step_names"]]
    sd, sn, sc = z["step_depth"], z["step_normal"], z["step_cost"]
    dr = tuple(z["depth_range"])
    order = ["eval"] + [s for it in range(int(z["iterations"])) for s in (f"rb{it}.0", f"rb{it}.1", f"refine{it}")]
    flips = 0
    checked = 0
    for i in range(1, len(names)):
        if order.index(names[i]) != order.index(names[i - 1]) + 1:
            continue  # not consecutive in the stored subset
        prev = (sd[i - 1], sn[i - 1], sc[i - 1])
        if names[i].startswith("rb"):
            d, n, c, _ = oracle.red_black_pass(g, int(names[i].split(".")[1]), *prev)
        else:
            d, n, c = oracle.refine_pass(g, *prev, tuple(z["tables"][int(names[i][6:])]), dr)
        assert np.abs(c - sc[i]).max() <= COST_ATOL, names[i]
        flips += int(((d != sd[i]) | (n != sn[i]).any(-1)).sum())
        checked += d.size
    assert checked > 0
    assert flips <= max(2, checked // 20000)  # near-tie decisions only


def test_refine_bit_exact_identity_rotation(oracle):
    z = load_golden("hot_64x32_ident")
    g = golden_group(oracle, z)
    names = [str(s) for s in z["step_names"]]
    i = names.index("refine0")
    d, n, c = oracle.refine_pass(g, z["step_depth"][i - 1], z["step_normal"][i - 1], z["step_cost"][i - 1],
                                 tuple(z["tables"][0]), tuple(z["depth_range"]))
    assert np.array_equal(d, z["step_depth"][i])
    assert np.array_equal(n, z["step_normal"][i])
    assert np.array_equal(c, z["step_cost"][i])


def test_refinement_tables(oracle):
    z = load_golden("hot_64x32_ident")
    tabs = oracle.refinement_draw_tables(int(z["seed"]), int(z["iterations"]), tuple(z["depth_range"]))
    assert np.array_equal(np.stack([np.stack(t) for t in tabs]), z["tables"])


def test_run_patchmatch_end_to_end(oracle):
    z = load_golden("hot_64x32_ident")
    g = golden_group(oracle, z)
    d, n, c, valid = oracle.run_patchmatch(g, z["init_depth"], z["init_normal"], tuple(z["depth_range"]),
                                           int(z["iterations"]), int(z["seed"]))
    ref_d, ref_c = z["step_depth"][-1], z["step_cost"][-1]
    ok = np.abs(d - ref_d) <= 0.005 * ref_d
    assert ok.mean() >= 0.995
    assert (valid == z["pano_valid"]).mean() >= 0.995
    assert np.abs(c - ref_c)[ok].max() <= 1e-4


@pytest.mark.parametrize("name", HOT_CASES)
def test_median_filter(oracle, name):
    z = load_golden(name)
    got = oracle.median_support_mask(z["step_depth"][-1], z["pano_valid"], 2, 0.2)
    assert np.array_equal(got, z["median_valid"])


def test_misc_known_answers(oracle):
    z = load_golden("misc_32x16")
    assert np.array_equal(oracle.to_gray(z["gray_in"]), z["gray_out"])
    assert np.array_equal(oracle.to_gray(z["gray_in"][..., 0]), z["gray2_out"])
    assert np.array_equal(oracle.camera_rays64(32, 16).astype(np.float32), z["rays32"])
    assert np.array_equal(oracle.median_support_mask(z["med_depth"], z["med_valid"], 1, 0.2), z["med3"])
    assert np.array_equal(oracle.median_support_mask(z["med_depth"], z["med_valid"], 3, 0.35), z["med7"])
    # random_init with PCG64 draws (E:262-283), one pre-filled pixel preserved
    d = np.zeros((16, 32), np.float32); n = np.zeros((16, 32, 3), np.float32)
    c = np.full((16, 32), np.inf, np.float32); v = np.zeros((16, 32), bool)
    d[3, 7] = 2.25; n[3, 7] = (0, 0, -1); v[3, 7] = True
    d, n, c, v = oracle.random_init(d, n, c, v, (0.5, 8.0), 42)
    assert np.array_equal(d, z["ri_depth"]) and np.array_equal(n, z["ri_normal"])
    assert np.array_equal(c, z["ri_cost"]) and np.array_equal(v, z["ri_valid"])


def test_warp_plane_map(oracle):
    z = load_golden("stage_64x32")
    rot, tr = z["rotations"], z["translations"]
    d, n, c, v = oracle.warp_plane_map(z["warp_src_depth"], z["warp_src_normal"], z["warp_src_cost"],
                                       z["warp_src_valid"], (rot[1], tr[1]), (rot[2], tr[2]),
                                       tuple(z["depth_range"]))
    assert np.array_equal(v, z["warp_out_valid"])
    assert np.array_equal(c, z["warp_out_cost"])
    assert np.allclose(d, z["warp_out_depth"], rtol=1e-6, atol=0)
    assert np.allclose(n, z["warp_out_normal"], rtol=0, atol=1e-7)


def test_consistency_filter(oracle):
    z = load_golden("stage_64x32")
    rot, tr = z["rotations"], z["translations"]
    cd, cv = z["cons_depth"], z["cons_valid"]
    window = [(cd[i], cv[i], (rot[i + 1], tr[i + 1])) for i in (0, 1, 3, 4)]
    got = oracle.consistency_filter(cd[2], cv[2], (rot[3], tr[3]), window, 2, 0.01)
    assert np.array_equal(got, z["cons_out_valid"])


def test_fuse_oldest(oracle):
    z = load_golden("stage_64x32")
    rot, tr = z["rotations"], z["translations"]
    cd, cv = z["cons_depth"], z["cons_valid"]
    newer = [(cd[i], cv[i], (rot[i + 1], tr[i + 1])) for i in (1, 2, 3)]
    pts, col = oracle.fuse_oldest(cd[0], cv[0], (rot[1], tr[1]), z["images"][1], newer, 1.0, 0.01)
    assert pts.shape == z["fuse_points"].shape
    assert np.allclose(pts, z["fuse_points"], rtol=0, atol=1e-12)
    assert np.array_equal(col, z["fuse_colors"])


def test_depth_stage_chain(oracle):
    """P:216-243 over 7 jobs with warp carry-over: statistical end-to-end agreement."""
    z = load_golden("stage_64x32")
    imgs, rot, tr = z["images"], z["rotations"], z["translations"]
    dr = tuple(z["depth_range"])
    prev = None
    agree = []
    for j, k in enumerate(z["stage_ids"]):
        k = int(k)
        g = oracle.Group(imgs[k], [imgs[k - 1], imgs[k + 1]], (rot[k], tr[k]),
                         [(rot[k - 1], tr[k - 1]), (rot[k + 1], tr[k + 1])])
        plane, depth, valid = oracle.depth_stage(g, k, dr, int(z["iterations"]), int(z["seed"]), prev,
                                                 (rot[k], tr[k]))
        prev = (*plane, (rot[k], tr[k]))
        agree.append(float((valid == z["stage_valid"][j]).mean()))
        both = valid & z["stage_valid"][j]
        rel = np.abs(depth - z["stage_depth"][j])[both] / z["stage_depth"][j][both]
        assert (rel <= 0.005).mean() >= 0.995, (k, (rel <= 0.005).mean())  # north_star's bar, on every map
    assert min(agree) >= 0.995, agree


def test_philox_known_answers(oracle):
    """Random123 kat_vectors for philox4x32-10."""
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        assert tuple(int(x) for x in oracle.philox4x32_10(ctr, key)) == want


def test_thread_count_invariance(oracle):
    z = load_golden("hot_64x32_ident")
    g = golden_group(oracle, z)
    oracle.set_threads(1)
    a = oracle.red_black_pass(g, 0, z["step_depth"][0], z["step_normal"][0], z["step_cost"][0])
    oracle.set_threads(4)
    b = oracle.red_black_pass(g, 0, z["step_depth"][0], z["step_normal"][0], z["step_cost"][0])
    oracle.set_threads(0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_lanczos_coefficients_reproduce_the_reference_resample():
    """Host half of row f4's ingest (paper_2211_16266_b200/ingest.py): Pillow's precompute_coeffs /
    normalize_coeffs_8bpc restated; a numpy emulation of the two integer passes with those windows equals the
    reference's resample_keyframe outputs (golden), so the device kernels only have to do integer sums."""
    from paper_2211_16266_b200 import ingest

    def passes(img, w, h):
        sh, sw = img.shape[:2]
        bx, kx = ingest._identity_coefficients(sw) if sw == w else ingest.lanczos_coefficients(sw, w)
        by, ky = ingest._identity_coefficients(sh) if sh == h else ingest.lanczos_coefficients(sh, h)
        a = img.astype(np.int64).reshape(sh, sw, -1)
        tmp = np.zeros((sh, w, a.shape[2]), np.int64)
        for x in range(w):
            lo, n = bx[x]
            tmp[:, x] = np.clip(((a[:, lo:lo + n] * kx[x, :n, None].astype(np.int64)).sum(1) + (1 << 21)) >> 22, 0, 255)
        out = np.zeros((h, w, a.shape[2]), np.int64)
        for y in range(h):
            lo, n = by[y]
            out[y] = np.clip(((tmp[lo:lo + n] * ky[y, :n, None, None].astype(np.int64)).sum(0) + (1 << 21)) >> 22, 0, 255)
        return out.astype(np.uint8).reshape((h, w) + img.shape[2:])

    z = load_golden("resample_128x64")
    for name, src, (w, h) in (("box_down", "src_box", (64, 32)), ("box_up", "src_box", (192, 96)),
                              ("noise_to_64", "src_noise", (64, 32)), ("noise_up", "src_noise", (256, 128))):
        assert np.array_equal(passes(z[src], w, h), z[name]), name
    bounds, kk = ingest.lanczos_coefficients(128, 64)
    assert kk.shape == (64, 13) and (kk.sum(1) - (1 << 22)).__abs__().max() <= 8  # weights sum to 1 in 22-bit fixed point
