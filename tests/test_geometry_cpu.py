"""Camera model and rigid transforms (host side, no GPU): the behaviours the reference's test_geometry.py
asserts - image centre looks forward, poles map to the boundary rows, pixel <-> ray round trips, pose algebra,
plane / ray intersection against a linear-solve oracle - restated for this package's geometry module."""
import numpy as np
import pytest

import paper_2211_16266_b200 as p
from paper_2211_16266_b200 import geometry as G

CAM = p.EquirectCamera(512, 256)


def rot(axis, deg):
    a = np.radians(deg)
    c, s = np.cos(a), np.sin(a)
    return np.array({0: [[1, 0, 0], [0, c, -s], [0, s, c]], 1: [[c, 0, s], [0, 1, 0], [-s, 0, c]],
                     2: [[c, -s, 0], [s, c, 0], [0, 0, 1]]}[axis], np.float64)


def test_camera_aspect_and_shape():
    assert CAM.shape == (256, 512) and CAM.scaled(64, 32) == p.EquirectCamera(64, 32)
    for w, h in ((100, 40), (0, 0), (-2, -1), (7, 3)):
        with pytest.raises(G.GeometryError):
            p.EquirectCamera(w, h)

    class Other:  # any object with width / height, e.g. the reference's own camera
        width, height = 64, 32
    assert p.EquirectCamera.of(Other()) == p.EquirectCamera(64, 32)


def test_pixel_to_ray_conventions():
    centre = p.pixel_to_ray(CAM, (CAM.width / 2 - 0.5, CAM.height / 2 - 0.5))
    assert np.allclose(centre, [0, 0, 1], atol=1e-12)                       # z forward
    left = p.pixel_to_ray(CAM, (CAM.width / 4 - 0.5, CAM.height / 2 - 0.5))
    assert np.allclose(left, [-1, 0, 0], atol=1e-12)                        # x right: a quarter turn left is -x
    top = p.pixel_to_ray(CAM, (10.0, 0.0))
    assert top[1] < -0.99                                                   # y down: the top row looks up
    lat = np.arcsin(-top[1])
    assert abs(lat - (np.pi / 2 - np.pi * 0.5 / CAM.height)) < 1e-12
    grid = np.stack(np.meshgrid(np.linspace(0, CAM.width - 1e-9, 37), np.linspace(0, CAM.height - 1e-9, 19)), -1)
    assert np.allclose(np.linalg.norm(p.pixel_to_ray(CAM, grid), axis=-1), 1.0, atol=1e-14)
    for bad in ((-0.1, 3.0), (CAM.width, 3.0), (3.0, CAM.height), (3.0, -1e-9)):
        with pytest.raises(G.GeometryError):
            p.pixel_to_ray(CAM, bad)
    with pytest.raises(G.GeometryError):
        p.pixel_to_ray(CAM, (1.0, 2.0, 3.0))


def test_ray_to_pixel_conventions():
    assert np.allclose(p.ray_to_pixel(CAM, (0, 0, 1)), [CAM.width / 2 - 0.5, CAM.height / 2 - 0.5])
    assert np.allclose(p.ray_to_pixel(CAM, (0, -1, 0))[1], -0.5)            # north pole: above the first row centre
    assert np.allclose(p.ray_to_pixel(CAM, (0, 1, 0))[1], CAM.height - 0.5)
    seam = p.ray_to_pixel(CAM, (-1e-15, 0, -1))
    assert -0.5 <= seam[0] < CAM.width - 0.5                               # longitude wraps into the domain
    d = np.array([0.3, -0.2, 0.9])
    assert np.allclose(p.ray_to_pixel(CAM, d), p.ray_to_pixel(CAM, 17.5 * d), atol=1e-12)
    with pytest.raises(G.GeometryError):
        p.ray_to_pixel(CAM, (0, 0, 0))
    with pytest.raises(G.GeometryError):
        p.ray_to_pixel(CAM, (1.0, 2.0))


def test_round_trips():
    rng = np.random.default_rng(0)
    px = np.stack([rng.uniform(0, CAM.width - 1, 2000), rng.uniform(8, CAM.height - 9, 2000)], -1)  # off the poles
    back = p.ray_to_pixel(CAM, p.pixel_to_ray(CAM, px))
    assert np.abs(back - px).max() < 1e-9
    d = rng.normal(size=(500, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = d[np.abs(d[:, 1]) < 0.99]
    xy = p.ray_to_pixel(CAM, d)
    xy[:, 0] = np.mod(xy[:, 0], CAM.width)  # pixel_to_ray wants [0, W)
    ok = (xy[:, 0] >= 0) & (xy[:, 1] >= 0) & (xy[:, 1] < CAM.height)
    assert np.abs(p.pixel_to_ray(CAM, xy[ok]) - d[ok]).max() < 1e-12
    rays = p.camera_rays(p.EquirectCamera(64, 32))
    xs, ys = np.meshgrid(np.arange(64.0), np.arange(32.0))
    assert np.array_equal(rays, p.pixel_to_ray(p.EquirectCamera(64, 32), np.stack([xs, ys], -1)))
    assert np.allclose(p.row_latitudes(p.EquirectCamera(64, 32)), np.arcsin(-rays[:, 0, 1]), atol=1e-14)


def test_rigid_pose_algebra():
    for bad in (2 * np.eye(3), np.diag([1.0, 1.0, -1.0]), np.ones((3, 3)), np.eye(4)):
        with pytest.raises(G.GeometryError):
            p.RigidPose(bad, np.zeros(3))
    with pytest.raises(G.GeometryError):
        p.RigidPose(np.eye(3), np.zeros(2))
    a = p.RigidPose(rot(1, 30) @ rot(0, -10), np.array([0.4, -0.2, 1.0]))
    b = p.RigidPose(rot(2, 75) @ rot(1, 5), np.array([-1.0, 0.3, 0.2]))
    ident = a.compose(a.inverse())
    assert np.allclose(ident.rotation, np.eye(3), atol=1e-14) and np.allclose(ident.translation, 0, atol=1e-14)
    pts = np.random.default_rng(1).normal(size=(50, 3))
    assert np.allclose(G.transform_point(a, a, pts), pts, atol=1e-13)
    shift = p.RigidPose(np.eye(3), np.array([0.0, 0.0, 0.5]))
    assert np.allclose(G.transform_point(p.RigidPose.identity(), shift, pts), pts - [0, 0, 0.5])
    assert np.allclose(G.transform_point(b, a, G.transform_point(a, b, pts)), pts, atol=1e-13)
    # against 4x4 matrices
    def mat(q):
        m = np.eye(4); m[:3, :3] = q.rotation; m[:3, 3] = q.translation
        return m
    h = np.c_[pts, np.ones(len(pts))]
    assert np.allclose(G.transform_point(a, b, pts), (np.linalg.inv(mat(b)) @ mat(a) @ h.T).T[:, :3], atol=1e-13)
    r, t = p.relative_transform(a, b)
    assert np.allclose(pts @ r.T + t, G.transform_point(a, b, pts), atol=1e-13)
    assert np.allclose(a.compose(b).apply(pts), a.apply(b.apply(pts)), atol=1e-13)
    assert a.apply(pts).shape == (50, 3) and np.allclose(a.apply_direction(pts) + a.translation, a.apply(pts))

    class Ref:  # a pose object of another package
        rotation, translation = a.rotation.tolist(), a.translation.tolist()
    q = p.RigidPose.of(Ref())
    assert np.array_equal(q.rotation, a.rotation) and p.RigidPose.of(a) is a


def test_plane_hypothesis_and_intersection():
    with pytest.raises(G.GeometryError):
        p.PlaneHypothesis(0.0)
    with pytest.raises(G.GeometryError):
        p.PlaneHypothesis(1.0, np.array([0.0, 0.0, -2.0]))
    with pytest.raises(G.GeometryError):
        p.PlaneHypothesis(1.0, np.array([0.0, -1.0]))
    front = p.PlaneHypothesis(2.0)  # normal (0, 0, -1): faces a camera looking down +z
    z = np.array([0.0, 0.0, 1.0])
    assert front.faces(z) and not front.faces(-z)
    assert G.plane_depth_along_ray(front, z, z) == 2.0
    oblique = np.array([np.sin(0.3), 0.0, np.cos(0.3)])
    assert abs(G.plane_depth_along_ray(front, z, oblique) - 2.0 / np.cos(0.3)) < 1e-14
    assert np.isnan(G.plane_depth_along_ray(front, z, np.array([1.0, 0.0, 0.0])))
    rng = np.random.default_rng(2)
    for _ in range(1000):  # linear-solve oracle: n . (t q) = n . (d a)
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        a = rng.normal(size=3); a /= np.linalg.norm(a)
        q = rng.normal(size=3); q /= np.linalg.norm(q)
        if abs(n @ q) < 1e-3:
            continue
        d = rng.uniform(0.5, 10)
        t = G.plane_depth_along_ray(p.PlaneHypothesis(d, n), a, q)
        assert abs(n @ (t * q) - n @ (d * a)) < 1e-9 * max(1.0, abs(t))
