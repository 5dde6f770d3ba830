"""Pins of the oracle's SO(3) maps (oracle/oracle.c: orc_rot, orc_logrot, orc_ax, orc_skew).

Pinned against things other than the oracle itself:
- scipy.linalg.expm / logm (library routines): rot(v) = expm(-[v]x), logrot(R) = -vee(logm R);
- an independent unit-quaternion construction of the same rotation;
- the sign of w = ax(Q dQ^T/dt) by finite differences;
- the hand-derived quarter turn in tests/golden/so3_sign.json.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "so3_sign.json")))


def skew_np(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])


def quat_rotation(axis, angle):
    """Rotation by `angle` about unit `axis` from a unit quaternion (textbook formula)."""
    w = np.cos(angle / 2)
    x, y, z = np.sin(angle / 2) * axis
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def rand_vecs(n, maxnorm, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v * rng.uniform(0, maxnorm, (n, 1))


def test_skew_is_cross_product(orc):
    rng = np.random.default_rng(1)
    for _ in range(50):
        v, u = rng.standard_normal(3), rng.standard_normal(3)
        assert np.allclose(orc.skew(v) @ u, np.cross(v, u), atol=1e-15, rtol=0)


def test_ax_inverts_skew_and_projects(orc):
    rng = np.random.default_rng(2)
    for _ in range(50):
        w = rng.standard_normal(3)
        assert np.array_equal(orc.ax(skew_np(w)), w)
        U = rng.standard_normal((3, 3))
        # eps_ijk U_kj / 2 expanded by hand: ((U21-U12)/2, (U02-U20)/2, (U10-U01)/2)
        expect = 0.5 * np.array([U[2, 1] - U[1, 2], U[0, 2] - U[2, 0], U[1, 0] - U[0, 1]])
        assert np.allclose(orc.ax(U), expect, atol=1e-15, rtol=0)
    assert np.array_equal(orc.ax(np.zeros((3, 3))), np.zeros(3))


@pytest.mark.parametrize("maxnorm,seed", [(3.0, 3), (1e-3, 4), (1e-6, 5)])
def test_rot_equals_matrix_exponential(orc, maxnorm, seed):
    for v in rand_vecs(200, maxnorm, seed):
        R = orc.rot(v)
        assert np.max(np.abs(R - sla.expm(-skew_np(v)))) <= 1e-13
        th = np.linalg.norm(v)
        if th > 0:
            assert np.max(np.abs(R - quat_rotation(v / th, -th))) <= 1e-13
        assert np.max(np.abs(R @ R.T - np.eye(3))) <= 1e-15 * 8
        assert abs(np.linalg.det(R) - 1) <= 1e-14


def test_rot_zero_is_identity_exactly(orc):
    assert np.array_equal(orc.rot(np.zeros(3)), np.eye(3))


def test_rot_series_branch_continuous(orc):
    """Both branches of C.2 agree at the switch (C.4 #19)."""
    for th in (1e-4 * (1 - 1e-9), 1e-4 * (1 + 1e-9)):
        v = np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8]) * th
        assert np.max(np.abs(orc.rot(v) - sla.expm(-skew_np(v)))) <= 1e-16 * 4


def test_quarter_turn_sign(orc):
    g = GOLD["quarter_turn"]
    R = orc.rot(np.array(g["v"]))
    assert np.allclose(R @ np.eye(3), np.array(g["rows_after"]), atol=1e-15, rtol=0)


def test_rot_sign_matches_angular_velocity_definition(orc):
    """w = ax(Q dQ^T/dt) for Q(t) = rot(t w) Q0, by central differences."""
    rng = np.random.default_rng(6)
    Q0 = sla.expm(skew_np(rng.standard_normal(3)))
    w = np.array([0.7, -1.3, 0.4])
    h = 1e-5
    dQ = (orc.rot(h * w) @ Q0 - orc.rot(-h * w) @ Q0) / (2 * h)
    got = orc.ax(Q0 @ dQ.T)
    assert np.allclose(got, w, atol=1e-9, rtol=0)


@pytest.mark.parametrize("maxnorm,seed", [(3.0, 7), (1e-2, 8), (1e-7, 9)])
def test_logrot_inverts_rot(orc, maxnorm, seed):
    for v in rand_vecs(200, maxnorm, seed):
        got, fault = orc.logrot(orc.rot(v))
        assert fault == 0
        assert np.max(np.abs(got - v)) <= 1e-13 * max(1.0, np.linalg.norm(v))
        if np.linalg.norm(v) > 0:
            assert np.linalg.norm(got - v) <= 1e-13 * np.linalg.norm(v) + 1e-30


def test_logrot_matches_matrix_log(orc):
    rng = np.random.default_rng(10)
    for _ in range(200):
        R = quat_rotation(*(lambda a: (a / np.linalg.norm(a), rng.uniform(0, 3.0)))(rng.standard_normal(3)))
        L = np.real(sla.logm(R))
        expect = -np.array([L[2, 1], L[0, 2], L[1, 0]])
        got, _ = orc.logrot(R)
        assert np.max(np.abs(got - expect)) <= 1e-12
        assert np.max(np.abs(orc.rot(got) - R)) <= 1e-14


def test_logrot_small_angle_accuracy(orc):
    """atan2 form keeps ~1 ulp relative accuracy at tiny angles (C.2)."""
    for th in (1e-3, 1e-6, 1e-9, 1e-12):
        v = np.array([1.0, 2.0, -2.0]) / 3.0 * th
        R = quat_rotation(v / th, -th)
        got, _ = orc.logrot(R)
        assert np.linalg.norm(got - v) <= 4e-16 * th * 8


def test_logrot_antipodal_flag(orc):
    R = quat_rotation(np.array([0.0, 0.0, 1.0]), np.pi - 1e-7)
    _, fault = orc.logrot(R)
    assert fault == orc.F_ANTIPODAL
    _, fault = orc.logrot(quat_rotation(np.array([0.0, 0.0, 1.0]), np.pi - 1e-3))
    assert fault == 0
