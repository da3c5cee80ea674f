"""Pins for the deformation-transfer oracle (Eq.12-13), -m "not gpu".

Checked against closed forms (identity, global translation / rotation / affine maps, for
which Eq.12-13 are exact), scipy's matrix exponential for the rotation log/exp, the
SPEC examples S:472-478, and structural invariants."""
import math

import numpy as np
import pytest
from scipy.linalg import expm
from scipy.spatial.transform import Rotation

from paper_2601_19233_b200 import scenes


def _skew(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])


def _sig(sc):
    """Rest covariances from quats/scales (Sigma = R S^2 R^T) in float64."""
    q = sc.gaussians.quats.astype(np.float64)
    R = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
    s2 = sc.gaussians.scales.astype(np.float64) ** 2
    return np.einsum("nij,nj,nkj->nik", R, s2, R)


def _cov6(S):
    return np.stack([S[:, 0, 0], S[:, 0, 1], S[:, 0, 2], S[:, 1, 1], S[:, 1, 2], S[:, 2, 2]], -1)


@pytest.fixture(scope="module")
def dscene():
    return scenes.make_deform(n_gauss=3000)


def _run(oracle_mod, sc, binding, field):
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    return o.deform(binding, field, sc.mesh.faces)


def test_rodrigues_matches_expm(oracle_mod):
    rng = np.random.default_rng(0)
    ws = [rng.standard_normal(3) * s for s in (1e-9, 1e-7, 1e-3, 0.5, 2.0, 3.1)] + [np.zeros(3)]
    for w in ws:
        np.testing.assert_allclose(oracle_mod.rodrigues(w), expm(_skew(w)), atol=1e-12)


def test_identity_field(oracle_mod, dscene):
    sc, b = dscene
    mu, cv = _run(oracle_mod, sc, b, scenes.uniform_field(sc.mesh.num_vertices))
    np.testing.assert_allclose(mu, sc.gaussians.means, atol=1e-7)
    np.testing.assert_allclose(cv, _cov6(_sig(sc)), rtol=1e-6, atol=1e-12)


def test_global_translation(oracle_mod, dscene):
    sc, b = dscene
    t0 = np.array([0.3, -1.2, 0.7])
    mu, cv = _run(oracle_mod, sc, b, scenes.uniform_field(sc.mesh.num_vertices, delta=t0))
    bound = (b.face >= 0).any(1)
    np.testing.assert_allclose(mu[bound], sc.gaussians.means[bound] + t0.astype(np.float32), atol=1e-6)
    np.testing.assert_allclose(cv, _cov6(_sig(sc)), rtol=1e-6, atol=1e-12)


def test_global_rotation(oracle_mod, dscene):
    """R' = R0, Sigma' = R0 Sigma R0^T, mu' = mu + (R0 - I) Pbar (mean anchor point)."""
    sc, b = dscene
    w0 = np.array([0.2, -0.9, 0.4])
    R0 = expm(_skew(w0))
    P = sc.mesh.positions.astype(np.float64)
    delta = (P @ R0.T - P).astype(np.float32)
    field = scenes.VertexField(delta, np.tile(w0.astype(np.float32), (len(P), 1)),
                               np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(P), 1)))
    mu, cv = _run(oracle_mod, sc, b, field)
    S = _sig(sc)
    bound = (b.face >= 0).any(1)
    np.testing.assert_allclose(cv[bound], _cov6(R0 @ S[bound] @ R0.T), rtol=1e-5, atol=1e-10)
    anchors = np.einsum("nkj,nkjd->nkd", b.bary.astype(np.float64), P[sc.mesh.faces[np.maximum(b.face, 0)]])
    w = (b.face >= 0)[..., None]
    pbar = (anchors * w).sum(1) / np.maximum(w.sum(1), 1)
    exp_mu = sc.gaussians.means + pbar @ (R0 - np.eye(3)).T
    np.testing.assert_allclose(mu[bound], exp_mu[bound], atol=2e-6)


def test_global_affine(oracle_mod, dscene):
    """Eq.13 is exact for a global affine D0 = R0 S0: Sigma' = D0 Sigma D0^T (S:593 #10)."""
    sc, b = dscene
    w0 = np.array([-0.5, 0.1, 0.8])
    S0 = np.array([[1.3, 0.2, -0.1], [0.2, 0.8, 0.05], [-0.1, 0.05, 1.1]])
    D0 = expm(_skew(w0)) @ S0
    V = sc.mesh.num_vertices
    field = scenes.VertexField(np.zeros((V, 3), np.float32), np.tile(w0.astype(np.float32), (V, 1)),
                               np.tile(_cov6(S0[None])[0].astype(np.float32), (V, 1)))
    _, cv = _run(oracle_mod, sc, b, field)
    bound = (b.face >= 0).any(1)
    S = _sig(sc)
    S0f = _cov6(S0[None])[0].astype(np.float32).astype(np.float64)
    S0q = np.array([[S0f[0], S0f[1], S0f[2]], [S0f[1], S0f[3], S0f[4]], [S0f[2], S0f[4], S0f[5]]])
    D0q = expm(_skew(w0.astype(np.float32).astype(np.float64))) @ S0q
    exp = _cov6(D0q @ S[bound] @ D0q.T)
    scale = np.abs(exp).max(1, keepdims=True)
    # the float32 barycentrics sum to 1 within ~1e-7, which is the only deviation
    assert (np.abs(cv[bound] - exp) / scale).max() < 1e-6
    del D0


def test_log_blend_cancels(oracle_mod):
    """vertex rotations of +-30 deg about z blended with (0.5, 0.5, 0) give the identity."""
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    mesh = scenes.Mesh(P, np.array([[0, 1, 2]], np.int32), np.ones(1, np.float32))
    g = scenes.Gaussians(np.array([[0.2, 0.2, 0.5]], np.float32), np.array([[1, 0, 0, 0]], np.float32),
                         np.array([[0.1, 0.2, 0.3]], np.float32), np.ones(1, np.float32), np.zeros((1, 1, 3), np.float32), 0)
    sc = scenes.Scene("one", g, mesh, [])
    a = math.pi / 6
    field = scenes.VertexField(np.zeros((3, 3), np.float32), np.array([[0, 0, a], [0, 0, -a], [0, 0, 0]], np.float32),
                               np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (3, 1)))
    b = scenes.Binding(np.zeros((1, 1), np.int32), np.array([[[0.5, 0.5, 0.0]]], np.float32))
    _, cv = _run(oracle_mod, sc, b, field)
    np.testing.assert_allclose(cv[0], [0.01, 0, 0, 0.04, 0, 0.09], atol=1e-9)


def test_center_equals_bbx8_when_anchors_coincide(oracle_mod, dscene):
    """8 identical anchors == the centre-ray binding."""
    sc, b = dscene
    field = scenes.twist_field(sc.mesh)
    b1 = scenes.Binding(np.maximum(b.face[:, :1], 0), b.bary[:, :1])
    b8 = scenes.Binding(np.repeat(b1.face, 8, 1), np.repeat(b1.bary, 8, 1))
    m1, c1 = _run(oracle_mod, sc, b1, field)
    m8, c8 = _run(oracle_mod, sc, b8, field)
    np.testing.assert_allclose(m8, m1, atol=1e-12)
    np.testing.assert_allclose(c8, c1, rtol=1e-12, atol=1e-15)


def test_unbound_gaussian_is_unchanged(oracle_mod, dscene):
    sc, b = dscene
    b0 = scenes.Binding(np.full_like(b.face, -1), b.bary)
    mu, cv = _run(oracle_mod, sc, b0, scenes.twist_field(sc.mesh))
    np.testing.assert_allclose(mu, sc.gaussians.means, atol=0)
    np.testing.assert_allclose(cv, _cov6(_sig(sc)), rtol=1e-6, atol=1e-12)


def test_psd_and_symmetric(oracle_mod, dscene):
    sc, b = dscene
    _, cv = _run(oracle_mod, sc, b, scenes.twist_field(sc.mesh, shear_eps=0.3))
    S = np.stack([np.stack([cv[:, 0], cv[:, 1], cv[:, 2]], -1), np.stack([cv[:, 1], cv[:, 3], cv[:, 4]], -1),
                  np.stack([cv[:, 2], cv[:, 4], cv[:, 5]], -1)], 1)
    assert np.linalg.eigvalsh(S).min() > -1e-12


def test_cov3d_input_matches_quat_scale(oracle_mod):
    """Rendering with cov3d = R S^2 R^T (float32) gives the same image within 1e-4 as quats/scales."""
    sc = scenes.make_random(30, n_gauss=500, n_tris=20)
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    a = o.full(sc.cameras[0], **oracle_mod.scene_settings(sc))
    g2 = scenes.Gaussians(sc.gaussians.means, sc.gaussians.quats, sc.gaussians.scales, sc.gaussians.opacities,
                          sc.gaussians.sh, sc.gaussians.sh_degree)
    g2.cov3d = _cov6(_sig(sc)).astype(np.float32)
    o2 = oracle_mod.Oracle(g2, sc.mesh)
    b_ = o2.full(sc.cameras[0], **oracle_mod.scene_settings(sc))
    assert np.abs(a - b_).max() < 1e-3
