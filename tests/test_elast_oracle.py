"""CPU: the Q1 elasticity oracle (BASELINE configs[4]; no reference implementation, so these
are the discretisation's own invariants) and the product's host-side K_ref against it."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1604_07163_b200 import tmgx as T


def test_kref_invariants():
    K = O.el_kref(0.3)
    assert np.max(np.abs(K - K.T)) < 1e-15
    xyz = np.array([[(l & 1), (l >> 1) & 1, (l >> 2) & 1] for l in range(8)], float)
    modes = []
    for c in range(3):  # translations
        t = np.zeros(24)
        t[c::3] = 1.0
        modes.append(t)
    for a, b in ((0, 1), (1, 2), (2, 0)):  # infinitesimal rotations
        r = np.zeros(24)
        r[a::3] = -xyz[:, b]
        r[b::3] = xyz[:, a]
        modes.append(r)
    for mvec in modes:
        assert np.max(np.abs(K @ mvec)) < 1e-15
    w = np.linalg.eigvalsh(K)
    assert np.sum(w > 1e-12) == 18  # 24 dofs - 6 rigid-body modes


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_product_kref_bitwise_equals_oracle(nu):
    assert np.array_equal(T.elast_kref(nu), O.el_kref(nu))


def test_operator_symmetric_and_clamped_rows():
    n = 9
    mg = O.ElastMG((n,) * 3, 2)
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(3 * n ** 3), rng.standard_normal(3 * n ** 3)
    a, b = u @ mg.apply(1, v), v @ mg.apply(1, u)
    assert abs(a - b) <= 1e-13 * abs(a)
    # clamped x = 0 dofs: diagonal-only rows
    e = np.zeros(3 * n ** 3)
    dof = 3 * (0 + n * (4 + n * 4)) + 1
    e[dof] = 1.0
    col = mg.apply(1, e)
    assert np.count_nonzero(col) == 1 and col[dof] > 0


def test_coarse_modulus_is_mean_of_children():
    mg = O.ElastMG((9,) * 3, 2, seed_e=11)
    Ef, Ec = mg.elements(1).reshape(8, 8, 8), mg.elements(0).reshape(4, 4, 4)
    want = Ef.reshape(4, 2, 4, 2, 4, 2).mean(axis=(1, 3, 5))
    assert np.allclose(Ec, want, rtol=1e-15)


def test_load_and_modulus_distribution():
    n = 17
    b = O.el_rhs((n,) * 3)
    h = 1.0 / (n - 1)
    assert np.all(b[0::3] == 0) and np.all(b[1::3] == 0)
    bz = b[2::3].reshape(n, n, n)
    assert np.all(bz[:, :, 0] == 0)                       # clamped face
    assert bz[8, 8, 8] == -8 * h ** 3 / 8                 # interior vertex: 8 elements
    # total load = unit body force over the cube minus the share carried by the clamped face
    assert -1.0 < bz.sum() < -(1.0 - 1.0 / (n - 1))
    mg = O.ElastMG((n,) * 3, 3)
    E = mg.elements(2)
    le = np.log10(E)
    assert le.min() >= 0 and le.max() <= 3 and abs(le.mean() - 1.5) < 0.1


@pytest.mark.parametrize("n,nl", [(9, 2), (17, 3), (33, 4)])
def test_mgcg_converges_h_independently(n, nl):
    mg = O.ElastMG((n,) * 3, nl)
    b = O.el_rhs((n,) * 3)
    x, rep = mg.solve(b, rtol=1e-6)
    assert rep["reason"] == "rtol" and rep["iterations"] <= 20
    r = b - mg.apply(nl - 1, x)  # the stop test is on the preconditioned norm (solver.cpp:71-77)
    assert np.linalg.norm(r) < 1e-2 * np.linalg.norm(b)
