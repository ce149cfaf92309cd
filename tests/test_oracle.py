"""CPU: the plain-C oracle restatement pinned against the compiled reference,
its golden vectors and the reference tests' known-answer cases."""
import numpy as np
import pytest

from conftest import bitwise_equal, golden_csr, rel_l2


def test_random_vector_matches_libstdcxx(ref, port):
    # dense_oracles.hpp:202-208 uses std::mt19937 + uniform_real_distribution
    for seed in (0, 17, 1729):
        assert bitwise_equal(port.random_vector(777, seed), ref.random_vector(777, seed))


def test_spmv_and_gs_bitwise_on_dominant(ref, port, golden):
    g = golden("dominant")
    for seed in (3, 14):
        a = golden_csr(g, f"A{seed}", 100)
        z0 = g[f"gs_z0_{seed}"]
        assert bitwise_equal(port.spmv(a, z0), g[f"spmv_{seed}"])
        assert bitwise_equal(port.sor_sweep(a, z0, g[f"b{seed}"], 1.0), g[f"gs_z1_{seed}"])
        assert bitwise_equal(port.sor_sweep(a, z0, g[f"b{seed}"], 0.7), g[f"gs_z1w_{seed}"])


def test_gs_hand_computation(port):
    # test_precond.cpp:83-101: [[2,1],[1,2]] z = (1,1) from zero -> (0.5, 0.25)
    from oracle.refpy import Csr
    a = Csr.from_dense([[2.0, 1.0], [1.0, 2.0]])
    z = port.sor_sweep(a, np.zeros(2), np.ones(2), 1.0)
    assert z[0] == 0.5 and z[1] == 0.25
    d = Csr.from_dense([[2.0, 0.0], [0.0, 4.0]])
    assert np.array_equal(port.sor_sweep(d, np.zeros(2), [2.0, 4.0], 1.0), [1.0, 1.0])


def test_gs_zero_diagonal_raises(port):
    from oracle.refpy import Csr
    a = Csr.from_dense([[0.0, 1.0], [1.0, 1.0]])
    with pytest.raises(RuntimeError, match="zero diagonal in row 0"):
        port.sor_sweep(a, np.zeros(2), np.ones(2), 1.0)


def test_aggregation_matches_reference(ref, port):
    s = ref.assemble(16, permeability=1e-2)
    from conftest import to_sdc  # noqa: F401
    td = ref.td(s)
    for h in (td.v_hierarchy, td.d_hierarchy):
        levels = h.levels()
        comps = None
        if h is not None and levels[0].a.n_rows == s.n_vel:
            comps = np.r_[np.zeros(s.n_u, np.int32), np.ones(s.n_vel - s.n_u, np.int32)]
        agg, n = port.aggregate(levels[0].a, 0.08, comps)
        assert n == levels[0].n_coarse
        assert np.array_equal(agg, levels[0].aggregate_of)


@pytest.mark.parametrize("name", ["system_n6", "system_n16", "system_c1"])
def test_port_td_bgs_and_solves_bitwise(ref, port, golden, name):
    """The restated V-cycle / Uzawa / td_bgs / GMRES / BiCGSTAB reproduce the
    reference bit for bit on the same hierarchy (arithmetic order restated)."""
    from oracle.refpy import Csr, OHier
    import scipy.sparse as sp
    g = golden(name)
    s = ref.assemble(int(g["n"]), permeability=float(g["permeability"]))
    assert bitwise_equal(s.rhs, g["rhs"]) and bitwise_equal(s.a.val, g["A_val"])
    td = ref.td(s)
    assert td.omega == float(g["omega"])
    vh, dh = OHier.from_ref(td.v_hierarchy), OHier.from_ref(td.d_hierarchy)
    A = sp.csr_matrix((s.a.val, s.a.col, s.a.rowptr), shape=(s.n, s.n))

    def sub(rb, re, cb, ce):
        m = A[rb:re, cb:ce].tocsr()
        m.sort_indices()
        return Csr(m.shape[0], m.shape[1], m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data)

    bundle = port.td_bundle(vh, sub(s.n_vel, s.n_ff, 0, s.n_vel), td.omega, sub(s.n_ff, s.n, 0, s.n_ff), dh,
                            s.n_vel, s.n_pff, s.n_ppm)
    assert bitwise_equal(port.td_bgs_apply(bundle, g["apply_r"]), g["apply_z"])
    tol = float(g["tol"])
    x, rep = port.pd_gmres(s.a, s.rhs, tol, 400, precond=bundle, m_init=50, m_min=50, m_max=50)
    assert rep.iterations == int(g["gmres50_iters"]) and bitwise_equal(x, g["gmres50_x"])
    x, rep = port.pd_gmres(s.a, s.rhs, tol, 400, precond=bundle)
    assert rep.iterations == int(g["pdgmres_iters"]) and bitwise_equal(x, g["pdgmres_x"])
    assert bitwise_equal(rep.residual_history, g["pdgmres_hist"])
    x, rep = port.bicgstab(s.a, s.rhs, tol, 20000, precond=bundle)
    assert rep.iterations == int(g["bicgstab_iters"]) and bitwise_equal(x, g["bicgstab_x"])


def test_krylov_known_answers(ref, port, golden):
    from oracle.refpy import Csr
    # test_krylov.cpp:32-40 / 95-100: identity converges in one iteration
    ident = Csr.from_dense(np.eye(5))
    b = np.array([1.0, -2, 3, -4, 5])
    x, rep = port.pd_gmres(ident, b, 1e-13, 10)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b, rtol=1e-13)
    x, rep = port.bicgstab(Csr.from_dense(np.eye(4)), [1.0, 2, 3, 4], 1e-13, 10)
    assert rep.converged and rep.iterations == 1
    # test_krylov.cpp:42-60: SPD diagonal, GMRES vs exact solve
    d = 1.0 + 0.35 * np.arange(50)
    bb = ref.random_vector(50, 91)
    x, rep = port.pd_gmres(Csr.from_dense(np.diag(d)), bb, 1e-12, 60, m_init=20, m_min=5)
    assert rep.converged and rel_l2(x, bb / d) < 1e-12
    # test_krylov.cpp:75-93: random dominant vs LU, against the golden vectors
    g = golden("dominant")
    for seed in (3, 14):
        a = golden_csr(g, f"A{seed}", 100)
        tol = 1e-12 * np.linalg.norm(g[f"b{seed}"])
        x, rep = port.pd_gmres(a, g[f"b{seed}"], tol, 200)
        assert rep.iterations == int(g[f"ig{seed}"]) and bitwise_equal(x, g[f"xg{seed}"])
        assert rel_l2(x, g[f"xlu{seed}"]) < 1e-8
        x, rep = port.bicgstab(a, g[f"b{seed}"], tol, 500)
        assert rep.iterations == int(g[f"ib{seed}"]) and bitwise_equal(x, g[f"xb{seed}"])


def test_power_iteration_matches_reference(ref, port):
    a = ref.random_dominant(60, 0.2, 5, symmetric=True)
    assert ref.power_iteration(a, 1e-3, 200, 1729) == port.power_iteration(a, 1e-3, 200, 1729)
    # test_krylov.cpp:141-157: within 1% of the dominant eigenvalue
    lam = np.max(np.abs(np.linalg.eigvalsh(a.to_dense())))
    v, _, cv = port.power_iteration(a, 1e-6, 2000, 1729)
    assert cv and abs(abs(v) - lam) <= 0.01 * lam


def test_restart_controller_rule(port):
    from oracle.refpy import _ORestart
    from paper_2108_13229_b200.sdc import RestartController
    c = _ORestart(3, 3, 5, 53, 3, 0.0, 0, -3.0, 5.0, 0.05)
    mine = RestartController.defaults()
    import ctypes
    for rate in [-0.5, -0.01, -2.0, -2.1, 0.3, -16.5, -0.04, -0.9]:
        port.L.orc_restart_update(ctypes.byref(c), rate)
        mine.update(rate)
        assert mine.current_m == c.current_m
        assert 3 <= mine.current_m <= 53
