"""CPU: the C-ABI library loads and exports every declared symbol; the host
setup (assembly, aggregation hierarchy, schedules) that feeds the device is
bitwise identical to the reference; scenario generators are deterministic."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, bitwise_equal, to_sdc

from paper_2108_13229_b200 import scenarios, sdc


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sdg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sdg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(sdc.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a():
    data = open(sdc.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_python_mirror_binds_every_symbol():
    L = sdc.lib()
    for s in declared_symbols():
        assert getattr(L, s).argtypes is not None or getattr(L, s).restype is not None, s


@pytest.mark.parametrize("n,K", [(2, 1.0), (6, 1.0), (16, 1e-2), (50, 1.0), (50, 1e-2), (160, 1.0)])
def test_assembly_bitwise_matches_reference(ref, n, K):
    cfg = sdc.ScenarioConfig(cells_per_unit_square=n, permeability=K, alpha_bj=1.0, kinematic_viscosity=1.0,
                             density=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0)
    mine = sdc.assemble_monolithic(cfg)
    theirs = ref.assemble(n, permeability=K)
    assert (mine.n_u, mine.n_vel, mine.n_pff, mine.n_ppm) == (theirs.n_u, theirs.n_vel, theirs.n_pff, theirs.n_ppm)
    assert np.array_equal(mine.matrix.row_offsets, theirs.a.rowptr)
    assert np.array_equal(mine.matrix.col_indices, theirs.a.col)
    assert bitwise_equal(mine.matrix.values, theirs.a.val)
    assert bitwise_equal(mine.rhs, theirs.rhs)


def test_transient_assembly_bitwise(ref):
    n = 12
    cfg = sdc.ScenarioConfig(cells_per_unit_square=n, permeability=3e-3, alpha_bj=0.7, kinematic_viscosity=1.3,
                             density=0.9, dt=0.1, t_end=1.0, dp_max=2.0)
    vp = ref.random_vector(2 * n * (n + 1), 4)
    mine = sdc.assemble_monolithic(cfg, t=0.3, v_prev=vp)
    theirs = ref.assemble(n, permeability=3e-3, alpha_bj=0.7, nu=1.3, rho=0.9, dt=0.1, t_end=1.0, dp_max=2.0,
                          t=0.3, v_prev=vp)
    assert bitwise_equal(mine.matrix.values, theirs.a.val)
    assert bitwise_equal(mine.rhs, theirs.rhs)


def test_uniform_k_field_reduces_to_scalar_assembly():
    """The per-cell K extension with a constant field is bitwise the scalar path."""
    n = 20
    cfg = sdc.ScenarioConfig(cells_per_unit_square=n, permeability=0.37, alpha_bj=1.0, kinematic_viscosity=1.0,
                             density=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0)
    a = sdc.assemble_monolithic(cfg)
    b = sdc.assemble_monolithic(cfg, k_cell=np.full(n * n, 0.37))
    assert bitwise_equal(a.matrix.values, b.matrix.values) and bitwise_equal(a.rhs, b.rhs)


def test_lognormal_field_properties():
    k = scenarios.lognormal_k(160)
    assert k.shape == (160 * 160,)
    assert np.array_equal(k, scenarios.lognormal_k(160))  # deterministic
    lg = np.log10(k)
    assert abs(lg.mean()) < 0.03 and abs(lg.std() - 1.0) < 0.03
    # golden: SplitMix64(13229) first outputs are fixed by the algorithm
    assert scenarios.splitmix64(13229, 1)[0] == np.uint64(scenarios.splitmix64(13229, 3)[0])
    assert not np.array_equal(scenarios.lognormal_k(16, seed=1), scenarios.lognormal_k(16, seed=2))


def test_lognormal_system_is_well_formed():
    s = scenarios.build_system(scenarios.CONFIGS["c2"])
    assert s.n_total() == 102720
    assert s.matrix.nnz() == 791042  # same sparsity as the uniform-K system
    assert np.all(np.isfinite(s.matrix.values))


@pytest.mark.parametrize("n,K", [(16, 1e-2), (50, 1.0), (160, 1.0)])
def test_host_hierarchy_bitwise_matches_reference(ref, n, K):
    s = ref.assemble(n, permeability=K)
    td = ref.td(s)
    A = to_sdc(s.a)
    V = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
    comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
    D = sdc.ground_dof(sdc.submatrix(A, s.n_ff, s.n, s.n_ff, s.n))
    for mine, theirs in ((sdc.host_hierarchy(V, sdc.AmgOptions(components=comps)), td.v_hierarchy.levels()),
                         (sdc.host_hierarchy(D), td.d_hierarchy.levels())):
        assert len(mine) == len(theirs)
        for a, b in zip(mine, theirs):
            assert np.array_equal(a.a.row_offsets, b.a.rowptr)
            assert np.array_equal(a.a.col_indices, b.a.col)
            assert bitwise_equal(a.a.values, b.a.val)
            assert a.n_coarse == b.n_coarse
            if b.aggregate_of is not None:
                assert np.array_equal(a.aggregate_of, b.aggregate_of)


def test_ground_dof_matches_reference(ref):
    s = ref.assemble(10)
    A = to_sdc(s.a)
    D = sdc.submatrix(A, s.n_ff, s.n, s.n_ff, s.n)
    theirs = ref.ground_dof(s.a.__class__(D.n_rows, D.n_cols, D.row_offsets, D.col_indices, D.values))
    assert bitwise_equal(sdc.ground_dof(D).values, theirs.val)
    with pytest.raises(ValueError, match="out of range"):
        sdc.ground_dof(D, D.n_rows)


def test_schedule_depths_are_the_wavefront_depths():
    """Level-schedule depth of the finest velocity block is ~2n, i.e. the u and
    v wavefronts interleave."""
    s = scenarios.build_system(scenarios.CONFIGS["c2u"])
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    h = sdc.host_hierarchy(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u)))
    assert h[0].schedule_depth == 321
    assert [lv.a.n_rows for lv in h] == [51520, 8852, 1407]


def test_host_errors_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        sdc.host_hierarchy(sdc.SparseMatrix(3, 4, [0, 0, 0, 0]))
    with pytest.raises(ValueError, match="component label length"):
        sdc.host_hierarchy(sdc.SparseMatrix.identity(4), sdc.AmgOptions(components=[0, 1]))
    with pytest.raises(ValueError, match="bad range"):
        sdc.submatrix(sdc.SparseMatrix.identity(3), 0, 4, 0, 3)


def test_coo_builder_semantics():
    m = sdc.SparseMatrix.from_coo(2, 2, [(1, 1, 2.0), (0, 1, 1.0), (1, 1, 3.0), (0, 0, 5.0)])
    assert m.row_offsets.tolist() == [0, 2, 3]
    assert m.col_indices.tolist() == [0, 1, 1]
    assert m.values.tolist() == [5.0, 1.0, 5.0]
    assert m.at(1, 1) == 5.0 and m.at(1, 0) == 0.0


@pytest.mark.parametrize("n,k", [(6, 1.0), (16, 1e-2), (50, 1.0)])
def test_partitioned_subproblems_bitwise(ref, n, k):
    """assemble_stokes / assemble_darcy with interface data and the two traces
    (coupling.cpp:218-242, assembly.cpp:287-325,382-402): bitwise the reference."""
    from paper_2108_13229_b200 import sdc
    cfg = sdc.ScenarioConfig(cells_per_unit_square=n, permeability=k, alpha_bj=1.0, kinematic_viscosity=1.0,
                             density=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0)
    rng = np.random.default_rng(n)
    vg, pg = rng.standard_normal(n), rng.standard_normal(n)
    a, b = sdc.assemble_stokes(cfg, vg)
    ar, br = ref.stokes(n, permeability=k, v_gamma=vg)
    assert np.array_equal(a.row_offsets, ar.rowptr) and np.array_equal(a.col_indices, ar.col)
    assert np.array_equal(a.values, ar.val) and np.array_equal(b, br)
    d, db = sdc.assemble_darcy(cfg, pg)
    dr, dbr = ref.darcy(n, k, pg)
    assert np.array_equal(d.row_offsets, dr.rowptr) and np.array_equal(d.col_indices, dr.col)
    assert np.array_equal(d.values, dr.val) and np.array_equal(db, dbr)
    x, p = rng.standard_normal(a.n_rows), rng.standard_normal(d.n_rows)
    assert np.array_equal(sdc.stokes_pressure_trace(cfg, x), ref.stokes_pressure_trace(n, 1.0, x))
    assert np.array_equal(sdc.darcy_velocity_trace(cfg, p, pg), ref.darcy_velocity_trace(n, k, p, pg))
    with pytest.raises(ValueError):
        sdc.assemble_stokes(cfg, vg[:-1])


@pytest.mark.parametrize("block,k,cap", [("V", 2, 0), ("V", 4, 8), ("D", 2, 0), ("D", 4, 0), ("D", 4, 8)])
def test_gs_level_merging_equals_reference_sweep(ref, block, k, cap):
    """The merged form of the fast smoother (groups of k dependency levels,
    substituted inside each group: gs.cu merge_levels), evaluated on the host,
    against the reference sor_sweep (precond.cpp:92-108) from zero (pre-smoother)
    and from an old iterate (post-smoother), c1 blocks."""
    from oracle.refpy import Csr
    s = ref.assemble(50)
    A = to_sdc(s.a)
    if block == "V":
        a = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
    else:
        a = sdc.ground_dof(sdc.submatrix(A, s.n_ff, s.n, s.n_ff, s.n))
    ra = Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values)
    r = ref.random_vector(a.n_rows, 21)
    z_old = ref.random_vector(a.n_rows, 22)
    z, groups = sdc.gs_merged_sweep_host(a, r, k, cap)
    want = ref.sor_sweep(ra, np.zeros(a.n_rows), r, 1.0)
    assert np.linalg.norm(z - want) <= 1e-12 * np.linalg.norm(want)
    z2, _ = sdc.gs_merged_sweep_host(a, r, k, cap, z_old=z_old)
    want2 = ref.sor_sweep(ra, z_old, r, 1.0)
    assert np.linalg.norm(z2 - want2) <= 1e-12 * np.linalg.norm(want2)
    z1, g1 = sdc.gs_merged_sweep_host(a, r, 1)  # k = 1: the plain level walk
    assert np.linalg.norm(z1 - want) <= 1e-12 * np.linalg.norm(want)
    assert groups < g1 if (cap == 0 or block == "D") else groups <= g1
    if cap == 0:
        assert groups == -(-g1 // k)


@pytest.mark.parametrize("cfg_name", ["c1", "c2"])
def test_lattice_planner_host_check(cfg_name):
    """The lattice planner (gs_lattice.cu) emulated on the host equals the
    sequential lower solve z_i = b_i - sum_{j<i} a_ij z_j / a_ii to rounding on
    every block / level of the config that is a lattice (no GPU)."""
    import ctypes as C
    import scipy.sparse as sp
    from paper_2108_13229_b200 import scenarios, sdc
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    L = sdc.lib()
    L.sdg_lattice_check_host.restype = C.c_double

    def sub(A, lo, hi):
        m = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n_rows, A.n_rows))[lo:hi, lo:hi].tocsr()
        m.sort_indices()
        return sdc.SparseMatrix(hi - lo, hi - lo, m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data)

    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    hv = sdc.host_hierarchy(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u),
                                              max_levels=cfg.v_max_levels))
    nu1 = int(hv[0].aggregate_of[: s.n_u].max()) + 1
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    checked = 0
    for A in (sub(V, 0, s.n_u), sub(hv[1].a, nu1, hv[1].a.n_rows), D):
        b = np.random.default_rng(0).standard_normal(A.n_rows)
        P = C.c_void_p
        rp, ci, v = (np.ascontiguousarray(A.row_offsets, np.int32), np.ascontiguousarray(A.col_indices, np.int32),
                     np.ascontiguousarray(A.values))
        e = L.sdg_lattice_check_host(A.n_rows, rp.ctypes.data_as(P), ci.ctypes.data_as(P), v.ctypes.data_as(P),
                                     b.ctypes.data_as(P))
        if e < 0:
            continue
        checked += 1
        assert e <= 1e-13
    assert checked >= 2


# ---------------------------------------------------------------------------
# coarse direct solve (csrc/coarse.hpp; replaces lu_factor / lu_solve, lu.cpp:91-203)

def _coarse_matrices(cfg_name):
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    hv = sdc.host_hierarchy(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u),
                                              max_levels=cfg.v_max_levels))
    hd = sdc.host_hierarchy(D, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    return hv[-1].a, hd[-1].a


def _check_dissection(a, r):
    import scipy.sparse as sp
    n = a.n_rows
    perm, nodes = r["perm"], r["nodes"]
    assert sorted(perm.tolist()) == list(range(n))
    A = sp.csr_matrix((a.values, a.col_indices, a.row_offsets), shape=(n, n))
    P = (abs(A) + abs(A).T)[perm][:, perm].tocsr()
    # post-order: the last node is the root and covers everything
    assert nodes[-1][0] == 0 and nodes[-1][2] == n
    stack = []
    for lo, mid, hi, depth in nodes.tolist():
        assert lo <= mid <= hi
        kids = []
        while stack and stack[-1][0] >= lo:
            kids.append(stack.pop())
        if kids:  # internal: its two subtrees tile [lo, mid) and do not touch each other
            assert len(kids) == 2
            (l2, h2), (l1, h1) = kids
            assert l1 == lo and h1 == l2 and h2 == mid
            assert P[l1:h1][:, l2:h2].nnz == 0
        else:
            assert mid == hi
        stack.append((lo, hi))
    assert len(stack) == 1


@pytest.mark.parametrize("leaf", [64, 128, 1024])
def test_nd_host_solve_matches_reference_lu(ref, leaf):
    """The block elimination equals the reference's lu_factor + lu_solve on the
    coarsest matrices of the c2 hierarchies (n = 1,407 and 1,903)."""
    from oracle.refpy import Csr
    rng = np.random.default_rng(5)
    for a in _coarse_matrices("c2"):
        b = rng.standard_normal(a.n_rows)
        r = sdc.nd_solve_host(a, b, leaf_rows=leaf)
        _check_dissection(a, r)
        if leaf < 1024:
            assert r["depth"] >= 3 and r["stored_doubles"] < 0.35 * a.n_rows ** 2
        x_ref = ref.lu_solve(Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values), b)
        assert np.linalg.norm(r["x"] - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_nd_host_solve_edge_cases(ref):
    # nonsymmetric KAT matrix (test_krylov.cpp:75-93 generator), forced deep dissection
    a = to_sdc(ref.random_dominant(300, 0.02, 7))
    b = ref.random_vector(300, 8)
    r = sdc.nd_solve_host(a, b, leaf_rows=16)
    _check_dissection(a, r)
    assert np.allclose(sdc_spmv_host(a, r["x"]), b, rtol=0, atol=1e-11)
    # disconnected graph: block diagonal, empty separators
    d = np.zeros((40, 40))
    for k in range(4):
        blk = np.random.default_rng(k).standard_normal((10, 10)) + 10 * np.eye(10)
        d[10 * k:10 * k + 10, 10 * k:10 * k + 10] = blk
    a = sdc.SparseMatrix.from_dense(d)
    b = np.arange(40.0)
    r = sdc.nd_solve_host(a, b, leaf_rows=8)
    _check_dissection(a, r)
    assert np.allclose(d @ r["x"], b, atol=1e-11)
    # tiny and empty systems
    r = sdc.nd_solve_host(sdc.SparseMatrix.from_dense(np.array([[4.0]])), np.array([2.0]))
    assert r["x"][0] == 0.5
    r = sdc.nd_solve_host(sdc.SparseMatrix(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0)), np.zeros(0))
    assert r["x"].size == 0
    # partial pivoting inside a block: zero diagonal
    p = np.array([[0.0, 2.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 3.0]])
    r = sdc.nd_solve_host(sdc.SparseMatrix.from_dense(p), np.array([2.0, 1.0, 3.0]))
    assert np.allclose(r["x"], [1.0, 1.0, 1.0])
    # singular: like lu_factor's runtime_error (lu.cpp:142)
    with pytest.raises(RuntimeError):
        sdc.nd_solve_host(sdc.SparseMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 4.0]])), np.ones(2))


def sdc_spmv_host(a, x):
    import scipy.sparse as sp
    return sp.csr_matrix((a.values, a.col_indices, a.row_offsets), shape=(a.n_rows, a.n_cols)) @ x
