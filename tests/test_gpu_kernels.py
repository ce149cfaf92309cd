"""GPU: kernel-level parity through the C-ABI against the compiled reference.

SpMV, spmv_add, Gauss-Seidel, restriction/prolongation and the Uzawa
pressure step are BITWISE kernels (same operation order, no FMA), so they
must equal the reference bit for bit.  The AMG coarse solve is a dense
inverse on the device instead of the reference's sparse LU, so V-cycles and
preconditioner applies agree to rounding (tolerances stated per test)."""
import numpy as np
import pytest

from conftest import bitwise_equal, golden_csr, rel_l2, to_sdc

from paper_2108_13229_b200 import sdc

pytestmark = pytest.mark.gpu


def test_spmv_bitwise(ref, golden):
    g = golden("dominant")
    for seed in (3, 14):
        a = golden_csr(g, f"A{seed}", 100)
        assert bitwise_equal(sdc.spmv(to_sdc(a), g[f"gs_z0_{seed}"]), g[f"spmv_{seed}"])
    s = ref.assemble(50)
    x = ref.random_vector(s.n, 5)
    A = to_sdc(s.a)
    assert bitwise_equal(sdc.spmv(A, x), ref.spmv(s.a, x))
    y = ref.random_vector(s.n, 6)
    assert bitwise_equal(sdc.spmv_add(A, x, y, -0.75), ref.spmv_add(s.a, x, y, -0.75))


def test_spmv_bitwise_full_c3_size(ref):
    """BASELINE config 3 size (1,001,000 DoF, 7.74 M nnz)."""
    cfg = sdc.ScenarioConfig(cells_per_unit_square=500, permeability=1e-2, alpha_bj=1.0,
                             kinematic_viscosity=1.0, density=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0)
    s = sdc.assemble_monolithic(cfg)
    assert s.n_total() == 1001000 and s.matrix.nnz() == 7742002
    from oracle.refpy import Csr
    a = Csr(s.n_total(), s.n_total(), s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values)
    x = ref.random_vector(s.n_total(), 11)
    assert bitwise_equal(sdc.spmv(s.matrix, x), ref.spmv(a, x))


def test_spmv_edge_cases():
    e = sdc.SparseMatrix(3, 3, [0, 0, 0, 0])  # all rows empty
    assert np.array_equal(sdc.spmv(e, np.ones(3)), np.zeros(3))
    ident = sdc.SparseMatrix.identity(4)
    assert np.array_equal(sdc.spmv(ident, [1.0, 2, 3, 4]), [1.0, 2, 3, 4])
    rect = sdc.SparseMatrix.from_dense([[1.0, 2.0, 0.0], [0.0, 0.0, 3.0]])
    assert np.array_equal(sdc.spmv(rect, [1.0, 1.0, 1.0]), [3.0, 3.0])
    with pytest.raises(ValueError):
        sdc.spmv(rect, [1.0, 1.0])


def test_gs_bitwise(ref, golden):
    g = golden("dominant")
    for seed in (3, 14):
        a = to_sdc(golden_csr(g, f"A{seed}", 100))
        z0, b = g[f"gs_z0_{seed}"], g[f"b{seed}"]
        assert bitwise_equal(sdc.sor_sweep(a, z0, b, 1.0), g[f"gs_z1_{seed}"])
        assert bitwise_equal(sdc.sor_sweep(a, z0, b, 0.7), g[f"gs_z1w_{seed}"])
    # the velocity block of the coupled system (structured, 2D wavefronts)
    s = ref.assemble(50)
    A = to_sdc(s.a)
    V = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
    from oracle.refpy import Csr
    Vr = Csr(V.n_rows, V.n_cols, V.row_offsets, V.col_indices, V.values)
    z0 = ref.random_vector(V.n_rows, 1)
    r = ref.random_vector(V.n_rows, 2)
    assert bitwise_equal(sdc.sor_sweep(V, z0, r, 1.0), ref.sor_sweep(Vr, z0, r, 1.0))


def test_gs_hand_computation_and_errors():
    # test_precond.cpp:83-101
    a = sdc.SparseMatrix.from_dense([[2.0, 1.0], [1.0, 2.0]])
    z = sdc.gauss_seidel_apply(a, [1.0, 1.0])
    assert z[0] == 0.5 and z[1] == 0.25
    assert np.array_equal(sdc.gauss_seidel_apply(a, [1.0, 1.0], 1.0, 0), [0.0, 0.0])
    bad = sdc.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 1.0]])
    with pytest.raises(RuntimeError, match="zero diagonal in row 0"):
        sdc.sor_sweep(bad, np.zeros(2), np.ones(2), 1.0)


def test_amg_vcycle_matches_reference(ref, golden):
    g = golden("dominant")
    for seed in (3, 14):
        a = golden_csr(g, f"A{seed}", 100)
        amg = sdc.AmgPreconditioner(to_sdc(a), sdc.AmgOptions(coarse_threshold=10))
        assert len(amg.hierarchy()) == int(g[f"vcyc_levels_{seed}"])
        z = amg.apply(g[f"b{seed}"])
        assert rel_l2(z, g[f"vcyc_{seed}"]) < 1e-13


def test_amg_single_level_is_exact(ref):
    # test_precond.cpp:103-111
    a = ref.random_dominant(30, 0.2, 5)
    A = to_sdc(a)
    amg = sdc.AmgPreconditioner(A)
    assert len(amg.hierarchy()) == 1
    r = ref.random_vector(30, 6)
    assert np.allclose(sdc.spmv(A, amg.apply(r)), r, rtol=1e-11, atol=1e-12)


def test_amg_on_system_blocks(ref):
    s = ref.assemble(50)
    td = ref.td(s)
    A = to_sdc(s.a)
    V = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
    amg = sdc.AmgPreconditioner(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u)))
    assert [r for r, _ in amg.hierarchy()] == [lv.a.n_rows for lv in td.v_hierarchy.levels()]
    r = ref.random_vector(s.n_vel, 8)
    assert rel_l2(amg.apply(r), td.v_hierarchy.vcycle(r)) < 1e-11


@pytest.mark.parametrize("mode", [{"SDG_GS_SPLIT": "1"}, {"SDG_GS_PIPE": "1"}, {"SDG_GS_WALK": "0"},
                                  {"SDG_GS_BANDS": "4"}, {"SDG_GS_MERGE": "1"}, {"SDG_GS_MERGE": "2"},
                                  {"SDG_GS_MERGE": "4"}, {"SDG_GS_MERGE": "4", "SDG_GS_MERGE_CAP": "8"},
                                  {"SDG_TD_SPLIT": "0"}, {"SDG_SELL": "0"}, {"SDG_WALK_ROLES": "0"},
                                  {"SDG_TD_EARLY": "0"}, {"SDG_GS_WAVE": "0"}],
                         ids=["label-block-walks", "2-cta-pipe", "cluster-kernel", "cluster-4-bands", "no-merge",
                              "merge-2", "merge-4", "merge-dynamic", "no-interface-split", "csr-spmv", "no-walk-roles",
                              "late-interface-gemv", "no-wave"])
def test_smoother_paths_match_reference(ref, golden, monkeypatch, mode):
    """The other lower-solve plans (one walk per u/v block with a coupling
    step; the u/v blocks walked concurrently on a 2-CTA cluster; the banded
    cluster kernel) against the reference V-cycle and the golden td_bgs
    apply."""
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    s = ref.assemble(50)
    td = ref.td(s)
    A = to_sdc(s.a)
    V = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
    amg = sdc.AmgPreconditioner(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u)))
    r = ref.random_vector(s.n_vel, 8)
    assert rel_l2(amg.apply(r), td.v_hierarchy.vcycle(r)) < 1e-11
    g = golden("system_c1")
    n = int(g["n_total"])
    system = sdc.CoupledSystem(to_sdc(golden_csr(g, "A", n)), g["rhs"], int(g["n"]), int(g["n_u"]),
                               int(g["n_vel"]), int(g["n_pff"]), int(g["n_ppm"]))
    p = sdc.TdPreconditioner(system, "td_bgs", omega_override=float(g["omega"]))
    assert rel_l2(p.apply(g["apply_r"]), g["apply_z"]) < 1e-10


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3"])
def test_wave_smoother_bitwise_vs_walks(monkeypatch, cfg_name):
    """The multi-SM wavefront lower solve (gs_wave.cu, the default on the
    structured finest levels) does every row's arithmetic in the order of the
    level walks: the velocity AMG V-cycle equals the one with label-block
    walks on its finest level (u block, coupling step, v block) bit for bit,
    and the porous one equals the plain finest walk.  c1 runs 2 bands, c2 6,
    c3 16 (one CTA each), so the cross-band flag hand-off is exercised; two
    applies in a row check the epoch-tagged flags."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    rng = np.random.default_rng(3)
    for mat, opts, knobs, feat in (
            (V, sdc.AmgOptions(components=comps, max_levels=cfg.v_max_levels),
             {"SDG_GS_WAVE": "0", "SDG_GS_SPLIT": "1"}, "wave_v"),
            (D, sdc.AmgOptions(max_levels=cfg.d_max_levels), {"SDG_GS_WAVE": "0", "SDG_GS_MERGE": "1"}, "wave_v")):
        r = [rng.standard_normal(mat.n_rows) for _ in range(2)]
        monkeypatch.delenv("SDG_GS_KNOB_ROWS", raising=False)
        wave = sdc.AmgPreconditioner(mat, opts)
        assert feat in wave.features()
        zw = [wave.apply(x) for x in r] + [wave.apply(r[0])]
        del wave
        monkeypatch.setenv("SDG_GS_KNOB_ROWS", str(mat.n_rows))  # the knobs act on the finest level only
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        walk = sdc.AmgPreconditioner(mat, opts)
        assert feat not in walk.features()
        zk = [walk.apply(x) for x in r]
        for k in knobs:
            monkeypatch.delenv(k)
        assert np.array_equal(zw[0], zk[0]) and np.array_equal(zw[1], zk[1])
        assert np.array_equal(zw[2], zw[0])


@pytest.mark.parametrize("wave_w", ["1", "2", "4"])
def test_wave_bands_per_cta_bitwise(monkeypatch, wave_w):
    """The wavefront with 1, 2 or 4 bands per CTA (SDG_WAVE_W; the hand-off
    between two bands of one CTA goes through shared memory, between CTAs
    through L2) gives the same bits: velocity and porous V-cycles at c2
    (6 bands) against the default plan."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS["c2"]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    rng = np.random.default_rng(5)
    for mat, opts in ((V, sdc.AmgOptions(components=comps, max_levels=cfg.v_max_levels)),
                      (D, sdc.AmgOptions(max_levels=cfg.d_max_levels))):
        r = rng.standard_normal(mat.n_rows)
        monkeypatch.delenv("SDG_WAVE_W", raising=False)
        base = sdc.AmgPreconditioner(mat, opts)
        assert "wave_v" in base.features()
        z0 = [base.apply(r), base.apply(r)]
        del base
        monkeypatch.setenv("SDG_WAVE_W", wave_w)
        alt = sdc.AmgPreconditioner(mat, opts)
        z1 = [alt.apply(r), alt.apply(r)]
        assert np.array_equal(z0[0], z1[0]) and np.array_equal(z0[1], z1[1]) and np.array_equal(z0[0], z0[1])


@pytest.mark.parametrize("cfg_name", ["c1", "c2"])
def test_wave_mac_split_bitwise_vs_fused(monkeypatch, cfg_name):
    """The MAC wavefront with the u and v recurrences on two warps per band
    (k_gs_wave_mac, the default) against the same sweep on one warp
    (SDG_WAVE_SPLIT=0): the velocity V-cycle gives the same bits, with one and
    with two bands per CTA, and repeated applies are bitwise reproducible."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    opts = sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u), max_levels=cfg.v_max_levels)
    rng = np.random.default_rng(11)
    r = [rng.standard_normal(V.n_rows) for _ in range(2)]
    monkeypatch.setenv("SDG_WAVE_SPLIT", "0")
    fused = sdc.AmgPreconditioner(V, opts)
    assert "wave_v" in fused.features()
    z0 = [fused.apply(x) for x in r]
    del fused
    for w in ("1", "2"):
        monkeypatch.setenv("SDG_WAVE_SPLIT", "1")
        monkeypatch.setenv("SDG_WAVE_W", w)
        split = sdc.AmgPreconditioner(V, opts)
        assert "wave_v" in split.features()
        z1 = [split.apply(x) for x in r] + [split.apply(r[0])]
        del split
        assert np.array_equal(z0[0], z1[0]) and np.array_equal(z0[1], z1[1]) and np.array_equal(z1[0], z1[2])


@pytest.mark.parametrize("cfg_name", ["c3"])
def test_lattice_smoother_matches_walks(monkeypatch, cfg_name):
    """The multi-SM lattice lower solve (gs_lattice.cu, opt-in SDG_GS_LATTICE=1)
    on the first coarse level: the velocity AMG V-cycle (lattice on both label
    blocks of level 1) and the porous one agree with the plain level-1 walks to
    rounding (the lattice sums a row in a fixed source order, the walk in
    column order); two applies in a row are bitwise equal."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    rng = np.random.default_rng(4)
    for mat, opts, knobs in (
            (V, sdc.AmgOptions(components=comps, max_levels=cfg.v_max_levels), {"SDG_GS_LATTICE": "0"}),
            (D, sdc.AmgOptions(max_levels=cfg.d_max_levels), {"SDG_GS_LATTICE": "0", "SDG_GS_MERGE": "1"})):
        r = [rng.standard_normal(mat.n_rows) for _ in range(2)]
        monkeypatch.delenv("SDG_GS_KNOB_ROWS", raising=False)
        monkeypatch.setenv("SDG_GS_LATTICE", "1")  # opt-in
        lat = sdc.AmgPreconditioner(mat, opts)
        assert "lattice_v" in lat.features()
        zl = [lat.apply(x) for x in r] + [lat.apply(r[0])]
        n1 = lat.hierarchy()[1][0]
        del lat
        monkeypatch.setenv("SDG_GS_KNOB_ROWS", str(n1))  # the knobs act on level 1 only
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        walk = sdc.AmgPreconditioner(mat, opts)
        assert "lattice_v" not in walk.features()
        zk = [walk.apply(x) for x in r]
        for k in knobs:
            monkeypatch.delenv(k)
        assert rel_l2(zl[0], zk[0]) < 1e-12 and rel_l2(zl[1], zk[1]) < 1e-12
        assert np.array_equal(zl[2], zl[0])


@pytest.mark.parametrize("cfg_name,lat_w", [("c1", None), ("c2", None), ("c3", None), ("c3", "1"), ("c3", "3"),
                                             ("c3", "4")])
def test_lattice_kernel_bitwise_vs_emulation(monkeypatch, cfg_name, lat_w):
    """k_gs_lattice on the device equals its host emulation (same records,
    registers, windows, boundary buffer) bit for bit on every label block /
    level of the config that is a lattice, also when replayed (the boundary
    buffer's parities), for every number of bands per CTA (SDG_LAT_W: the
    hand-off inside a CTA goes through shared memory, between CTAs through L2)."""
    import ctypes as C
    if lat_w is not None:
        monkeypatch.setenv("SDG_LAT_W", lat_w)
    import scipy.sparse as sp
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    L = sdc.lib()
    ctx = sdc.default_context()

    def sub(A, lo, hi):
        m = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n_rows, A.n_rows))[lo:hi, lo:hi].tocsr()
        m.sort_indices()
        return sdc.SparseMatrix(hi - lo, hi - lo, m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data)

    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    hv = sdc.host_hierarchy(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u),
                                              max_levels=cfg.v_max_levels))
    nu1 = int(hv[0].aggregate_of[: s.n_u].max()) + 1
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    hd = sdc.host_hierarchy(D, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    checked = 0
    for A in (sub(V, 0, s.n_u), sub(hv[1].a, 0, nu1), sub(hv[1].a, nu1, hv[1].a.n_rows), D, hd[1].a):
        n = A.n_rows
        b = np.random.default_rng(n).standard_normal(n)
        zh, zd = np.zeros(n), np.zeros(n)
        P = C.c_void_p
        rp, ci, v = (np.ascontiguousarray(A.row_offsets, np.int32), np.ascontiguousarray(A.col_indices, np.int32),
                     np.ascontiguousarray(A.values))
        rc = L.sdg_debug_lattice_sweep(ctx.h, n, rp.ctypes.data_as(P), ci.ctypes.data_as(P), v.ctypes.data_as(P),
                                       b.ctypes.data_as(P), zh.ctypes.data_as(P), zd.ctypes.data_as(P), 3)
        if rc != 0:
            continue  # not a lattice
        checked += 1
        assert np.array_equal(zh, zd), (cfg_name, n)
    assert checked >= 2


def test_c2_merge_and_interface_split_agree(monkeypatch):
    """The c2 bench system: the td_bgs apply with the interface split and the
    merged walks (defaults) against the plain sequential apply with unmerged
    walks, and merged AMG V-cycles against the bitwise Gauss-Seidel path."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS["c2"]
    s = scenarios.build_system(cfg)
    r = np.random.default_rng(7).standard_normal(s.n_total())
    fast = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
    z_fast = fast.apply(r)
    monkeypatch.setenv("SDG_TD_SPLIT", "0")
    monkeypatch.setenv("SDG_GS_MERGE", "1")
    plain = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, omega_override=fast.omega())
    assert rel_l2(z_fast, plain.apply(r)) < 1e-11
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    x = r[: D.n_rows]
    monkeypatch.setenv("SDG_GS_MERGE", "4")
    merged = sdc.AmgPreconditioner(D, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    monkeypatch.setenv("SDG_GS_EXACT", "1")
    exact = sdc.AmgPreconditioner(D, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    assert rel_l2(merged.apply(x), exact.apply(x)) < 1e-11


@pytest.mark.parametrize("cfg_name", ["c2", "c2u"])
def test_c2_td_bgs_apply_matches_reference(ref, cfg_name):
    """The td_bgs apply at the c2 size against the compiled reference's own
    apply on the same matrix (its amg_setup, lu_factor, power iteration): the
    default GPU plan (wavefront, merged walks, interface split with early
    correction, dense Gauss-Jordan coarse inverse) agrees to 1e-9, omega to
    2e-3 (the power iteration stops at 1e-3)."""
    from oracle.refpy import Csr, System
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    n = s.n_total()
    rs = System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm,
                Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values), s.rhs)
    rtd = ref.td(rs, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
    # same omega on both sides: the apply is compared, not the eigenvalue estimate
    p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, omega_override=rtd.omega)
    assert abs(sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels).omega() - rtd.omega) <= \
        2e-3 * abs(rtd.omega)
    for seed in (17, 18):
        r = ref.random_vector(n, seed)
        assert rel_l2(p.apply(r), rtd.apply(r)) < 1e-9


def test_c2_walk_roles_bitwise(monkeypatch):
    """Walks with the small and wide rows on separate warps (the default)
    compute every row with the same instructions as the shared-warp walk: the
    c2 td_bgs apply is bitwise equal."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS["c2"]
    s = scenarios.build_system(cfg)
    r = np.random.default_rng(11).standard_normal(s.n_total())
    z_roles = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels).apply(r)
    monkeypatch.setenv("SDG_WALK_ROLES", "0")
    z_plain = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels).apply(r)
    assert np.array_equal(z_roles, z_plain)


@pytest.mark.parametrize("split", ["0", "1"], ids=["v0-wave", "label-block-walks"])
def test_c2_early_interface_correction_bitwise(monkeypatch, split):
    """td_bgs with the interface GEMV started on the side stream from the
    Uzawa post-smoother's mark (SDG_TD_EARLY=1) against the GEMV after the join:
    bitwise equal, for the V0 wavefront and for label-block walks."""
    from paper_2108_13229_b200 import scenarios
    monkeypatch.setenv("SDG_GS_SPLIT", split)
    cfg = scenarios.CONFIGS["c2"]
    s = scenarios.build_system(cfg)
    r = np.random.default_rng(5).standard_normal(s.n_total())
    monkeypatch.setenv("SDG_TD_EARLY", "1")  # unset, the faster of early and late is timed at setup
    early = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
    assert {"split", "early"} <= early.features()
    assert ("wave_v" in early.features()) == (split == "0")
    z_early = [early.apply(r), early.apply(2.0 * r)]
    monkeypatch.setenv("SDG_TD_EARLY", "0")
    late = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, omega_override=early.omega())
    assert "early" not in late.features() and "split" in late.features()
    z_late = [late.apply(r), late.apply(2.0 * r)]
    assert all(np.array_equal(a, b) for a, b in zip(z_early, z_late))


def check_linear(p, seed, n, tol=1e-13):
    # test_precond.cpp:33-47
    rng = np.random.default_rng(seed)
    r, s_ = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    a, b = 0.731, -1.44
    zr, zs, zc = p.apply(r), p.apply(s_), p.apply(a * r + b * s_)
    assert np.max(np.abs(zc - a * zr - b * zs)) <= tol * (np.linalg.norm(zc) + 1e-30)


@pytest.mark.parametrize("name", ["system_n6", "system_n16", "system_c1"])
def test_td_bgs_apply_matches_reference(golden, name):
    g = golden(name)
    n = int(g["n_total"])
    A = to_sdc(golden_csr(g, "A", n))
    system = sdc.CoupledSystem(A, g["rhs"], int(g["n"]), int(g["n_u"]), int(g["n_vel"]), int(g["n_pff"]),
                               int(g["n_ppm"]))
    p = sdc.TdPreconditioner(system, "td_bgs", omega_override=float(g["omega"]))
    assert rel_l2(p.apply(g["apply_r"]), g["apply_z"]) < 1e-10
    check_linear(p, 500, n, tol=1e-12)
    assert np.array_equal(p.apply(np.zeros(n)), np.zeros(n))
    # omega from the device power iteration: within the 1e-3 estimator tolerance
    q = sdc.TdPreconditioner(system, "td_bgs")
    assert abs(q.omega() - float(g["omega"])) <= 2e-3 * abs(float(g["omega"]))


def test_block_kinds_and_uzawa_toy(ref):
    # test_precond.cpp:190-209 restated with an AMG inner solve (V = I, single level)
    v = sdc.SparseMatrix.identity(2)
    b = sdc.SparseMatrix.from_dense([[1.0], [-1.0]])
    c = sdc.SparseMatrix.from_dense([[1.0, -1.0]])
    uz = sdc.UzawaPreconditioner(v, b, c)
    assert abs(uz.omega() - 0.5) < 1e-10
    z = uz.apply([1.0, 2.0, 3.0])
    assert np.allclose(z, [1.0, 2.0, 0.5 * ((1.0 - 2.0) - 3.0)], rtol=1e-12)
    with pytest.raises(ValueError, match="inconsistent block dimensions"):
        sdc.UzawaPreconditioner(v, c, c)
    # identity subs: pv_bj is the identity, every kind maps zero to zero (test_precond.cpp:267-301)
    s = ref.assemble(6)
    A = to_sdc(s.a)
    idv, idff, idpm = (sdc.IdentityPreconditioner(k) for k in (s.n_vel, s.n_ff, s.n_ppm))
    r = ref.random_vector(s.n, 77)
    pv = sdc.BlockPreconditioner(sdc.BlockPrecondKind.pv_bj, A, s.n_vel, s.n_pff, s.n_ppm, idv, idpm)
    assert np.array_equal(pv.apply(r), r)
    for kind in (sdc.BlockPrecondKind.td_bj, sdc.BlockPrecondKind.td_bgs):
        p = sdc.BlockPreconditioner(kind, A, s.n_vel, s.n_pff, s.n_ppm, idff, idpm)
        assert np.array_equal(p.apply(np.zeros(s.n)), np.zeros(s.n))
    with pytest.raises(ValueError, match="first sub-block size mismatch"):
        sdc.BlockPreconditioner(sdc.BlockPrecondKind.pv_bj, A, s.n_vel, s.n_pff, s.n_ppm,
                                sdc.IdentityPreconditioner(s.n_vel + 1), idpm)
    # td_bgs with identity subs: z_pm = r_pm - C' r_ff exactly (bitwise spmv_add)
    p = sdc.BlockPreconditioner(sdc.BlockPrecondKind.td_bgs, A, s.n_vel, s.n_pff, s.n_ppm, idff, idpm)
    z = p.apply(r)
    Cp = sdc.submatrix(A, s.n_ff, s.n, 0, s.n_ff)
    assert np.array_equal(z[: s.n_ff], r[: s.n_ff])
    from oracle.refpy import Csr
    assert bitwise_equal(z[s.n_ff:], ref.spmv_add(Csr(Cp.n_rows, Cp.n_cols, Cp.row_offsets, Cp.col_indices,
                                                          Cp.values), r[: s.n_ff], r[s.n_ff:], -1.0))


def test_applications_counter_and_determinism(golden):
    g = golden("system_n16")
    n = int(g["n_total"])
    A = to_sdc(golden_csr(g, "A", n))
    system = sdc.CoupledSystem(A, g["rhs"], int(g["n"]), int(g["n_u"]), int(g["n_vel"]), int(g["n_pff"]),
                               int(g["n_ppm"]))
    p = sdc.TdPreconditioner(system, "td_bgs")
    z1 = p.apply(g["apply_r"])
    z2 = p.apply(g["apply_r"])
    assert np.array_equal(z1, z2)
    assert p.applications() == 2


def test_ilu0_matches_reference(ref):
    """Ilu0Preconditioner (precond.cpp:13-87): the reference's factors restated
    on the host (setup.cpp ilu0_factor), the two triangular solves on the device
    (the 5-point porous block runs both on the wavefront, the unstructured KAT
    matrix on level walks); applies agree with the reference's to rounding."""
    from oracle.refpy import Csr
    s = ref.assemble(50)
    D = ref.ground_dof(Csr(s.n_ppm, s.n_ppm, *_sub(s.a, s.n_ff, s.n, s.n_ff, s.n)))
    for a in (D, ref.random_dominant(400, 0.02, 3)):
        p_ref = ref.ilu0(a)
        p = sdc.Ilu0Preconditioner(to_sdc(a))
        for seed in (1, 2):
            r = ref.random_vector(a.n_rows, seed)
            assert rel_l2(p.apply(r), ref.precond_apply(p_ref, r)) < 1e-12
    assert "wave_v" not in p.features()


def _sub(a, r0, r1, c0, c1):
    import scipy.sparse as sp
    m = sp.csr_matrix((a.val, a.col, a.rowptr), shape=(a.n_rows, a.n_cols))[r0:r1, c0:c1].tocsr()
    m.sort_indices()
    return m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data


# ---------------------------------------------------------------------------
# coarse direct solve on the device (csrc/coarse.cu; lu_factor / lu_solve, lu.cpp:91-203)

def _coarse_level(cfg_name, which):
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    if which == "V":
        m = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
        o = sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u), max_levels=cfg.v_max_levels)
    else:
        m = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
        o = sdc.AmgOptions(max_levels=cfg.d_max_levels)
    return sdc.host_hierarchy(m, o)[-1].a


def _host_spmv(a, x):
    import scipy.sparse as sp
    return sp.csr_matrix((a.values, a.col_indices, a.row_offsets), shape=(a.n_rows, a.n_cols)) @ x


@pytest.mark.parametrize("mode", [{"SDG_COARSE": "dense"}, {"SDG_COARSE": "nd", "SDG_ND_LEAF": "128"},
                                  {"SDG_COARSE": "nd", "SDG_ND_LEAF": "40"}], ids=["dense", "nd128", "nd40"])
def test_lu_solve_matches_reference(ref, monkeypatch, mode):
    """Device direct solve (dense Gauss-Jordan inverse, and the nested-dissection
    block elimination at two leaf sizes) against the reference's lu_factor +
    lu_solve on the coarsest matrices of the c2 hierarchies, and bitwise against
    a second solve (deterministic)."""
    from oracle.refpy import Csr
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    for which in ("V", "D"):
        a = _coarse_level("c2", which)
        f = sdc.lu_factor(a)
        info = f.info()
        assert info["dense"] == (mode["SDG_COARSE"] == "dense")
        if not info["dense"]:
            assert info["depth"] >= 3 and info["stored_doubles"] < 0.4 * a.n_rows ** 2
        b = rng.standard_normal(a.n_rows)
        x = f.solve(b)
        x_ref = ref.lu_solve(Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values), b)
        assert rel_l2(x, x_ref) < 1e-10
        assert bitwise_equal(x, f.solve(b))


def test_lu_solve_c3_coarse_levels_residual():
    """Default policy at c3 (V: 12,246 rows, D: 4,704 rows -> nested dissection):
    the residual of the device solve is at rounding level."""
    rng = np.random.default_rng(12)
    for which in ("V", "D"):
        a = _coarse_level("c3", which)
        f = sdc.lu_factor(a)
        info = f.info()
        assert not info["dense"] and info["stored_doubles"] < 0.2 * a.n_rows ** 2
        b = rng.standard_normal(a.n_rows)
        x = f.solve(b)
        assert np.linalg.norm(_host_spmv(a, x) - b) <= 1e-11 * np.linalg.norm(b) * max(1.0, np.abs(x).max())
        xh = sdc.nd_solve_host(a, b)["x"] if which == "D" else None
        if xh is not None:  # same algebra on the host (different rounding: FMA, reduction trees)
            assert rel_l2(x, xh) < 1e-10


def test_lu_factor_pivoting_and_errors(ref):
    # needs row exchanges: zero diagonal
    p = np.array([[0.0, 2.0, 0.0, 0.0], [1.0, 0.0, 0.0, 3.0], [0.0, 0.0, 0.0, 1.0], [0.0, 1.0, 5.0, 0.0]])
    f = sdc.lu_factor(sdc.SparseMatrix.from_dense(p))
    b = np.array([1.0, 2.0, 3.0, 4.0])
    assert np.allclose(p @ f.solve(b), b, atol=1e-13)
    # nonsymmetric KAT matrix (test_krylov.cpp:75-93 generator)
    a = ref.random_dominant(200, 0.05, 3)
    r = ref.random_vector(200, 4)
    x = sdc.lu_solve(sdc.lu_factor(to_sdc(a)), r)
    assert rel_l2(x, ref.lu_solve(a, r)) < 1e-12
    with pytest.raises(RuntimeError):  # lu.cpp:142
        sdc.lu_factor(sdc.SparseMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 4.0]])))
    with pytest.raises(ValueError):
        sdc.lu_factor(sdc.SparseMatrix.from_dense(np.ones((2, 3))))
    assert sdc.lu_factor(sdc.SparseMatrix(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0))).solve(
        np.zeros(0)).size == 0


def test_forced_nd_singular_block_falls_back_to_dense(monkeypatch):
    """An indefinite but regular matrix whose diagonal blocks are singular: the
    dissection's blocks cannot be inverted, the whole-matrix pivoting can."""
    monkeypatch.setenv("SDG_COARSE", "nd")
    monkeypatch.setenv("SDG_ND_LEAF", "32")
    n = 120
    d = np.zeros((n, n))
    for i in range(n):  # a chain of 2-cycles: zero diagonal everywhere
        j = i + 1 if i % 2 == 0 else i - 1
        d[i, j] = 2.0 + i
        if i + 2 < n:
            d[i, i + 2] = 0.5
    f = sdc.lu_factor(sdc.SparseMatrix.from_dense(d))
    b = np.arange(1.0, n + 1)
    assert np.allclose(d @ f.solve(b), b, atol=1e-9)


@pytest.mark.parametrize("cfg_name", ["c1", "c2"])
def test_galerkin_device_bitwise(cfg_name):
    """galerkin_product on the device (csrc/galerkin.cu) equals the host product
    -- itself bitwise the reference's CooBuilder order (tests/test_host.py) --
    on every level of both hierarchies, and the device AMG setup (which uses
    it) builds the same hierarchy as the host-only setup."""
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[cfg_name]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    for m, o in ((V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u), max_levels=cfg.v_max_levels)),
                 (D, sdc.AmgOptions(max_levels=cfg.d_max_levels))):
        h = sdc.host_hierarchy(m, o)
        assert len(h) >= 2
        for lev in range(len(h) - 1):
            c = sdc.galerkin_product_device(h[lev].a, h[lev].aggregate_of, h[lev].n_coarse)
            ref_c = h[lev + 1].a
            assert np.array_equal(c.row_offsets, ref_c.row_offsets) and np.array_equal(c.col_indices, ref_c.col_indices)
            assert bitwise_equal(c.values, ref_c.values)
        amg = sdc.AmgPreconditioner(m, o)
        assert [r for r, _ in amg.hierarchy()] == [lv.a.n_rows for lv in h]
        assert [z for _, z in amg.hierarchy()] == [lv.a.nnz() for lv in h]
