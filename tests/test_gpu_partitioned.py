"""GPU: the partitioned Dirichlet-Neumann driver (BASELINE config 5,
CouplingDriver::coupled_timestep, coupling.cpp:252-332) against the same loop
composed from the reference's own pieces on the CPU: its assemble_stokes /
assemble_darcy with interface data, its Uzawa / AMG preconditioners, its
pd_gmres / bicgstab, its traces, and the IQN-ILS update (coupling.cpp:45-101,
restated bitwise in paper_2108_13229_b200/iqn.py).  The subproblem assembly
is bitwise the reference's (tests/test_host.py); here the coupling iteration
counts must agree and the interface traces and subdomain solutions match to
1e-6."""
import numpy as np
import pytest

from paper_2108_13229_b200 import drivers, sdc
from paper_2108_13229_b200.iqn import IqnIlsHistory, iqn_ils_update

pytestmark = pytest.mark.gpu


def _cfg(n, k):
    return sdc.ScenarioConfig(cells_per_unit_square=n, permeability=k, alpha_bj=1.0, kinematic_viscosity=1.0,
                              density=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0)


def _reference_loop(ref, n, k, max_it=100):
    a_s, _ = ref.stokes(n, permeability=k, v_gamma=np.zeros(n))
    uz = ref.uzawa_stokes(a_s, n, 3)
    d, _ = ref.darcy(n, k, np.zeros(n))
    amg = ref.amg_precond(d, 3)
    v, p_k = np.zeros(n), np.zeros(n)
    hist = IqnIlsHistory()
    for it in range(max_it):
        _, b = ref.stokes(n, permeability=k, v_gamma=v)
        x, _ = ref.pd_gmres(a_s, b, 1e-10 * np.linalg.norm(b), 400, precond=uz)
        pt = ref.stokes_pressure_trace(n, 1.0, x)
        _, db = ref.darcy(n, k, pt)
        p, _ = ref.bicgstab(d, db, 1e-10 * np.linalg.norm(db), 10000, precond=amg)
        vt = ref.darcy_velocity_trace(n, k, p, pt)
        if np.linalg.norm(pt - p_k) < 1e-8 * np.linalg.norm(pt) and np.linalg.norm(vt - v) < 1e-8 * np.linalg.norm(vt):
            return it + 1, np.concatenate([x, p]), pt, vt
        res = vt - v
        if not hist.has_previous():
            v = v + 0.5 * res
            hist.record(res, vt)
        else:
            v = iqn_ils_update(hist, v, res, vt)
        p_k = pt
    raise AssertionError("reference loop did not converge")


@pytest.mark.parametrize("n,k", [(16, 1.0), (16, 1e-2), (50, 1.0)])
def test_partitioned_matches_reference_loop(ref, n, k):
    its_ref, x_ref, p_ref, v_ref = _reference_loop(ref, n, k)
    drv = drivers.PartitionedDriver(_cfg(n, k))
    out = drv.coupled_step()
    assert out.converged
    assert abs(out.coupling_iterations - its_ref) <= max(1, 0.05 * its_ref), (out.coupling_iterations, its_ref)
    assert np.linalg.norm(out.solution - x_ref) / np.linalg.norm(x_ref) <= 1e-6
    assert np.linalg.norm(drv.trace_p - p_ref) / np.linalg.norm(p_ref) <= 1e-6
    assert np.linalg.norm(drv.trace_v - v_ref) / np.linalg.norm(v_ref) <= 1e-6


def test_rhs_patch_equals_reassembly():
    cfg = _cfg(16, 1e-2)
    drv = drivers.PartitionedDriver(cfg)
    rng = np.random.default_rng(5)
    vg, pg = rng.standard_normal(16), rng.standard_normal(16)
    assert np.array_equal(drv.stokes_rhs(vg), sdc.assemble_stokes(cfg, vg)[1])
    assert np.array_equal(drv.darcy_rhs(pg), sdc.assemble_darcy(cfg, pg)[1])


def test_partitioned_agrees_with_monolithic_solution():
    """The converged partitioned solution is the monolithic one (same PDE,
    same discretisation): Stokes block and Darcy pressures within the coupling
    tolerance of the monolithic GMRES solve."""
    n = 16
    cfg = _cfg(n, 1.0)
    out = drivers.PartitionedDriver(cfg).coupled_step()
    s = sdc.assemble_monolithic(cfg)
    p = sdc.TdPreconditioner(s, "td_bgs")
    mono = sdc.pd_gmres(s.matrix, p, s.rhs, 1e-12 * np.linalg.norm(s.rhs), 400, sdc.RestartController.fixed(50))
    assert out.converged and mono.report.converged
    assert np.linalg.norm(out.solution - mono.x) / np.linalg.norm(mono.x) <= 1e-6
