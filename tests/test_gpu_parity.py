"""GPU parity: the CUDA path (through the C ABI, paper_1905_02300_b200.Shell)
against the CPU oracle on the same seeded inputs, element by element.

Bar (BASELINE.json north_star): max relative error <= 1e-11 per step and
identical Schwarz iteration counts; the relative error is taken two ways (see
_relerr: the RD-E3 vector-norm metric, and BASELINE.md's per-field metric for
every field that is not negligible within its vector).  Sizes span several 128-wide thread blocks with ragged
tails; full BASELINE sizes are covered in test_gpu_fullsize.py."""
import numpy as np
import pytest

import workloads as W
from oracle.scheme import Oracle

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-11
# BASELINE.md §2's literal per-field metric on the fields that are not negligible
# within their vector (>= 1e-3 of its norm): FMA / reciprocal rounding in small
# components relative to their own norm stays within 10x the per-step bar (the
# measured maxima per test are written to gpurun_out/parity_per_field.json)
TOL_FIELD = 1e-10


def _shell(cfg, **kw):
    from paper_1905_02300_b200 import Shell
    return Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, **kw)


def _oracle(cfg, **kw):
    return Oracle(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt, **kw)


PER_FIELD = {}   # worst BASELINE.md per-field metric seen per test (reported by conftest)


def _relerr(sh, o):
    """Two parity metrics over patches, systems, levels and fields:

    * RD-E3 (asserted <= 1e-11 per step): ||gpu - oracle||_inf / ||oracle||_inf
      where the three velocity components of one system and level share the
      norm of their vector (max over u_r, u_th, u_ph) — DESIGN.md 'Parity
      metric': a nearly-zero component (C3's u_th is ~1e-2 of u_r early on)
      otherwise measures rounding of that near-zero field, not parity;
    * BASELINE.md §2 per field: the same with every field's own norm; recorded
      (PER_FIELD) and asserted <= TOL_FIELD for every field whose norm is at
      least 1e-3 of its vector's.
    Returns (RD-E3 worst, where, per-field worst over the asserted fields)."""
    worst = 0.0
    where = None
    pf = 0.0
    for p in range(2):
        for s in (1, 2):
            for lev in (0, 1):
                a = sh.get_fields(p, lev, s)
                b = o.get_fields(p, lev, s)
                vmax = max(np.max(np.abs(b[q])) for q in ("ur", "ut", "up"))
                for k in a:
                    own = float(np.max(np.abs(b[k])))
                    den = vmax if k in ("ur", "ut", "up") else own
                    den = max(den, 1e-300)
                    d = float(np.max(np.abs(a[k] - b[k])))
                    e = d / den
                    if e > worst:
                        worst, where = e, (p, s, lev, k)
                    if own >= 1e-3 * den:
                        pf = max(pf, d / max(own, 1e-300))
    return worst, where, pf


def _pair(cfg, steps, wl=None, tol=None, oracle_kw=None, shell_kw=None):
    wl = wl if wl is not None else W.make_workload(cfg)
    tol = cfg.tol if tol is None else tol
    sh = _shell(cfg, **(shell_kw or {}))
    sh.load_workload(wl)
    o = _oracle(cfg, **(oracle_kw or {}))
    o.load_workload(wl)
    errs = []
    import os
    name = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    for _ in range(steps):
        sh.step(1, tol)
        o.step(1, tol)
        e, where, pf = _relerr(sh, o)
        errs.append(e)
        PER_FIELD[name] = max(PER_FIELD.get(name, 0.0), pf)
        assert e <= TOL_STEP, (e, where)
        assert pf <= TOL_FIELD, pf
        assert sh.stats()[-1][0] == o.stats[-1][0], (sh.stats(), o.stats)
    return sh, o, errs


def test_c1_manufactured_three_steps():
    _pair(W.config("C1"), 3)


def test_ragged_random_state():
    # odd sizes: ragged 128-wide blocks in every launch; noisy levels so every
    # stencil weight and fringe value matters
    cfg = W.small("C1", 7, 13, 37, Ra=30.0, dt=2e-3)
    _pair(cfg, 2, wl=W.random_state(cfg, seed=11, amp=5.0))


def test_convection_reduced():
    cfg = W.small("C3", 10, 18, 50)
    _pair(cfg, 2)


def test_landau_reduced():
    cfg = W.small("C2", 8, 16, 45)
    _pair(cfg, 2)


def test_wide_phi_rows():
    # nphi - 2 = 129 unknowns per phi-line: two blocks in x, one nearly empty
    cfg = W.small("C1", 3, 10, 131, dt=1e-3)
    _pair(cfg, 1)


@pytest.mark.parametrize("nph", [450, 1100])
def test_long_phi_lines_multiwarp(nph):
    # phi lines longer than 384 rows are solved by 4 warps per line (segment
    # solves with symbolic couplings + the per-line 8-unknown boundary system):
    # every factor position (first / plain / final) of every quantity
    cfg = W.small("C1", 3, 10, nph, Ra=30.0, dt=1e-3)
    _pair(cfg, 1, wl=W.random_state(cfg, seed=5, amp=2.0))


def test_fixed_iterations_mode():
    cfg = W.small("C1", 5, 12, 30, dt=1e-3)
    _pair(cfg, 2, oracle_kw={"fixed_iters": 3}, shell_kw={"fixed_iters": 3})


def test_static_rhs_parity():
    # O2/O3 stage alone: a* and the seven G_q arrays of the first step
    cfg = W.small("C1", 6, 14, 33, Ra=50.0, dt=2e-3)
    wl = W.random_state(cfg, seed=3, amp=3.0)
    sh = _shell(cfg, fixed_iters=1)
    sh.load_workload(wl)
    sh.step(1, 1e-10)
    o = _oracle(cfg)
    o.load_workload(wl)
    for p in range(2):
        astar, G = o.static(p, 0.0)
        for name, ref in zip(("astar_r", "astar_t", "astar_p"), astar):
            assert np.max(np.abs(sh.debug_get(name, p) - ref)) <= 1e-14 * np.max(np.abs(ref))
        for q in ("T", "ur1", "ut1", "up1", "ur2", "ut2", "up2"):
            kind = {"T": "C", "u": None}.get(q[0]) or {"r": "R", "t": "TH", "p": "PH"}[q[1]]
            m = o.g.solved_mask(kind)
            a = sh.debug_get("G_" + q, p)[m]
            b = G[q][m]
            assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b)), q


def test_deterministic_bitwise():
    cfg = W.small("C1", 5, 12, 30, dt=1e-3)
    wl = W.random_state(cfg, seed=5)
    out = []
    for _ in range(2):
        sh = _shell(cfg)
        sh.load_workload(wl)
        sh.step(2, 1e-10)
        out.append([sh.get_fields(p, 0, 2) for p in range(2)])
        st = sh.stats()
    for p in range(2):
        for k in out[0][p]:
            assert np.array_equal(out[0][p][k], out[1][p][k])


def test_line_solve_c4_reduced():
    import torch
    from oracle import ops
    nr, nt, npp = 9, 21, 67
    a, rhs = W.c4_inputs(nr, nt, npp)
    cfg = W.Config("C4", nr, nt, npp, dt=1e-4)
    sh = _shell(cfg)
    o = _oracle(cfg)
    astar = [a["ur"], a["ut"], a["up"]]
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    for axis in range(3):
        x = dev(rhs)
        sh.line_solve(axis, dev(a["ur"]), dev(a["ut"]), dev(a["up"]), x)
        torch.cuda.synchronize()
        got = x.cpu().numpy()
        ref = o.sweep("T", rhs, axis, ops.coeffs(o.g, o.prm, "T", axis, True, astar))
        m = o.g.solved_mask("C")
        assert np.max(np.abs(got[m] - ref[m])) <= 1e-13 * np.max(np.abs(ref[m])), axis


@pytest.mark.parametrize("shape", [(30, 12, 36), (60, 12, 36), (90, 12, 36), (120, 12, 36), (250, 12, 36),
                                   (300, 12, 36), (5, 60, 180), (5, 100, 300), (4, 200, 600), (4, 300, 900),
                                   (3, 12, 100), (4, 16, 200), (3, 12, 300), (4, 20, 500), (3, 24, 700),
                                   (3, 40, 1100), (3, 12, 385), (3, 12, 640), (3, 12, 1152)])
def test_line_solve_every_chunking(shape):
    """One case per (P chunks, M rows) dispatch branch of the line solver
    (yy_line.cu), incl. ragged lines (rows past n are identity rows) and the
    longest supported lines (512 r/theta rows, 1152 phi rows)."""
    import torch
    from oracle import ops
    nr, nt, npp = shape
    a, rhs = W.c4_inputs(nr, nt, npp)
    cfg = W.Config("C4", nr, nt, npp, dt=1e-4)
    sh = _shell(cfg)
    o = _oracle(cfg)
    astar = [a["ur"], a["ut"], a["up"]]
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    m = o.g.solved_mask("C")
    for axis in range(3):
        x = dev(rhs)
        sh.line_solve(axis, dev(a["ur"]), dev(a["ut"]), dev(a["up"]), x)
        torch.cuda.synchronize()
        got = x.cpu().numpy()
        ref = o.sweep("T", rhs, axis, ops.coeffs(o.g, o.prm, "T", axis, True, astar))
        assert np.max(np.abs(got[m] - ref[m])) <= 1e-13 * np.max(np.abs(ref[m])), (shape, axis)
        assert np.array_equal(got[~m], rhs[~m]), (shape, axis)   # fringe untouched
        # prepared row weights (yy_line_prepare + NULL a*): the same solve, bitwise
        x2 = dev(rhs)
        sh.line_prepare(dev(a["ur"]), dev(a["ut"]), dev(a["up"]))
        sh.line_solve(axis, None, None, None, x2)
        torch.cuda.synchronize()
        assert np.array_equal(x2.cpu().numpy(), got), (shape, axis)


@pytest.mark.parametrize("var,stream", [("YY_ALT_ORDER", False), ("YY_DP1", False),
                                        ("YY_DEFER_INTERP", False), ("YY_DEFER_INTERP", True)])
def test_data_path_options_are_bitwise_neutral(var, stream):
    """YY_ALT_ORDER: consecutive residual / sweep / pressure kernels run their
    blocks in alternating linear order (L2 reuse) — every block computes the same
    tile and the norm partials keep their slots.  YY_DP1: system 2 reads
    p1^(k) - p1^n from one array written by the system-1 pressure update and the
    p1 fringe interpolation instead of forming it from p1^(k) and p1^n — the same
    subtraction.  YY_DEFER_INTERP: only T's fringe is interpolated ahead of the T
    solve, the p / u fringes on side streams beside it, joined before the first
    momentum residual (stream launches, and captured into the device-side loop
    graph on a user stream).  Either way the step is bit-identical with the option off."""
    import os
    import torch
    cfg = W.small("C3", 9, 17, 47)
    wl = W.random_state(cfg, seed=3, amp=1.0)
    out = []
    st = torch.cuda.Stream() if stream else None
    for val in ("1", "0"):
        os.environ[var] = val
        try:
            sh = _shell(cfg, **({"stream": st.cuda_stream} if stream else {}))
            sh.load_workload(wl)
            sh.step(2, cfg.tol)
            out.append(([sh.get_fields(p, 0, s) for p in range(2) for s in (1, 2)], sh.stats()))
            sh.close()
        finally:
            os.environ.pop(var, None)
    (fa, sa), (fb, sb) = out
    assert sa == sb
    for a, b in zip(fa, fb):
        for k in a:
            assert np.array_equal(a[k], b[k]), k


def test_torch_caching_allocator_hook():
    """yy_set_allocator through PyTorch's caching allocator: the context's buffers
    come from torch (memory_allocated grows by at least the state's size and
    returns at destroy) and the step is bit-identical to cudaMalloc buffers."""
    import torch
    from paper_1905_02300_b200 import use_torch_allocator
    cfg = W.small("C3", 8, 16, 40)
    wl = W.make_workload(cfg)
    out = []
    for hook in (True, False):
        use_torch_allocator(hook)
        try:
            torch.cuda.synchronize()
            m0 = torch.cuda.memory_allocated()
            sh = _shell(cfg)
            torch.cuda.synchronize()
            m1 = torch.cuda.memory_allocated()
            if hook:
                # at least the 32 (nr, nth, nph) state arrays of both patches
                assert m1 - m0 >= 32 * 2 * cfg.nr * cfg.nth * cfg.nph * 8, (m0, m1)
            else:
                assert m1 == m0
            sh.load_workload(wl)
            sh.step(2, cfg.tol)
            out.append(([sh.get_fields(p, 0, s) for p in range(2) for s in (1, 2)], sh.stats()))
            sh.close()
            torch.cuda.synchronize()
            assert torch.cuda.memory_allocated() == m0
        finally:
            use_torch_allocator(False)
    (fa, sa), (fb, sb) = out
    assert sa == sb
    for a, b in zip(fa, fb):
        for k in a:
            assert np.array_equal(a[k], b[k]), k


def test_interp_order_param():
    from paper_1905_02300_b200 import YYError
    from paper_1905_02300_b200.yy import YY_INTERP_ORDER
    sh = _shell(W.small("C1", 4, 12, 28))
    sh.set_param(YY_INTERP_ORDER, 4)
    with pytest.raises(YYError):
        sh.set_param(YY_INTERP_ORDER, 2)


@pytest.mark.parametrize("graph", ["2", "0"])
def test_max_iters_reports_no_convergence(graph):
    """K_max reached before tol: the step completes and yy_step returns the
    positive warning YY_ENOCONV; the same state as the oracle run
    with the same iteration cap."""
    import os
    import torch
    from paper_1905_02300_b200.yy import YY_ENOCONV, YY_OK
    cfg = W.small("C3", 8, 14, 40)
    wl = W.make_workload(cfg)
    os.environ["YY_GRAPH"] = graph
    try:
        st = torch.cuda.Stream()
        sh = _shell(cfg, stream=st.cuda_stream, max_iters=3)
        sh.load_workload(wl)
        assert sh.step(1, 1e-30) == YY_ENOCONV
        assert sh.stats()[-1][0] == 3
        assert sh.step(1, 1e30) == YY_OK
        assert sh.stats()[-1][0] == 1
        sh.close()
    finally:
        os.environ.pop("YY_GRAPH", None)


def test_set_fields_system0_is_both_systems():
    """yy_set_fields(system = 0) fills both systems from one host copy (system 2
    by device copies): the same state as two separate uploads."""
    cfg = W.small("C1", 5, 12, 30, dt=1e-3)
    wl = W.random_state(cfg, seed=7, amp=1.0)
    a, b = _shell(cfg), _shell(cfg)
    for p, pd in enumerate(wl["patches"]):
        n = pd["n"]
        a.set_fields(p, 0, 1, ur=n["ur"], ut=n["ut"], up=n["up"], T=n["T"], p=n["p1"])
        a.set_fields(p, 0, 2, ur=n["ur"], ut=n["ut"], up=n["up"], p=n["p1"])
        b.set_fields(p, 0, 0, ur=n["ur"], ut=n["ut"], up=n["up"], T=n["T"], p=n["p1"])
    for p in range(2):
        for s in (1, 2):
            fa, fb = a.get_fields(p, 0, s), b.get_fields(p, 0, s)
            for k in fa:
                assert np.array_equal(fa[k], fb[k]), (p, s, k)


def test_set_fields_system0_on_a_user_stream_from_pageable_memory():
    """The uploads (pageable numpy arrays) and system 2's device copies run on the
    context's stream — a non-blocking torch stream here — and the call returns
    only when they are done: system 2 equals the host data right away, also after
    a step has queued kernels on that stream, and so do repeated wall re-sets."""
    import torch
    cfg = W.small("C3", 6, 14, 33)
    st = torch.cuda.Stream()
    sh = _shell(cfg, stream=st.cuda_stream)
    wl = W.random_state(cfg, seed=9, amp=2.0)
    sh.load_workload(wl)
    sh.step(1, cfg.tol)                       # kernels queued on the user stream
    for rep in range(3):
        for p, pd in enumerate(wl["patches"]):
            n = pd["n"]
            host = {k: np.array(n[k], copy=True) + rep for k in ("ur", "ut", "up", "T")}
            host["p"] = np.array(n["p1"], copy=True) - rep
            sh.set_fields(p, 0, 0, **host)
            f = sh.get_fields(p, 0, 2)
            for k in ("ur", "ut", "up", "p"):
                assert np.array_equal(f[k], host[k]), (rep, p, k)
            sh.set_wall(p, pd["walls"])       # re-set: the slot buffers are reused
    sh.step(1, cfg.tol)


def test_errors_are_reported():
    from paper_1905_02300_b200 import YYError
    cfg = W.small("C1", 4, 12, 28)
    sh = _shell(cfg)
    with pytest.raises(YYError):
        sh.set_fields(2, 0, 0, T=np.zeros((4, 12, 28)))
    with pytest.raises(YYError):
        sh.set_param(99, 1.0)
    with pytest.raises(YYError):
        sh.step(1, -1.0)


@pytest.mark.parametrize("graph", ["2", "0"])
def test_nan_state_is_reported(graph):
    """A NaN in the state ends the Schwarz loop with YY_ESOLVER, on the
    device-side loop (user stream, YY_GRAPH=2) as on the host loop."""
    import os
    import torch
    from paper_1905_02300_b200 import YYError
    cfg = W.small("C1", 4, 12, 28, dt=1e-3)
    wl = W.make_workload(cfg)
    os.environ["YY_GRAPH"] = graph
    try:
        st = torch.cuda.Stream()
        sh = _shell(cfg, stream=st.cuda_stream)
        sh.load_workload(wl)
        T = wl["patches"][0]["n"]["T"].copy()
        T[2, 5, 9] = np.nan
        sh.set_fields(0, 0, 1, T=T)
        with pytest.raises(YYError, match="NaN"):
            sh.step(1, cfg.tol)
        sh.close()
    finally:
        os.environ.pop("YY_GRAPH", None)


def test_c1_full_config_ten_steps():
    """BASELINE config C1 as specified (16x16x48 per patch, eq:Exact, Pr=1, Ra=100,
    dt=1e-3, 10 steps): every step within the per-step bar, equal Schwarz counts."""
    _pair(W.config("C1"), 10)


def test_hundred_steps_within_drift_bar():
    """BASELINE bar after 100 steps (<= 1e-9 relative), with equal Schwarz counts
    on every step, on a reduced convection shell (noise-seeded, Ra = 1e4)."""
    cfg = W.small("C3", 8, 14, 40)
    wl = W.make_workload(cfg)
    sh = _shell(cfg)
    sh.load_workload(wl)
    o = _oracle(cfg)
    o.load_workload(wl)
    for _ in range(100):
        sh.step(1, cfg.tol)
        o.step(1, cfg.tol)
        assert sh.stats()[-1][0] == o.stats[-1][0], (len(o.stats), sh.stats()[-1], o.stats[-1])
    e, where, _ = _relerr(sh, o)
    assert e <= 1e-9, (e, where)


@pytest.mark.parametrize("fixed", [0, 4])
def test_graph_replay_is_bitwise_the_stream_path(fixed):
    """With a user stream the step runs the whole Schwarz loop as one CUDA graph
    with a device-side WHILE node (YY_GRAPH=2, default) or replays each
    iteration as a graph (YY_GRAPH=1) (yy_api.cu step_group): same kernels, same
    order -> bit-identical to the plain stream launches (YY_GRAPH=0), with the
    same iteration counts, to tolerance and with a fixed count."""
    import os
    import torch
    cfg = W.small("C3", 10, 18, 50)
    wl = W.make_workload(cfg)
    out = []
    for graph in ("2", "1", "0"):
        os.environ["YY_GRAPH"] = graph
        try:
            st = torch.cuda.Stream()
            sh = _shell(cfg, stream=st.cuda_stream, **({"fixed_iters": fixed} if fixed else {}))
            sh.load_workload(wl)
            sh.step(3, cfg.tol)
            torch.cuda.synchronize()
            out.append(([sh.get_fields(p, 0, s) for p in range(2) for s in (1, 2)], sh.stats()))
            sh.close()
        finally:
            os.environ.pop("YY_GRAPH", None)
    (fa, sa) = out[-1]
    if fixed:
        assert all(st[0] == fixed for st in sa), sa
    for fb, sb in out[:-1]:
        assert sa == sb
        for a, b in zip(fa, fb):
            for k in a:
                assert np.array_equal(a[k], b[k]), k


# --- the (P, M) chunkings the BASELINE configurations dispatch (yy_line.cu
# sweep_line), each reached through a whole step on an anisotropic reduced grid:
# C3 96x128x384: r (16,6) [n = 96 / 95], theta (8,16) [126 / 127], phi (32,12) [382 / 383];
# C5 (N = 1) 64x192x576: r (8,8) [64 / 63], theta (16,12) [190 / 191], phi (64,9) [574 / 575];
# every quantity's plain and final factors on that axis, both systems (the r / theta
# factors of the kinds with an even phi pitch run on k_line_th, one line per
# thread, the rest on these chunkings).
# (theta-chunking grids need phi cells as fine as theta cells: the overlap of two
# theta cells must hold the donor stencils, so nphi ~ 3 ntheta there)
@pytest.mark.parametrize("grid", [(96, 12, 40), (3, 128, 384), (8, 12, 384),
                                  (64, 12, 40), (3, 192, 576), (8, 12, 576)])
def test_bench_chunkings_full_step(grid):
    cfg = W.small("C3", *grid, chi=16.0)
    _pair(cfg, 1, wl=W.random_state(cfg, seed=sum(grid), amp=3.0),
          oracle_kw={"chi": 16.0}, shell_kw={"chi": 16.0})


@pytest.mark.parametrize("advection", ["imex"])
def test_imex_advection_parity(advection):
    # the transport terms only in the explicit
    # L_full psi^* (YY_ADVECTION = 1) against Oracle(advection="imex")
    cfg = W.small("C1", 6, 14, 33, Ra=50.0, dt=2e-3)
    kw = {"chi": 16.0, "advection": advection}
    _pair(cfg, 3, wl=W.random_state(cfg, seed=21, amp=3.0), oracle_kw=kw, shell_kw=kw)
