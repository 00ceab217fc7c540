"""Multi-GPU layout, one patch per rank.

CPU (gloo, world size 2): the host plumbing — rank -> patch plan and the NCCL
unique-id handshake through torch.distributed — is the same on every rank.

GPU (one device): yy_create_pair runs the distributed data path (donor-side
fringe evaluation, transfer, target write, fixed-order norm merge) with two
one-patch contexts exchanging by device copies.  It must reproduce the
single-context step bit for bit (same kernels, same operands) and therefore the
oracle within the parity bar, with identical Schwarz iteration counts."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

import workloads as W
from oracle.scheme import Oracle


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_02300_b200 import dist
        uid = dist.share_unique_id(rank)
        q.put((rank, dist.plan(world, rank), uid))
    finally:
        td.destroy_process_group()


def test_plan_and_unique_id_handshake_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(2):
        r, plan, uid = q.get(timeout=120)
        got[r] = (plan, uid)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert got[0][0]["patches"] == (0,) and got[0][0]["partner"] == 1
    assert got[1][0]["patches"] == (1,) and got[1][0]["partner"] == 0
    assert len(got[0][1]) == 128 and got[0][1] == got[1][1] and any(got[0][1])


def test_plan_layout():
    """Yin on the first nslab ranks, Yang on the rest; fringe partner = same slab of
    the other patch, slab neighbours within the patch."""
    from paper_1905_02300_b200 import dist
    assert dist.plan(1, 0)["patches"] == (0, 1)
    p = [dist.plan(8, r, nr=512) for r in range(8)]
    assert [q["patch"] for q in p] == [0, 0, 0, 0, 1, 1, 1, 1]
    assert [q["slab"] for q in p] == [0, 1, 2, 3, 0, 1, 2, 3]
    assert [q["partner"] for q in p] == [4, 5, 6, 7, 0, 1, 2, 3]
    assert [q["below"] for q in p] == [None, 0, 1, 2, None, 4, 5, 6]
    assert [q["above"] for q in p] == [1, 2, 3, None, 5, 6, 7, None]
    for world in (3, 6, 32):
        with pytest.raises(ValueError):
            dist.plan(world, 0)
    with pytest.raises(ValueError):
        dist.plan(8, 0, nr=96 + 2)       # 98 rows do not split into 4 slabs


def test_c5_weak_scaling_layout():
    """BASELINE C5 (bench.py --workload C5 at N GPUs): patch Nr = 64 N, a 128-row
    slab per rank for N = 2, 4, 8, every slab solvable by the slab
    chunk menu (n = P M: 128 = 16 x 8)."""
    import workloads as W
    from paper_1905_02300_b200 import dist
    assert W.config("C5").nr == 64
    for world in (2, 4, 8):
        cfg = W.config("C5", G=world)
        plans = [dist.plan(world, r, cfg.nr) for r in range(world)]
        S = plans[0]["nslab"]
        assert cfg.nr // S == 128 and S == world // 2
        assert sorted((q["patch"], q["slab"]) for q in plans) == [(p, s) for p in (0, 1) for s in range(S)]


def _fields_all(shells, p, lev, s):
    for sh in shells:
        if p in sh.patches:
            return sh.get_fields(p, lev, s)
    raise AssertionError(p)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "convection", "random"])
def test_pair_reproduces_single_context_and_oracle(case):
    from paper_1905_02300_b200 import Shell
    if case == "c1":
        cfg, wl, steps = W.config("C1"), None, 2
    elif case == "convection":
        cfg, wl, steps = W.small("C3", 10, 18, 50), None, 2
    else:
        cfg = W.small("C1", 7, 13, 37, Ra=30.0, dt=2e-3)
        wl, steps = W.random_state(cfg, seed=11, amp=5.0), 2
    wl = wl if wl is not None else W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    one = Shell(*args)
    one.load_workload(wl)
    pair = Shell.pair(*args)
    for sh in pair:
        sh.load_workload(wl)
    o = Oracle(*args)
    o.load_workload(wl)
    for _ in range(steps):
        one.step(1, cfg.tol)
        pair[0].step(1, cfg.tol)           # advances both members
        o.step(1, cfg.tol)
        assert pair[0].stats()[-1] == one.stats()[-1] == pair[1].stats()[-1]
        assert one.stats()[-1][0] == o.stats[-1][0]
        for p in range(2):
            for s in (1, 2):
                a = one.get_fields(p, 0, s)
                b = _fields_all(pair, p, 0, s)
                c = o.get_fields(p, 0, s)
                vmax = max(np.max(np.abs(c[q])) for q in ("ur", "ut", "up"))
                for k in a:
                    assert np.array_equal(a[k], b[k]), (p, s, k)
                    den = vmax if k in ("ur", "ut", "up") else max(np.max(np.abs(c[k])), 1e-300)
                    assert np.max(np.abs(b[k] - c[k])) / den <= 1e-11, (p, s, k)


@pytest.mark.gpu
def test_pair_members_only_accept_their_patch():
    from paper_1905_02300_b200 import Shell, YYError
    cfg = W.small("C1", 4, 12, 28)
    yin, yang = Shell.pair(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    with pytest.raises(YYError):
        yin.set_fields(1, 0, 0, T=np.zeros((4, 12, 28)))
    with pytest.raises(YYError):
        yang.get_fields(0, 0, 2)
    yang.close()
    with pytest.raises(YYError):      # partner gone
        yin.step(1, 1e-10)


def _assemble(shells, p, lev, s):
    out = None
    for sh in shells:
        if p in sh.patches:
            if out is None:
                out = {n: np.full(sh.shape(n), np.nan) for n in ("ur", "ut", "up", "p", "T")}
            sh.get_fields(p, lev, s, out=out)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("nslab,case", [(2, "c1"), (2, "random"), (4, "convection"), (2, "c3rows"), (4, "c3rows")])
def test_radial_slabs_match_oracle(nslab, case):
    """Radial slabs (r-halos, partitioned r-sweep across slabs, per-slab norms)
    against the oracle: the slab solve changes only the rounding order of the
    r-line solves, so the bar is the parity bar, not bit equality."""
    from paper_1905_02300_b200 import Shell
    if case == "c1":
        cfg, wl = W.small("C1", 32, 12, 30, dt=1e-3), None
    elif case == "random":
        cfg = W.small("C1", 32, 13, 37, Ra=30.0, dt=2e-3)
        wl = W.random_state(cfg, seed=11, amp=5.0)
    elif case == "convection":
        cfg, wl = W.small("C3", 64, 14, 40), None
    else:                                   # C3's 96 radial rows: slabs of 48 / 24 rows
        cfg, wl = W.small("C3", 96, 14, 40), None
    wl = wl if wl is not None else W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    group = Shell.slabs(*args, nslab=nslab)
    for sh in group:
        sh.load_workload(wl)
    o = Oracle(*args)
    o.load_workload(wl)
    for _ in range(2):
        group[0].step(1, cfg.tol)
        o.step(1, cfg.tol)
        assert all(sh.stats()[-1] == group[0].stats()[-1] for sh in group)
        assert group[0].stats()[-1][0] == o.stats[-1][0], (group[0].stats(), o.stats)
        for p in range(2):
            for s in (1, 2):
                b = _assemble(group, p, 0, s)
                c = o.get_fields(p, 0, s)
                vmax = max(np.max(np.abs(c[q])) for q in ("ur", "ut", "up"))
                for k in c:
                    assert not np.isnan(b[k]).any(), (p, s, k)      # every row owned by exactly one slab
                    den = vmax if k in ("ur", "ut", "up") else max(np.max(np.abs(c[k])), 1e-300)
                    assert np.max(np.abs(b[k] - c[k])) / den <= 1e-11, (p, s, k)


@pytest.mark.gpu
@pytest.mark.parametrize("nslab,case", [(1, "c1"), (1, "random"), (2, "convection")])
def test_multiplicative_schwarz_matches_oracle(nslab, case):
    """Algorithm 1 as printed (Yin first with Yang's iterate k-1,
    then Yang with Yin's fresh iterate k), on one-patch contexts (pair / slabs),
    against the multiplicative oracle: parity bar and equal Schwarz counts."""
    from paper_1905_02300_b200 import Shell
    if case == "c1":
        cfg, wl = W.small("C1", 16, 12, 30, dt=1e-3), None
    elif case == "random":
        cfg = W.small("C1", 16, 13, 37, Ra=30.0, dt=2e-3)
        wl = W.random_state(cfg, seed=11, amp=5.0)
    else:
        cfg, wl = W.small("C3", 32, 14, 40), None
    wl = wl if wl is not None else W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    group = Shell.pair(*args, schwarz="multiplicative") if nslab == 1 else \
        Shell.slabs(*args, nslab=nslab, schwarz="multiplicative")
    for sh in group:
        sh.load_workload(wl)
    o = Oracle(*args, schwarz="multiplicative")
    o.load_workload(wl)
    for _ in range(2):
        group[0].step(1, cfg.tol)
        o.step(1, cfg.tol)
        assert group[0].stats()[-1][0] == o.stats[-1][0], (group[0].stats(), o.stats)
        for p in range(2):
            for s in (1, 2):
                b = _assemble(group, p, 0, s)
                c = o.get_fields(p, 0, s)
                vmax = max(np.max(np.abs(c[q])) for q in ("ur", "ut", "up"))
                for k in c:
                    den = vmax if k in ("ur", "ut", "up") else max(np.max(np.abs(c[k])), 1e-300)
                    assert np.max(np.abs(b[k] - c[k])) / den <= 1e-11, (p, s, k)


@pytest.mark.gpu
def test_multiplicative_needs_one_patch_per_context():
    from paper_1905_02300_b200 import YY_SCHWARZ, Shell, YYError
    cfg = W.small("C1", 4, 12, 28)
    sh = Shell(cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    with pytest.raises(YYError):
        sh.set_param(YY_SCHWARZ, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["single", "pair", "pair_mult"])
def test_flux_fix_matches_oracle(layout):
    """Algorithm 1 step 4 (closed-form minimiser of J, eps = 1e-6)
    every iteration, against the oracle with the same correction: parity bar and
    equal Schwarz counts; and the correction is active (results differ from the
    run without it)."""
    from paper_1905_02300_b200 import Shell
    cfg = W.small("C1", 8, 13, 37, Ra=30.0, dt=2e-3)
    wl = W.random_state(cfg, seed=11, amp=5.0)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    mode = "multiplicative" if layout == "pair_mult" else "additive"
    if layout == "single":
        group = [Shell(*args, flux_fix_eps=1e-6)]
    else:
        group = Shell.pair(*args, schwarz=mode, flux_fix_eps=1e-6)
    for sh in group:
        sh.load_workload(wl)
    o = Oracle(*args, schwarz=mode, flux_fix_eps=1e-6)
    o.load_workload(wl)
    off = Oracle(*args, schwarz=mode)
    off.load_workload(wl)
    for _ in range(2):
        group[0].step(1, cfg.tol)
        o.step(1, cfg.tol)
        off.step(1, cfg.tol)
        assert group[0].stats()[-1][0] == o.stats[-1][0]
    moved = 0.0
    for p in range(2):
        for s in (1, 2):
            b = _assemble(group, p, 0, s)
            c = o.get_fields(p, 0, s)
            d = off.get_fields(p, 0, s)
            vmax = max(np.max(np.abs(c[q])) for q in ("ur", "ut", "up"))
            for k in ("ur", "ut", "up", "p"):
                den = vmax if k != "p" else max(np.max(np.abs(c[k])), 1e-300)
                assert np.max(np.abs(b[k] - c[k])) / den <= 1e-11, (p, s, k)
                moved = max(moved, np.max(np.abs(c[k] - d[k])) / den)
    assert moved > 1e-9          # the correction changed the iterates


@pytest.mark.gpu
@pytest.mark.parametrize("nslab", [1, 2])
def test_loopback_group_graph_is_bitwise_the_stream_path(nslab):
    """A loopback group on a user stream replays each Schwarz iteration as one
    CUDA graph (all members' kernels and transfers, the slab V / W written every
    replay): bit-identical to the stream launches (YY_GRAPH=0), same counts."""
    import os
    import torch
    from paper_1905_02300_b200 import Shell
    cfg = W.small("C3", 32, 14, 40)        # slabs of 16 rows (the slab chunk menu)
    wl = W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    out = []
    for graph in ("1", "0"):
        os.environ["YY_GRAPH"] = graph
        try:
            st = torch.cuda.Stream()
            grp = (Shell.pair(*args, stream=st.cuda_stream) if nslab == 1
                   else Shell.slabs(*args, nslab=nslab, stream=st.cuda_stream))
            for sh in grp:
                sh.load_workload(wl)
            grp[0].step(3, cfg.tol)
            torch.cuda.synchronize()
            def whole(p, s):      # every member's rows of patch p, assembled
                names = ("ur", "ut", "up", "p", "T")
                f = {n: np.zeros(grp[0].shape(n)) for n in names}
                for sh in grp:
                    if p in sh.patches:
                        sh.get_fields(p, 0, s, out=f)
                return f
            out.append(([whole(p, s) for p in range(2) for s in (1, 2)], grp[0].stats()))
            for sh in grp:
                sh.close()
        finally:
            os.environ.pop("YY_GRAPH", None)
    (fa, sa), (fb, sb) = out
    assert sa == sb
    for a, b in zip(fa, fb):
        for k in a:
            assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_c5_layouts_match_oracle_full_r(G):
    """The C5 weak-scaling layouts of G GPUs (BASELINE configs[4], SURVEY §8(e):
    patch Nr = 64 G, Yin on ranks 0..G/2-1 and Yang on the others, G/2 radial
    slabs of 128 rows per patch; G = 2: one patch per rank) on the loopback
    contexts of one GPU, at the FULL radial extent and physics of C5 (manufactured,
    Ra = 1e5, dt = 1e-4, chi = 16) on a reduced 14 x 40 angular grid, against the
    oracle: the first step element by element with equal Schwarz counts."""
    from paper_1905_02300_b200 import Shell
    full = W.config("C5", G=G)
    cfg = W.small("C5", full.nr, 14, 40)
    wl = W.make_workload(cfg)
    args = (cfg.nr, cfg.nth, cfg.nph, cfg.R1, cfg.R2, cfg.Pr, cfg.Ra, cfg.dt)
    nslab = G // 2
    group = Shell.pair(*args, chi=cfg.chi) if nslab == 1 else Shell.slabs(*args, nslab=nslab, chi=cfg.chi)
    for sh in group:
        sh.load_workload(wl)
    o = Oracle(*args, chi=cfg.chi)
    o.load_workload(wl)
    group[0].step(1, cfg.tol)
    o.step(1, cfg.tol)
    assert all(sh.stats()[-1] == group[0].stats()[-1] for sh in group)
    assert group[0].stats()[-1][0] == o.stats[-1][0], (group[0].stats(), o.stats)
    for p in range(2):
        for s in (1, 2):
            b = _assemble(group, p, 0, s)
            c = o.get_fields(p, 0, s)
            vmax = max(np.max(np.abs(c[q])) for q in ("ur", "ut", "up"))
            for k in c:
                assert not np.isnan(b[k]).any(), (p, s, k)
                den = vmax if k in ("ur", "ut", "up") else max(np.max(np.abs(c[k])), 1e-300)
                assert np.max(np.abs(b[k] - c[k])) / den <= 1e-11, (G, p, s, k)
