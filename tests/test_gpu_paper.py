"""NEXT-4: the paper's own benchmark shape (R19)
-- 3 levels with ratio 2, van Leer limiter with corner transport, the ring,
levels 2-3 created by flagging + Berger-Rigoutsos clustering at t = 0 and
re-created every few coarse steps -- against the oracle's composition of the
same steps, through the C-ABI.

Regrid decisions are integer decisions taken from fp64 data: before each
regrid the GPU hierarchy is overwritten with the oracle's bytes, so both sides
build the same patch lists (checked exactly) and the same new data (checked
bitwise); between regrids the runs are compared at the north_star bar."""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


def params(wl, L, dxl):
    e, R = wl.extra, wl.extra["ratios"]
    return dict(tol=e["tol_per_dx"] * dxl, buffer=int(e["buffer_coarse_cells"] * np.prod(R[:L - 1])),
                cutoff=e["cutoff"], max_dim=e["max_dim"], min_dim=e["min_dim"], R=R[L - 1])


def regrid_both(g, o, wl, t, nlev):
    for L in range(1, nlev):
        if L > 1:
            g.fill_ghost(L, t)
            o.fill_ghost(L, t)
        p = params(wl, L, float(o.descs(L)["dx"][0]))
        ng = g.regrid_auto(L, **p)
        no = oracle.regrid_auto(o, L, **p)
        assert ng == no and ng > 0, (L, ng, no)
        dg, do = g.descs(L + 1), o.descs(L + 1)
        for k in ("mx", "my", "xlower", "ylower"):
            assert np.array_equal(dg[k], do[k]), (L, k)
        assert np.array_equal(g.read_level(L + 1), o.read_level(L + 1)), L


def bo_oracle(o, level, t, dt, R, nlev):
    o.fill_ghost(level, t)
    o.advance_level(level, dt)
    if level < nlev:
        for k in range(R[level - 1]):
            bo_oracle(o, level + 1, t + k * dt / R[level - 1], dt / R[level - 1], R, nlev)
        o.update_level(level + 1)


@pytest.mark.parametrize("n1,every", [(64, 2), (96, 3)])
def test_dynamic_van_leer_run_matches_oracle(n1, every):
    wl = W.paper(n1=n1, npx=4)
    R = wl.extra["ratios"]
    nlev = 1 + len(R)
    d1 = wl.levels[0].descs
    q1 = W.ring_ic(d1)
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans)
    for h in (g, o):
        h.set_level(1, d1, q1)
    regrid_both(g, o, wl, 0.0, nlev)
    dt = wl.dt0()
    for n in range(2 * every):
        g.advance_hierarchy(n * dt, dt, update=True)
        bo_oracle(o, 1, n * dt, dt, R, nlev)
        for L in range(1, nlev + 1):
            qg, qo = g.read_level(L), o.read_level(L)
            assert np.abs(qg - qo).max() <= TOL * np.abs(qo).max(), (n, L)
        if (n + 1) % every == 0:
            for L in range(1, nlev + 1):
                g.write_level(L, o.read_level(L))       # same bytes -> same flags
            regrid_both(g, o, wl, (n + 1) * dt, nlev)
    g.close()


def test_full_size_hierarchy_covers_every_flag():
    """At the benchmark's size (1000^2 base): after the initial regrid every
    buffered, nesting-clipped flag of level L lies under level L+1, the
    fine patches respect the size limit and nest (claw_set_level's
    ghost-donor validation passed), and one coarse step runs."""
    wl = W.paper()
    R = wl.extra["ratios"]
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    d1 = wl.levels[0].descs
    g.set_level(1, d1, W.ring_ic(d1))
    for L in (1, 2):
        if L > 1:
            g.fill_ghost(L, 0.0)
        p = params(wl, L, float(g.descs(L)["dx"][0]))
        f = g.flag(L, p["tol"], buffer=p["buffer"], clip=2)
        assert f.sum() > 1000
        g.regrid_auto(L, **p)
        d = g.descs(L + 1)
        assert len(d) > 0 and d["mx"].max() <= 260 and d["my"].max() <= 260
        nx, ny = g.level_extent(L + 1)
        cov = oracle.cover_map(d, wl.domain, nx, ny)
        r = R[L - 1]
        cov_c = cov.reshape(ny // r, r, nx // r, r).max(axis=(1, 3))
        assert cov_c[f == 1].all()
    cfl = g.advance_hierarchy(0.0, wl.dt0(), update=True)
    assert abs(cfl - wl.cfl) < 1e-12
    g.close()


def test_dynamic_run_with_conservation_fix_conserves_and_matches():
    """Dynamic hierarchy + updating + the conservation fix (periodic BCs):
    regrids re-create levels 2-3 (their registers rebuilt empty), and the
    level-1 totals of p, u, v stay constant to round-off through the steps
    and the regrids; GPU = oracle throughout."""
    wl = W.paper(n1=64, npx=4)
    wl.bc = W.PERIODIC
    R = wl.extra["ratios"]
    nlev = 1 + len(R)
    d1 = wl.levels[0].descs
    q1 = W.ring_ic(d1)
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, reflux=True)
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, reflux=True)
    for h in (g, o):
        h.set_level(1, d1, q1)
    regrid_both(g, o, wl, 0.0, nlev)
    dt = wl.dt0()
    totals = [g.read_level(1).reshape(len(d1), 3, -1).sum(axis=(0, 2))]
    for n in range(6):
        g.advance_hierarchy(n * dt, dt, update=True)
        bo_oracle(o, 1, n * dt, dt, R, nlev)
        for L in range(1, nlev + 1):
            qg, qo = g.read_level(L), o.read_level(L)
            assert np.abs(qg - qo).max() <= TOL * np.abs(qo).max(), (n, L)
        totals.append(g.read_level(1).reshape(len(d1), 3, -1).sum(axis=(0, 2)))
        if (n + 1) % 2 == 0:
            for L in range(1, nlev + 1):
                g.write_level(L, o.read_level(L))
            regrid_both(g, o, wl, (n + 1) * dt, nlev)
    scale = np.abs(g.read_level(1)).sum()
    drift = np.abs(np.array(totals[1:]) - totals[0]).max()
    assert drift <= 1e-13 * scale, (drift, scale)
    g.close()
