"""Pins of the oracle's *updating* (NEXT-1): covered
coarse cells become the mean of their R x R fine children."""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import workloads as W


def setup(R, fine_boxes, coarse_q, fine_q_fn, n=8, dom=(0.0, 1.0, 0.0, 1.0)):
    cd = W.uniform_level(1, 1, n, n, dom)
    dxf = (dom[1] - dom[0]) / n / R
    fd = np.concatenate([W.make_descs([a], [b], w, h, dxf, dxf, dom) for a, b, w, h in fine_boxes])
    fq = np.concatenate([fine_q_fn(a, b, w, h) for a, b, w, h in fine_boxes])
    o = oracle.Oracle(dom, W.EXTRAP, 4, 2)
    o.set_level(1, cd, coarse_q)
    o.set_level(2, fd, fq)
    return o, cd, fd


def test_mean_of_children_r2():
    # S:325 example: R=2 children {1,2,3,4} -> 2.5
    o, cd, fd = setup(2, [(4, 6, 2, 2)], np.zeros(3 * 64),
                      lambda a, b, w, h: np.tile(np.array([[1.0, 2.0], [3.0, 4.0]]).ravel(), 3))
    o.update_level(2)
    q = o.read(1, 0)
    assert q[0, 3, 2] == 2.5 and q[1, 3, 2] == 2.5 and q[2, 3, 2] == 2.5
    q[:, 3, 2] = 0
    assert not q.any()                      # nothing else touched


@pytest.mark.parametrize("R", [2, 4])
def test_constant_preserved_idempotent_and_area_identity(R):
    rng = np.random.default_rng(R)
    boxes = [(2 * R, R, 3 * R, 2 * R), (R, 5 * R, R, 2 * R)]
    cq = rng.uniform(-1, 1, 3 * 64)
    o, cd, fd = setup(R, boxes, cq, lambda a, b, w, h: rng.uniform(-1, 1, 3 * w * h))
    fine = [o.read(2, p) for p in range(len(fd))]
    o.update_level(2)
    c1 = o.read(1, 0)
    o.update_level(2)
    assert np.array_equal(o.read(1, 0), c1)            # idempotent
    # area identity: coarse area * sum(replaced coarse) == fine area * sum(fine)
    dxc = 1 / 8
    dxf = dxc / R
    covered = np.zeros((8, 8), bool)
    for a, b, w, h in boxes:
        covered[b // R:(b + h) // R, a // R:(a + w) // R] = True
    for m in range(3):
        lhs = dxc * dxc * c1[m][covered].sum()
        rhs = dxf * dxf * sum(f[m].sum() for f in fine)
        assert lhs == pytest.approx(rhs, rel=1e-14, abs=1e-15)
    # uncovered coarse cells keep their values
    assert np.array_equal(c1[:, ~covered], cq.reshape(3, 8, 8)[:, ~covered])
    # constant fine field -> covered coarse cells take the constant
    o2, _, _ = setup(R, boxes, cq, lambda a, b, w, h: np.full(3 * w * h, 0.375))
    o2.update_level(2)
    assert (o2.read(1, 0)[:, covered] == 0.375).all()


def test_linear_field_gives_cell_centre_value():
    R = 4
    f = lambda x, y: 3.0 * x - 2.0 * y + 0.5
    def fine(a, b, w, h):
        x = (a + np.arange(w) + 0.5) / (8 * R)
        y = (b + np.arange(h) + 0.5) / (8 * R)
        X, Y = np.meshgrid(x, y)
        return np.tile(f(X, Y).ravel(), 3)
    o, cd, fd = setup(R, [(8, 8, 16, 12)], np.zeros(3 * 64), fine)
    o.update_level(2)
    q = o.read(1, 0)
    for jc in range(2, 5):
        for ic in range(2, 6):
            assert q[0, jc, ic] == pytest.approx(f((ic + 0.5) / 8, (jc + 0.5) / 8), abs=1e-14)


def test_time_mismatch_is_an_error():
    o, cd, fd = setup(2, [(4, 4, 2, 2)], np.zeros(3 * 64), lambda a, b, w, h: np.zeros(12))
    o.fill_ghost(1, 0.0)
    o.advance_level(1, 0.01)                      # coarse ahead of fine
    with pytest.raises(oracle.OracleError):
        o.update_level(2)
