"""Host-side regridding logic of libclaw.so (no GPU): claw_cluster, the
native Berger-Rigoutsos clusterer (R18), must
return exactly the oracle's boxes (integer work: bit-exact, same order) and
satisfy the clustering postconditions on its own."""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding
from test_oracle_regrid import check_boxes


def ring_map(seed, ny=70, nx=90, noise=0.995):
    rng = np.random.default_rng(seed)
    Y, X = np.mgrid[0:ny, 0:nx]
    r = np.hypot(X - 40 - seed % 7, Y - 33)
    return ((np.abs(r - 22) < 3) | (rng.uniform(size=(ny, nx)) > noise)).astype(np.uint8)


def blob_map(seed, ny=64, nx=48):
    rng = np.random.default_rng(100 + seed)
    f = np.zeros((ny, nx), np.uint8)
    for _ in range(rng.integers(1, 6)):
        a, b = rng.integers(0, nx - 1), rng.integers(0, ny - 1)
        w, h = rng.integers(1, 20), rng.integers(1, 20)
        f[b:b + h, a:a + w] = 1
    f[rng.uniform(size=f.shape) > 0.98] = 1
    return f


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("cutoff,max_dim,min_dim", [(0.7, 32, 4), (0.9, 16, 2), (0.5, 64, 8), (0.8, 8, 1),
                                                    (1.0, 24, 3)])
def test_cluster_equals_oracle(seed, cutoff, max_dim, min_dim):
    for f in (ring_map(seed), blob_map(seed)):
        got = binding.cluster(f, cutoff, max_dim, min_dim)
        want = oracle.cluster(f, cutoff, max_dim, min_dim)
        assert np.array_equal(got, want), (got.tolist(), want.tolist())
        check_boxes(f, got, cutoff, max_dim, min_dim)


def test_cluster_edge_cases():
    assert len(binding.cluster(np.zeros((5, 7), np.uint8), 0.7, 16, 2)) == 0
    one = np.zeros((5, 7), np.uint8)
    one[3, 6] = 1
    assert binding.cluster(one, 0.7, 16, 2).tolist() == [[6, 3, 1, 1]]
    full = np.ones((40, 40), np.uint8)
    b = binding.cluster(full, 0.7, 16, 4)
    assert np.array_equal(b, oracle.cluster(full, 0.7, 16, 4))
    check_boxes(full, b, 0.7, 16, 4)
    # S:258 / S:259 worked examples
    f = np.zeros((20, 30), np.uint8)
    f[2:12, 3:13] = 1
    assert binding.cluster(f, 0.9, 64, 2).tolist() == [[3, 2, 10, 10]]
    g = np.zeros((10, 30), np.uint8)
    g[2:6, 2:6] = 1
    g[2:6, 16:20] = 1
    assert sorted(map(tuple, binding.cluster(g, 0.7, 64, 2).tolist())) == [(2, 2, 4, 4), (16, 2, 4, 4)]


def test_cluster_argument_errors():
    f = np.ones((4, 4), np.uint8)
    for args in [(0.0, 16, 2), (1.5, 16, 2), (0.7, 3, 2), (0.7, 16, 0)]:
        with pytest.raises(binding.ClawError):
            binding.cluster(f, *args)


@pytest.mark.parametrize("threads", ["1", "3", "8"])
def test_cluster_parallel_subtrees_equal_oracle(threads):
    """Large maps: after the first cuts the clusterer hands the stacked boxes'
    subtrees to host workers and concatenates their outputs in pop order;
    the boxes (and their order) must still be the oracle's, for any thread
    count (CLAW_HOST_THREADS is read once per process, so the thread count is
    varied in a subprocess)."""
    import subprocess, sys, os
    code = (
        "import numpy as np, oracle\n"
        "from paper_1808_02638_b200 import binding\n"
        "Y, X = np.mgrid[0:400, 0:520]\n"
        "r = np.hypot(X - 260.5, Y - 200.5) / 200\n"
        "rng = np.random.default_rng(4)\n"
        "f = ((np.abs(r - 0.5) < 0.06) | (np.abs(r - 0.8) < 0.03) | (rng.uniform(size=r.shape) > 0.999)).astype(np.uint8)\n"
        "for c, M, m in [(0.7, 40, 4), (0.8, 16, 2), (0.6, 64, 8)]:\n"
        "    got = binding.cluster(f, c, M, m); want = oracle.cluster(f, c, M, m)\n"
        "    assert len(got) > 40, len(got)\n"
        "    assert np.array_equal(got, want)\n"
        "print('ok')\n")
    env = dict(os.environ, CLAW_HOST_THREADS=threads)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_host_worker_pool_after_fork():
    """The planner's persistent host workers do not survive fork(): a child
    process starts its own pool and clusters like the parent."""
    import os
    import sys
    if not hasattr(os, "fork") or sys.platform != "linux":
        pytest.skip("fork")
    Y, X = np.mgrid[0:300, 0:300]
    f = (np.abs(np.hypot(X - 150, Y - 150) / 150 - 0.5) < 0.05).astype(np.uint8)
    a = binding.cluster(f, 0.7, 40, 4)
    pid = os.fork()
    if pid == 0:
        ok = np.array_equal(binding.cluster(f, 0.7, 40, 4), a)
        os._exit(0 if ok else 3)
    _, st = os.waitpid(pid, 0)
    assert os.WEXITSTATUS(st) == 0 and len(a) > 4
