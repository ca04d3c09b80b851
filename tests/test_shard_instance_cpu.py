"""Per-rank instance generation for subtree-sharded runs (host only): a
rank's instance (scenopt_problem_gen_random_shard) draws the reference's
random stream in full (generators.hpp:255-328 order) but builds only the
nodes it holds -- its subtrees under scenopt_shard_plan, the stages above and
the shard-stage nodes. Those nodes equal the full instance bit for bit, every
dual row is complete, and the instance refuses uses that need other nodes."""
import ctypes as C

import numpy as np
import pytest

import paper_2107_01745_b200 as so

CASES = [(3, 6, 3, 7, [4, 3, 2], 2, -1), (5, 4, 2, 9, [3, 2, 2, 2], 3, 2), (1, 5, 3, 6, [8, 2], 4, 1)]


def _held(prob, world, stage, rank):
    st = C.c_int32()
    b = (C.c_int32 * (world + 1))()
    so.api.check(so.lib().scenopt_shard_plan(prob._h, world, stage, C.byref(st), b))
    f = prob.flat()
    so_, anc, n = f["stage_offsets"], f["ancestor"], f["num_nodes"]
    s = st.value
    mine = np.zeros(n, bool)
    mine[: so_[s + 1]] = True  # top + every shard-stage node
    own = np.zeros(n, bool)
    own[b[rank]:b[rank + 1]] = True
    for c in range(so_[s + 1], n):
        own[c] = own[anc[c]]
    return mine | own


@pytest.mark.parametrize("seed,nx,nu,N,br,world,stage", CASES)
def test_shard_instance_matches_full_instance_on_held_nodes(_built_libraries, seed, nx, nu, N, br, world, stage):
    full = so.gen_random_instance(seed, nx, nu, N, br)
    ff = full.flat()
    n, F = ff["num_nodes"], ff["stage_offsets"][N]
    for rank in range(world):
        part = so.gen_random_instance_shard(seed, nx, nu, N, br, rank, world, stage)
        pf = part.flat()
        held = _held(full, world, stage, rank)
        assert 0 < held.sum() < n
        for key, per in (("A", nx * nx), ("B", nx * nu), ("Q", nx * nx), ("R", nu * nu), ("S", nx * nu)):
            a = ff[key].reshape(n, per)
            b = pf[key].reshape(n, per)
            assert np.array_equal(a[held], b[held]), key
            assert not np.any(b[~held]), key  # never built
        leaves = held[F:]
        for key, per in (("P", nx * nx), ("p", nx)):
            a = ff[key].reshape(n - F, per)
            b = pf[key].reshape(n - F, per)
            assert np.array_equal(a[leaves], b[leaves]), key
        for key in ("F", "G", "FN", "zmin", "zmax", "probability", "q", "r", "c"):  # every dual row / cheap draw
            assert np.array_equal(ff[key], pf[key]), key
        with pytest.raises(so.InvalidParams):
            so.factor(part)
        with pytest.raises(so.InvalidParams):
            so.serialize_problem(part)


_RSS_SCRIPT = r"""
import json, sys, psutil
import paper_2107_01745_b200 as so
proc = psutil.Process()
r0 = proc.memory_info().rss
p = so.gen_random_instance_shard(1, 50, 20, 20, [8, 8, 8, 2], 0, 8)
r1 = proc.memory_info().rss
print(json.dumps({"delta": r1 - r0, "n": p.flat()["num_nodes"]}))
"""


def test_shard_instance_leaves_unheld_matrices_unbacked(_built_libraries):
    """Host RAM per rank ~1/N: at C3 (17,993 nodes, nx=50, nu=20) the per-node
    matrices A, B, Q, R, S are ~1.07 GB in a full instance; a rank of 8 writes
    only the blocks of the nodes it holds, and the rest of those arrays are
    never-touched anonymous pages (model.hpp NoInitAlloc), so the process grows
    by a fraction of that (0.23x measured). Run in a fresh interpreter for a clean RSS delta."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    out = subprocess.run([sys.executable, "-c", _RSS_SCRIPT], env=env, capture_output=True, text=True, timeout=600,
                         check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    full = r["n"] * (2 * 50 * 50 + 2 * 50 * 20 + 20 * 20) * 8
    assert r["delta"] < 0.35 * full, (r["delta"], full)
