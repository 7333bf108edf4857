"""The subtree-sharded C-ABI (hpsg_shard_*, include/hps_cuda.h) on one B200: examples/sharded_emulate_b200
runs `world` rank threads with an in-process mailbox transport in place of NCCL send/recv and compares the
gathered solution with a single-context build + solve (the Python twin is sharded.py)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "sharded_emulate_b200")


def run(world, L, p, dim, nrhs):
    src = EXE + ".cpp"
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2503_17535_b200"), "example"], check=True)
    r = subprocess.run([EXE, str(world), str(L), str(p), str(dim), str(nrhs)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout)


@pytest.mark.parametrize("world,L,p,dim,cut", [
    (1, 4, 16, 2, 0), (2, 5, 16, 2, 1), (3, 5, 16, 2, 1), (4, 5, 16, 2, 1), (8, 5, 16, 2, 2), (16, 5, 12, 2, 2),
    (8, 3, 8, 3, 1), (5, 3, 6, 3, 1),
])
def test_shard_matches_single_context(world, L, p, dim, cut):
    rep = run(world, L, p, dim, 2)
    assert rep["cut_depth"] == cut
    assert rep["rel_diff"] < 1e-10
    if world == 1:
        assert rep["messages"] == 0
    else:
        assert rep["messages"] > 0


def test_shard_exchange_volume():
    """world 4 on a quadtree: the three depth-1 children not owned by rank 0 send [h|T] (nb x (1+nb)) up and
    receive nrhs x nb boundary values down, nb = 4 q 2^(L-1) -- and nothing else moves."""
    L, p, nrhs = 5, 16, 2
    rep = run(4, L, p, 2, nrhs)
    nb = 4 * (p - 2) * 2 ** (L - 1)
    assert rep["messages"] == 6
    assert rep["bytes"] == 3 * 8 * (nb * (1 + nb) + nrhs * nb)
