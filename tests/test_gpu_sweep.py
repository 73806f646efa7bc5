"""GPU parity sweep over generator parameters (beyond the BASELINE configs): directed
preferential-attachment graphs with different attachment counts m and reciprocities rho,
Erdős–Rényi graphs from sparse to dense, some under random vertex orders, k = 3 and 4,
directed and undirected motifs -- every entry of every matrix vs the oracle (bit-exact)."""
import numpy as np
import pytest

import graphgen as G
from test_gpu_undirected import ucount

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests need a B200")
    from paper_2201_11655_b200 import build as b
    b.build()
    from paper_2201_11655_b200 import vdmc
    return vdmc


CASES = [("ba", 3000, 3, 0.0), ("ba", 4000, 5, 0.3), ("ba", 2500, 8, 0.1), ("ba", 1500, 16, 0.5),
         ("gnp", 3000, 6.0, None), ("gnp", 800, 40.0, None), ("gnp", 200, 60.0, None)]


def _graph(kind, n, x, rho, seed):
    if kind == "ba":
        return G.ba_directed(n, int(x), seed, rho)
    return G.gnp_directed(n, x / (n - 1), seed)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_sweep(vd, oracle_mod, case):
    import torch
    kind, n, x, rho = CASES[case]
    g = _graph(kind, n, x, rho, 9100 + case)
    rank = np.random.default_rng(case).permutation(n) if case % 2 else None
    gr = vd.Graph(g[0], torch.from_numpy(g[1]).cuda(), torch.from_numpy(g[2]).cuda(), rank=rank)
    for k in (3, 4):
        got = gr.count(k).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, oracle_mod.count_esu(g, k)), (CASES[case], k)
    gr.close()
    if case < 4:
        assert np.array_equal(ucount(vd, g, 4), oracle_mod.count_undirected(g, 4)), CASES[case]
