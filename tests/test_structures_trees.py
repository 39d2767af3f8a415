"""HCLT tree shapes (bench workloads hclt256_grid / hclt256_chain): valid
circuits, the expected depths, and the BFS grid tree joining neighbours."""
import numpy as np

from paper_2406_00766_b200 import structures as S


def test_chain_and_grid_trees():
    p = S.chain_tree_parents(6)
    assert p.tolist() == [-1, 0, 1, 2, 3, 4]
    g = S.grid_tree_parents((4, 5, 3))
    assert g[0] == -1 and np.all(g[1:] >= 0)
    # every edge joins grid neighbours (L1 distance 1 in (y, x, c))
    C, W = 3, 5
    for v in range(1, g.size):
        u = g[v]
        dv = np.array([v // (C * W), (v // C) % W, v % C])
        du = np.array([u // (C * W), (u // C) % W, u % C])
        assert np.abs(dv - du).sum() == 1
    # depth of the BFS tree = graph distance from the corner
    depth = np.zeros(g.size, np.int64)
    for v in range(1, g.size):
        d, u = 0, v
        while u != 0:
            u, d = g[u], d + 1
        depth[v] = d
    assert depth.max() == (4 - 1) + (5 - 1) + (3 - 1)


def test_deep_tree_circuits_validate():
    for tree, kw in (("chain", dict(num_vars=12)), ("grid", dict(num_vars=12, shape=(2, 2, 3)))):
        g = S.build_hclt(S.StructureConfig(kind="hclt", hidden_dim=4, num_categories=3, seed=1,
                                           tree=tree, **kw))
        assert g.validate().ok
        assert g.num_vars == 12
