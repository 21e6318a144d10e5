"""A small seeded Chung-Lu power-law graph (the reference has no power-law generator; BASELINE
configs[4] is a power-law graph trained in hybrid mode). Written with save_dataset so the reference
(`ref_driver ... spec=dir:PATH`) and the GPU engine load identical bytes; the dataset directory is
committed as a test fixture and the reference's training outputs on it become golden files via
make_golden.py.

    python tests/golden/make_powerlaw.py      # writes tests/golden/powerlaw_2k/
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def chung_lu(n, avg_deg, gamma, seed):
    """Edge list (u < v) with P(u, v) = min(1, w_u w_v / sum w), w_i ~ (i + 1)^(-1 / (gamma - 1))."""
    rng = np.random.default_rng(seed)
    w = (np.arange(n) + 1.0) ** (-1.0 / (gamma - 1.0))
    w *= avg_deg * n / w.sum()
    W = w.sum()
    edges = []
    for u in range(n - 1):
        p = np.minimum(1.0, w[u] * w[u + 1:] / W)
        hit = np.nonzero(rng.random(n - 1 - u) < p)[0]
        edges.extend((u, u + 1 + int(v)) for v in hit)
    return np.array(edges, np.uint32)


def main(out=os.path.join(HERE, "powerlaw_2k")):
    import paper_2308_10087_b200 as gp
    n, F, C = 2000, 24, 6
    e = chung_lu(n, 12.0, 2.2, 2308)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n, F)).astype(np.float32)
    lab = rng.integers(0, C, n).astype(np.uint32)
    sp = rng.choice(np.array([1, 1, 1, 2, 3], np.uint8), n)
    ds = gp.Dataset.from_edges(n, e, x, lab, C, sp)
    ds.save(out)
    deg = np.diff(ds.graph()[0].astype(np.int64))
    print(f"{out}: {n} vertices, {len(e)} edges, degree max {deg.max()} median {int(np.median(deg))}")


if __name__ == "__main__":
    main()
