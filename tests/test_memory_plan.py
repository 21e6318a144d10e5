"""Device memory plan (gp_stage_footprint: the engine's own stash layout pass plus graph,
features and labels; no GPU needed). BASELINE.json configs[3] (products, 64-layer GCNII) and
configs[4] (10 M-vertex hybrid, 4 stages x 2 partitions, 32-layer GCNII) must fit one B200
(179 GiB usable) per stage / worker under the default lean layout."""
import pytest

B200_BYTES = 179 * 2**30


def _worst(gp, monkeypatch, lean, N, nnz, F, C, H, L, S, K, G=1):
    monkeypatch.setenv("GP_LEAN", lean)
    monkeypatch.setenv("GP_MERGED_G", lean)
    specs = gp.build_layer_specs(gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=L, hidden=H), F, C)
    ranges = gp.make_stage_assignment(L, S)
    return max(gp.stage_footprint(nnz_norm=nnz, num_features=F, specs=specs, num_vertices=N, num_chunks=K, stage=s,
                                  num_stages=S, layer_range=ranges[s], hidden=H, num_classes=C, dropout=0.5, seed=1,
                                  group_size=G, group_rank=0)
               for s in range(S))


REDDIT = dict(N=232965, nnz=114615892 + 232965, F=602, C=41, H=100, L=64)
PRODUCTS = dict(N=2449029, nnz=123718280 + 2449029, F=100, C=47, H=128, L=64)
POWERLAW10M = dict(N=10_000_000, nnz=400_000_000 + 10_000_000, F=128, C=64, H=128, L=32)


def test_reddit_headline_footprint(gp, monkeypatch):
    # the round-1 swap layout measured 41.7 GiB on the device (bench.py stage_stash_gib), without
    # the per-epoch done-filtered backward CSR (8 B per entry, 0.86 GiB here) it did not have
    monkeypatch.setenv("GP_BWD_CSR", "0")
    swap = _worst(gp, monkeypatch, "0", S=1, K=4, **REDDIT)
    assert abs(swap / 2**30 - 41.7) < 0.1
    monkeypatch.delenv("GP_BWD_CSR")
    lean = _worst(gp, monkeypatch, "1", S=1, K=4, **REDDIT)
    assert lean < 0.62 * swap
    monkeypatch.setenv("GP_BWD_CSR", "0")
    assert 0.8 * 2**30 < lean - _worst(gp, monkeypatch, "1", S=1, K=4, **REDDIT) < 0.9 * 2**30


@pytest.mark.parametrize("S", [2, 4, 8])
def test_products_64_layers_fits_from_two_stages(gp, monkeypatch, S):
    assert _worst(gp, monkeypatch, "1", S=S, K=4 * S, **PRODUCTS) < B200_BYTES
    if S == 2:  # the swap layout needs four stages
        assert _worst(gp, monkeypatch, "0", S=S, K=4 * S, **PRODUCTS) > B200_BYTES


def test_powerlaw_hybrid_worker_fits(gp, monkeypatch):
    """configs[4]: a 4 x 2 hybrid worker under 180 GB (decimal): lean stashes with full-N rows for
    the tables halos land in, owner rows only for pre / h0 / dh0 / the chunk gradients."""
    assert _worst(gp, monkeypatch, "1", S=4, K=16, G=2, **POWERLAW10M) < 180e9
    assert _worst(gp, monkeypatch, "0", S=4, K=16, G=2, **POWERLAW10M) > B200_BYTES


def test_footprint_rejects_bad_config(gp):
    specs = gp.build_layer_specs(gp.ModelConfig(kind=gp.ModelKind.GCN, layers=3, hidden=16), 8, 4)
    with pytest.raises(gp.InvalidArgument):
        gp.stage_footprint(nnz_norm=10, num_features=8, specs=specs, num_vertices=10, num_chunks=65, stage=0,
                           num_stages=1, layer_range=(0, 3), hidden=16, num_classes=4, dropout=0.5, seed=1)
