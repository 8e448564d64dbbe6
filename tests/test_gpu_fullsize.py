"""Parity at BASELINE.json's full sizes.

Every (pair, bin) output depends only on its two nodes (spectral.py:204-241), so
the oracle is exact on node subsets: each config runs whole on
the GPU and is compared, on a subset of nodes that includes planted-coupling
nodes, with the pinned oracle run on just those nodes' samples.  Over all
P x nb entries the domain's size-independent identities are checked: value
ranges, DSWPLI = WPLI^2, USPLI = (K PLI^2 - 1)/(K - 1), K PLI an integer,
|IMAGCOHY| <= COH, band = mean of the per-bin values; and sharded row ranges
reproduce the single run (the multi-GPU partition).  Tolerances: north_star.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200 import synth
from paper_2303_03279_b200.plan import SEVEN, compute_connectivity, make_taper, row_tile_range

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3}


def _subset(c, rng, n_rand=24):
    tab = synth._planted(c)
    planted = np.asarray(tab.get("nodes", tab.get("pairs", []))).reshape(-1)
    pick = set(rng.choice(c.N, size=min(n_rand, c.N), replace=False).tolist())
    pick.update(planted[: min(8, planted.size)].tolist())
    pick.update([0, c.N - 1])                      # first and last rows / columns of the tiling
    return np.array(sorted(pick))


def _pair_index(idx, N):
    a, b = np.triu_indices(len(idx), 1)
    i, j = idx[a], idx[b]
    return i * (N - 1) - i * (i - 1) // 2 + (j - i - 1)


def _taper_for_oracle(c):
    tp = make_taper(c.taper, min(c.T, c.nfft))
    return None if tp is None else (tp[0] if tp.shape[0] == 1 else tp)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_size_subset_parity_and_identities(cfg):
    c = synth.CONFIGS[cfg]
    metrics = c.metrics
    x = synth.generate(c, "cuda")                 # cfg4: the first 50-trial window of the stream
    out, plan = compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=metrics, taper=c.taper)
    K, nb = c.K, c.n_bins

    # ---- identities over all P x nb entries ----
    g = {m: out[m]["bins"] for m in metrics}
    for m in metrics:
        assert bool(torch.isfinite(g[m]).all()), m
        if m in ("COH", "PLV", "PLI", "WPLI", "DSWPLI"):
            assert float(g[m].min()) >= -1e-6 and float(g[m].max()) <= 1 + 1e-5, m
        band_from_bins = g[m].double().mean(0)
        assert float((band_from_bins - out[m]["band"].double()).abs().max()) <= 2e-6, m
    if "WPLI" in g and "DSWPLI" in g:
        assert float((g["DSWPLI"] - g["WPLI"] ** 2).abs().max()) <= 2e-6
    if "PLI" in g:
        kp = g["PLI"].double() * K
        assert float((kp - kp.round()).abs().max()) <= 1e-3 * K
        if "USPLI" in g:
            want = (K * g["PLI"].double() ** 2 - 1) / (K - 1)
            assert float((g["USPLI"].double() - want).abs().max()) <= 1e-5
    if "IMAGCOHY" in g and "COH" in g:
        assert float((g["IMAGCOHY"].abs() - g["COH"]).max()) <= 1e-5

    # ---- node-subset parity against the oracle ----
    rng = np.random.default_rng(1000 + cfg)
    idx = _subset(c, rng)
    sub = x[:, torch.as_tensor(idx, device="cuda"), :].double().cpu().numpy()
    tp = _taper_for_oracle(c)
    want, _ = O.compute(list(sub), c.nfft, c.lo, c.hi, metrics, taper=tp)
    masks = O.well_conditioned(list(sub), c.nfft, c.lo, c.hi, metrics, TOL, taper=tp, ref=want)
    sens = O.flush_sensitive(list(sub), c.nfft, c.lo, c.hi, taper=tp)
    pidx = torch.as_tensor(_pair_index(idx, c.N), device="cuda")
    for m in metrics:
        got = g[m][:, pidx].T.cpu().numpy()       # [p, nb] reference layout
        keep = masks[m] & ~sens
        # non-adversarial data: every entry is well conditioned, none is excluded
        assert keep.all(), f"cfg{cfg}/{m}: {np.size(keep) - keep.sum()} ill-conditioned entries"
        err = np.where(keep, np.abs(got - want[m]["bins"]), 0.0)
        assert err.max() <= TOL[m], f"cfg{cfg}/{m}: max err {err.max():.3g}"
        kb = keep.all(axis=1)
        errb = np.abs(out[m]["band"][pidx].cpu().numpy() - want[m]["band"])[kb]
        assert errb.max() <= TOL[m], f"cfg{cfg}/{m} band: max err {errb.max():.3g}"


@pytest.mark.parametrize("cfg,shards", [(2, 3), (3, 4)])
def test_sharded_row_ranges_reproduce_the_single_run(cfg, shards):
    """The multi-GPU partition (cs_row_tile_range) run shard by shard on one GPU:
    the concatenated per-bin outputs are identical to the single run."""
    c = synth.CONFIGS[cfg]
    x = synth.generate(c, "cuda")
    full, plan = compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=c.metrics, taper=c.taper)
    slots = torch.arange(c.K, dtype=torch.int32, device="cuda")
    for s in range(shards):
        (rb, re), (p0, p1) = row_tile_range(c.N, shards, s)
        o = plan.pair_metrics(slots, c.metrics, 0, c.n_bins, row_tiles=(rb, re), pair_base=p0, pair_count=p1 - p0)
        for m in c.metrics:
            assert torch.equal(o[m]["bins"], full[m]["bins"][:, p0:p1]), (s, m)
            assert float((o[m]["band"] - full[m]["band"][p0:p1]).abs().max()) <= 1e-6, (s, m)


def test_pair_space_beyond_int32():
    """N = 65600 nodes: P = 2,151,657,200 pairs, so pair offsets past 2^31 (and
    i * i past 2^31 from i = 46341 on) must be 64-bit everywhere on the path.  Band
    outputs of a K2 and a K3 metric each; nodes whose pairs straddle the 2^31 pair
    index are checked against the oracle on just those nodes."""
    N, K, T, nfft, lo, hi = 65600, 4, 32, 32, 3, 4
    P = N * (N - 1) // 2
    assert P > 2 ** 31
    gen = torch.Generator(device="cuda").manual_seed(77)
    x = torch.randn((K, N, T), generator=gen, device="cuda", dtype=torch.float32)
    metrics = ("COH", "PLV", "PLI", "WPLI")
    out, plan = compute_connectivity(x, nfft, lo, hi, metrics=metrics, per_bin=False, band=True)
    idx = np.array([0, 1, 32767, 46340, 46341, 65534, 65535, 65536, 65597, 65598, 65599])
    pidx = _pair_index(idx, N)
    assert pidx.max() == P - 1 and (pidx > 2 ** 31).any()
    sub = x[:, torch.as_tensor(idx, device="cuda"), :].double().cpu().numpy()
    want, _ = O.compute(list(sub), nfft, lo, hi, metrics)
    masks = O.well_conditioned(list(sub), nfft, lo, hi, metrics, TOL, ref=want)
    tp = torch.as_tensor(pidx, device="cuda")
    for m in metrics:
        got = out[m]["band"][tp].cpu().numpy()
        keep = masks[m].all(axis=1)
        assert keep.mean() > 0.9, m
        err = np.abs(got - want[m]["band"])[keep]
        assert err.max() <= TOL[m], f"{m}: max err {err.max():.3g}"
        tail = out[m]["band"][-4_000_000:]          # the last rows of the pair space
        assert bool(torch.isfinite(tail).all()) and float(tail.min()) >= -1e-6 and float(tail.max()) <= 1 + 1e-5, m
