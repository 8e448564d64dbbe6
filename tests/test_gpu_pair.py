"""The CTA-pair tensor-core kernel (k_pairs_tc<true>: clusters of two CTAs, one
M = 256 x N = 128 cta_group::2 MMA per hi/lo product giving D_re and D_im together).

It is chosen per launch when the row range gives every SM pair two 256 x 64 tiles
and no more masked rows than 128 x 64 single-CTA tiles (config 5 on one GPU);
CSCONN_K2_PAIR=1 forces it on small shapes so the ragged edges (partial tiles, the
diagonal, N not a multiple of 64 / 256, odd K, multitaper, row-range shards) are
checked against the oracle, and CSCONN_K2_PAIR=0 gives the single-CTA kernel for a
like-for-like comparison.
Reference: spectral.py:204-241 (CSD and unit-phasor sums), metrics.py:32-56, 115-134.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200.plan import DevicePlan, compute_connectivity, make_taper, pow2_scale
from paper_2303_03279_b200.shard import shard_plan

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3}
SEVEN = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


class _pairs:
    def __init__(self, v):
        self.v = v

    def __enter__(self):
        self.old = os.environ.get("CSCONN_K2_PAIR")
        os.environ["CSCONN_K2_PAIR"] = self.v

    def __exit__(self, *exc):
        if self.old is None:
            del os.environ["CSCONN_K2_PAIR"]
        else:
            os.environ["CSCONN_K2_PAIR"] = self.old


def _epochs(K, N, T, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((K, N, T))
    x[:, 7] = 0.6 * x[:, 2]            # zero-lag copy (exact zeros, guard path)
    x[:, N // 2] = 0.0                 # dead node
    t = np.arange(T)
    for c in range(20, 30):            # a phase-lagged cluster
        x[:, c] += 0.8 * np.sin(2 * np.pi * 0.07 * t[None, :] + 0.3 * c + rng.uniform(0, 6.3, (K, 1)))
    return x


def _check(out, want, metrics, K):
    for m in metrics:
        got = out[m]["bins"].T.cpu().numpy()
        if m == "COHY":
            assert np.abs(got - want[m]["bins"]).max() <= 1e-4, "COHY"
            assert np.abs(out[m]["band"].cpu().numpy() - want[m]["cband"]).max() <= 1e-4, "COHY band"
            continue
        err = np.abs(got - want[m]["bins"])
        assert err.max() <= TOL[m], f"{m}: max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
        errb = np.abs(out[m]["band"].cpu().numpy() - want[m]["band"])
        assert errb.max() <= TOL[m], f"{m} band: max err {errb.max():.3g}"
    if "PLI" in metrics:
        kg = np.rint(out["PLI"]["bins"].T.cpu().numpy().astype(np.float64) * K)
        assert np.array_equal(kg, np.rint(want["PLI"]["bins"] * K))


@pytest.mark.parametrize("K,N,T,nfft,lo,hi,metrics", [
    (37, 300, 200, 256, 5, 20, SEVEN),                       # ragged N, odd K, the fused call
    (16, 513, 128, 128, 3, 9, ("COH", "COHY", "PLV")),       # exactly one K chunk, N = 2 * 256 + 1
    (20, 257, 160, 256, 2, 12, ("IMAGCOHY",)),               # IMAGCOHY from D_im with the exact-zero guard
    (50, 130, 100, 128, 1, 30, ("COH", "PLV", "PLI", "WPLI")),
])
def test_forced_pairs_against_oracle(K, N, T, nfft, lo, hi, metrics):
    x = _epochs(K, N, T, seed=K + N)
    with _pairs("1"):
        out, plan = compute_connectivity(torch.tensor(x, device="cuda"), nfft, lo, hi, metrics=metrics,
                                         taper="hann")
        torch.cuda.synchronize()
    want, _ = O.compute(list(x), nfft, lo, hi, metrics, taper=np.hanning(T))
    _check(out, want, metrics, K)


def test_forced_pairs_multitaper_against_oracle():
    """DPSS L = 3: the contraction runs over trials x tapers (K L = 54, 4 chunks of 16)."""
    K, N, T, nfft, lo, hi = 18, 270, 150, 256, 4, 15
    x = _epochs(K, N, T, seed=3)
    taper = ("dpss", 2.0, 3)
    metrics = ("COH", "IMAGCOHY", "PLV", "PLI", "WPLI")
    with _pairs("1"):
        out, plan = compute_connectivity(torch.tensor(x, device="cuda"), nfft, lo, hi, metrics=metrics, taper=taper)
        torch.cuda.synchronize()
    tp = make_taper(taper, min(T, nfft))
    want, _ = O.compute(list(x), nfft, lo, hi, metrics, taper=tp)
    _check(out, want, metrics, K)


def test_forced_pairs_row_shards():
    """Row-range shards (the multi-GPU split) with CTA pairs: concatenated shard outputs
    equal the single-CTA run of the whole pair space."""
    K, N, T, nfft, lo, hi = 21, 600, 128, 128, 2, 8
    x = torch.tensor(_epochs(K, N, T, seed=8), device="cuda", dtype=torch.float32)
    metrics = ("COH", "COHY", "PLV")
    with _pairs("0"):
        ref, plan = compute_connectivity(x, nfft, lo, hi, metrics=metrics)
    slots = torch.arange(K, dtype=torch.int32, device="cuda")
    world = 3
    with _pairs("1"):
        parts = []
        for r in range(world):
            (rb, re), (p0, p1) = shard_plan(N, world, r)
            parts.append(plan.pair_metrics(slots, metrics, row_tiles=(rb, re), pair_base=p0, pair_count=p1 - p0))
        torch.cuda.synchronize()
    for m in metrics:
        got = torch.cat([p[m]["bins"] for p in parts], dim=-1)
        want = ref[m]["bins"]
        assert got.shape == want.shape, m
        assert float((got - want).abs().max()) <= 2e-6, m
        gotb = torch.cat([p[m]["band"] for p in parts], dim=0)
        assert float((gotb - ref[m]["band"]).abs().max()) <= 2e-6, m


def test_default_pairs_match_single_cta_at_scale():
    """N = 2600: every per-bin and band value of COH / COHY / PLV /
    IMAGCOHY identical to the single-CTA kernel's (IMAGCOHY band means up to the order of
    the fp64 fallback's atomic adds), and a node subset against the oracle."""
    K, N, T, nfft, lo, hi = 24, 2600, 96, 128, 3, 6
    rng = np.random.default_rng(12)
    xh = rng.standard_normal((K, N, T)).astype(np.float32)
    xh[:, 2500] = 0.9 * xh[:, 11]
    x = torch.tensor(xh, device="cuda")
    metrics = ("COH", "COHY", "PLV", "IMAGCOHY")
    scale = pow2_scale(float(x.abs().amax()), T)
    plan = DevicePlan(N, T, nfft, lo, hi, slot_capacity=K, device="cuda", scale=scale)
    plan.spectra(x, 0)
    slots = torch.arange(K, dtype=torch.int32, device="cuda")
    with _pairs("0"):
        one = plan.pair_metrics(slots, metrics)
    with _pairs("1"):
        two = plan.pair_metrics(slots, metrics)
    torch.cuda.synchronize()
    for m in metrics:
        d = float((one[m]["bins"] - two[m]["bins"]).abs().max())
        db = float((one[m]["band"] - two[m]["band"]).abs().max())
        # same products in the same accumulation order per element: bit-identical per bin;
        # band means of IMAGCOHY get the fp64 fallback's atomics (order-dependent last bits)
        assert d == 0.0 and db <= (1e-6 if m == "IMAGCOHY" else 0.0), (m, d, db)
    sub = np.array([0, 1, 11, 255, 256, 257, 511, 1024, 2047, 2500, 2599])
    want, _ = O.compute(list(xh[:, sub].astype(np.float64)), nfft, lo, hi, ("COH", "PLV", "IMAGCOHY"))
    ii, jj = np.triu_indices(len(sub), 1)
    gi, gj = sub[ii], sub[jj]
    pidx = gi * (2 * N - gi - 1) // 2 + (gj - gi - 1)
    for m in ("COH", "PLV", "IMAGCOHY"):
        got = two[m]["bins"].cpu().numpy()[:, pidx].T
        assert np.abs(got - want[m]["bins"]).max() <= TOL[m], m
