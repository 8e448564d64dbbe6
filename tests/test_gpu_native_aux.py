"""The hand-written kernels around the spectral path
against the oracle at sizes that cross their tile boundaries: COR / XCOR on the
fp64 tensor cores (csrc/timedomain.cu), the source projection and apply_inverse
GEMM engine and the streaming FIR (csrc/upstream.cu)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200 import EpochMatrix, MetricId, compute_metric

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3}


def _epochs(K=4, C=70, T=300, seed=5):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((K, C, T))
    x[:, 9] = np.roll(x[:, 2], 5, axis=-1) + 0.05 * x[:, 9]     # y lags x by 5 samples
    x[:, min(40, C - 2)] = np.roll(x[:, 33], -3, axis=-1)       # x lags y
    x[:, min(60, C - 1)] = 2.5                                   # constant channel: (0, 0) / dead
    return x


@pytest.mark.parametrize("max_lag", [0, 1, 7, 299])
def test_xcor_kernel_matches_oracle(max_lag):
    # all 599 lags: one trial of 36 channels (the oracle is a Python loop over lags)
    x = _epochs() if max_lag < 299 else _epochs(K=1, C=36)
    eps = [EpochMatrix(e, 100.0, trial_index=k) for k, e in enumerate(x)]
    net = compute_metric(eps, MetricId.XCOR, 64, max_lag=max_lag)
    w, lags = O.xcor(list(x), max_lag)
    assert np.abs(np.asarray(net.weights) - w).max() <= 1e-12
    assert np.array_equal(np.asarray(net.lags), lags)


def test_cor_kernel_matches_oracle():
    x = _epochs(K=6, C=100, T=257, seed=6)
    eps = [EpochMatrix(e, 100.0, trial_index=k) for k, e in enumerate(x)]
    net = compute_metric(eps, MetricId.COR, 64)
    w, dead = O.cor(list(x))
    assert np.abs(np.asarray(net.weights) - w).max() <= 1e-12
    assert any("60" in s for s in net.warnings)


def test_fir_long_taps_streaming():
    from paper_2303_03279_b200.upstream import OverlapAddFilter
    rng = np.random.default_rng(7)
    for n_taps in (1, 5, 1500):
        taps = rng.standard_normal(n_taps)
        sig = rng.standard_normal((5, 3000))
        want = np.stack([np.convolve(s, taps)[:3000] for s in sig])
        f = OverlapAddFilter(taps)
        cuts = [0, 17, 400, 401, 2100, 3000]      # blocks shorter and longer than the taps
        got = np.concatenate([f.process(sig[:, a:b]).cpu().numpy() for a, b in zip(cuts, cuts[1:])], 1)
        np.testing.assert_allclose(got, want, atol=1e-9, err_msg=str(n_taps))


def test_projection_and_apply_inverse_across_tiles():
    from paper_2303_03279_b200.upstream import apply_inverse, source_connectivity
    rng = np.random.default_rng(8)
    K, C, T, Ns, nfft, lo, hi = 5, 40, 200, 150, 256, 5, 30
    x = rng.standard_normal((K, C, T))
    Mx = rng.standard_normal((Ns, C)) / np.sqrt(C)
    ep = EpochMatrix(x[0], 100.0, trial_index=2)
    np.testing.assert_allclose(apply_inverse(Mx, ep).data.cpu().numpy(), Mx @ x[0], atol=1e-11)
    out, _ = source_connectivity(torch.tensor(x, device="cuda"), Mx, nfft, lo, hi, taper="hann")
    want, _ = O.compute([Mx @ e for e in x], nfft, lo, hi, taper=np.hanning(T))
    for m in ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI"):
        err = np.abs(out[m]["bins"].T.cpu().numpy() - want[m]["bins"]).max()
        assert err <= TOL[m], (m, err)
