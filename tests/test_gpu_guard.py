"""The exact-sign guard at BASELINE scale, its negative control, and its
overflow safety (SURVEY.md section 7 hard part 1; reference spectral.py:227-239).

The phase-lag kernel computes t = Im(X_i conj X_j) in fp32; a (pair, bin) whose
smallest |t| over trials is inside the fp32 error bound is recomputed from the
fp64 spectrum ring with the reference's complex128 arithmetic (incl. the 1e-13
Im flush).  These tests check that claim where it matters:

* a 1024-node subset of config 5 (K=100, 6 bins: 3.1e8 updates, the scale at
  which unguarded fp32 sign flips were measured at a rate of ~4e-8) against the
  oracle with **no excluded entries**: K*PLI exactly, the rest within tolerance;
* the same run with the guard disabled (CSCONN_GUARD_G=0) must differ from the
  reference somewhere -- the test above is sensitive to sign flips;
* a guard work list that overflows (zero-lag copies of one channel: >5 % of
  the channels; and a forced capacity of 16 entries) loses no entry: every
  output matches the oracle through compute_metric and the batch path;
* K >= 2^17 trials (the packed 16-bit sign-count fields would wrap) still gives
  exact PLI counts.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200 import synth
from paper_2303_03279_b200.plan import compute_connectivity, make_taper

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3}


def _cfg5_subset(n=1024):
    """All 320 planted-cluster nodes of config 5 plus random others (sorted)."""
    c = synth.CONFIGS[5]
    planted = synth._planted(c)["nodes"].reshape(-1)
    rng = np.random.default_rng(2024)
    rest = np.setdiff1d(np.arange(c.N), planted)
    pick = np.concatenate([planted, rng.choice(rest, size=n - planted.size, replace=False)])
    return c, np.sort(pick)


@pytest.fixture(scope="module")
def cfg5_sub():
    c, idx = _cfg5_subset()
    x = synth.generate(c, "cuda")[:, torch.as_tensor(idx, device="cuda"), :].contiguous()
    sub = x.double().cpu().numpy()
    tp = make_taper(c.taper, min(c.T, c.nfft))[0]
    want, _ = O.compute(list(sub), c.nfft, c.lo, c.hi, c.metrics, taper=tp)
    return c, x, want


def _compare_all(c, out, want, K, metrics, exact_pli=True):
    """Every (pair, bin) entry and every band value, no exclusions."""
    for m in metrics:
        got = out[m]["bins"].T.cpu().numpy()
        ref = want[m]["bins"]
        assert got.shape == ref.shape, m
        err = np.abs(got - ref)
        assert err.max() <= TOL[m], f"{m}: max err {err.max():.3g} at {np.unravel_index(err.argmax(), err.shape)}"
        errb = np.abs(out[m]["band"].cpu().numpy() - want[m]["band"])
        assert errb.max() <= TOL[m], f"{m} band: max err {errb.max():.3g}"
    if exact_pli and "PLI" in metrics:
        kg = np.rint(out["PLI"]["bins"].T.cpu().numpy().astype(np.float64) * K)
        kr = np.rint(want["PLI"]["bins"] * K)
        assert np.array_equal(kg, kr), f"K*PLI differs at {int((kg != kr).sum())} entries"


def test_guard_at_baseline_scale_no_exclusions(cfg5_sub):
    c, x, want = cfg5_sub
    out, plan = compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=c.metrics, taper=c.taper)
    st = plan.guard_stats()
    n_upd = x.shape[1] * (x.shape[1] - 1) // 2 * c.n_bins * c.K
    assert n_upd >= 3e8
    assert st["flagged"] > 0, "the guard was never exercised"
    assert st["imag_handoff"], "the fused seven-metric call takes the IMAGCOHY hand-off"
    _compare_all(c, out, want, c.K, c.metrics)


def test_guard_negative_control(cfg5_sub):
    """With the guard factor at 0 only exact zeros go to fp64: fp32 sign flips must
    then show up as K*PLI mismatches -- proof the test above can see them."""
    c, x, want = cfg5_sub
    os.environ["CSCONN_GUARD_G"] = "0"
    try:
        out, plan = compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=("PLI",), taper=c.taper)
        torch.cuda.synchronize()
    finally:
        del os.environ["CSCONN_GUARD_G"]
    kg = np.rint(out["PLI"]["bins"].T.cpu().numpy().astype(np.float64) * c.K)
    kr = np.rint(want["PLI"]["bins"] * c.K)
    n_bad = int((kg != kr).sum())
    print(f"unguarded fp32: {n_bad} K*PLI mismatches in {kg.size} pair-bins x {c.K} trials")
    assert n_bad >= 1


def _zero_lag_epochs(K=30, N=400, T=256, n_copy=80, seed=5):
    """N channels of noise; channels 1..n_copy are scaled copies of channel 0 (zero
    lag: every pair among them has Im CSD at rounding level in every bin)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((K, N, T))
    gains = rng.uniform(0.5, 2.0, n_copy)
    x[:, 1:n_copy + 1] = gains[None, :, None] * x[:, :1]
    return x


def test_guard_list_overflow_through_compute_metric():
    """> 5 % zero-lag copies: 3240 pairs x 100 bins flagged, more than the list holds
    (cap = max(2^16, P nb / 64) = 124687): the overflow records carry the rest."""
    from paper_2303_03279_b200 import EpochMatrix, FrequencyBand, MetricId, compute_metric
    K, N, T, nfft, lo, hi = 30, 400, 256, 256, 10, 109
    x = _zero_lag_epochs(K, N, T)
    want, _ = O.compute(list(x), nfft, lo, hi, ("PLI", "WPLI", "IMAGCOHY"))
    eps = [EpochMatrix(e, 256.0) for e in x]
    band = FrequencyBand(lo, hi, 1.0)
    for m in ("PLI", "WPLI", "IMAGCOHY"):
        net = compute_metric(eps, MetricId.parse(m), nfft, band=band)
        err = np.abs(np.asarray(net.weights) - want[m]["band"])
        assert err.max() <= TOL[m], f"{m}: max err {err.max():.3g}"
    # the same data through the batch path: overflow records used, every entry exact
    xt = torch.tensor(x, device="cuda")
    out, plan = compute_connectivity(xt, nfft, lo, hi, metrics=("PLI", "USPLI", "WPLI", "DSWPLI", "IMAGCOHY"))
    st = plan.guard_stats()
    assert st["flagged"] >= 80 * 81 // 2 * (hi - lo + 1) and st["records"] > 0, st
    want, _ = O.compute(list(x), nfft, lo, hi, ("PLI", "USPLI", "WPLI", "DSWPLI", "IMAGCOHY"))
    _compare_all(None, out, want, K, ("PLI", "USPLI", "WPLI", "DSWPLI", "IMAGCOHY"))
    # zero-lag pairs: the reference's exact zeros (spectral.py:227-228 flush)
    i, j = np.triu_indices(N, 1)
    zl = (i <= 80) & (j <= 80)
    assert np.all(out["PLI"]["bins"].T.cpu().numpy()[zl] == 0.0)
    assert np.all(out["WPLI"]["bins"].T.cpu().numpy()[zl] == 0.0)


def test_imag_handoff_exact_zeros_and_overflow():
    """The fused seven-metric call: per-bin IMAGCOHY from the tensor-core kernel, the
    phase-lag kernel reads it; zero-lag copies (guard-flagged, > the list capacity) get
    the reference's exact zeros for IMAGCOHY as well, and every entry matches."""
    K, N, T, nfft, lo, hi = 30, 400, 256, 256, 10, 109
    x = _zero_lag_epochs(K, N, T)
    out, plan = compute_connectivity(torch.tensor(x, device="cuda"), nfft, lo, hi, metrics=SEVEN)
    st = plan.guard_stats()
    assert st["imag_handoff"] and st["records"] > 0, st
    want, _ = O.compute(list(x), nfft, lo, hi, SEVEN)
    _compare_all(None, out, want, K, SEVEN)
    i, j = np.triu_indices(N, 1)
    zl = (i <= 80) & (j <= 80)
    for m in ("IMAGCOHY", "PLI", "WPLI"):
        assert np.all(out[m]["bins"].T.cpu().numpy()[zl] == 0.0), m


SEVEN = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


@pytest.mark.parametrize("metrics", [("PLI", "USPLI", "WPLI", "DSWPLI", "IMAGCOHY"), ("PLI",), ("WPLI",), SEVEN])
def test_guard_forced_tiny_list(metrics):
    """A 16-entry work list (CSCONN_FLAG_CAP, read at plan creation): nearly every
    flagged entry goes through an overflow record; outputs still match exactly."""
    K, N, T, nfft, lo, hi = 12, 150, 128, 128, 3, 40
    x = _zero_lag_epochs(K, N, T, n_copy=12, seed=11)
    x[:, 100] = 0.0                                       # a dead channel as well
    os.environ["CSCONN_FLAG_CAP"] = "16"
    try:
        out, plan = compute_connectivity(torch.tensor(x, device="cuda"), nfft, lo, hi, metrics=metrics,
                                         taper="hann")
        st = plan.guard_stats()
    finally:
        del os.environ["CSCONN_FLAG_CAP"]
    assert st["records"] > 0, st
    assert st["imag_handoff"] == (metrics == SEVEN), st
    want, _ = O.compute(list(x), nfft, lo, hi, metrics, taper=np.hanning(T))
    _compare_all(None, out, want, K, metrics)


def test_trial_count_beyond_packed_sign_fields():
    """K = 140000 > 2^17: the per-stage decode of the packed sign counts."""
    K, N, T, nfft, lo, hi = 140_000, 12, 16, 16, 1, 2
    rng = np.random.default_rng(3)
    x = rng.standard_normal((K, N, T))
    # node 0 = node 1 delayed by one sample: Im CSD < 0 in (nearly) every trial, so each
    # 16-bit field would count ~70000 negatives without the wide decode
    x[:, 0] = np.roll(x[:, 1], 1, axis=-1) + 0.1 * x[:, 0]
    metrics = ("PLI", "USPLI", "WPLI")
    out, plan = compute_connectivity(torch.tensor(x, device="cuda"), nfft, lo, hi, metrics=metrics)
    want, _ = O.compute(list(x), nfft, lo, hi, metrics)
    _compare_all(None, out, want, K, metrics)
    assert float(want["PLI"]["bins"][0].min()) > 0.95     # the coupled pair's negative counts exceed 2^16


@pytest.mark.parametrize("cfg", [1, 2])
def test_full_config_against_oracle(cfg):
    """Configs 1 and 2 in full (every pair, every bin), no exclusions."""
    c = synth.CONFIGS[cfg]
    x = synth.generate(c, "cuda")
    out, plan = compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=c.metrics, taper=c.taper)
    tp = make_taper(c.taper, min(c.T, c.nfft))[0]
    want, _ = O.compute(list(x.double().cpu().numpy()), c.nfft, c.lo, c.hi, c.metrics, taper=tp)
    _compare_all(c, out, want, c.K, c.metrics)
