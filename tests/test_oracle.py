"""The oracle is pinned before it is trusted: it must reproduce the golden
vectors produced by running the unmodified reference (tests/golden/make_golden.py)
and the reference's own on-disk fixtures."""
import json

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, REFERENCE_SRC

CASES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem not in ("timedomain", "bins_count"))


def _load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_golden(case):
    g = _load(case)
    taper = g["taper"] if g["taper"].size else None
    mode = str(g["mode"]) if "mode" in g else "fixed"
    out, _ = O.compute(list(g["epochs"]), int(g["nfft"]), int(g["lo"]), int(g["hi"]), taper=taper, mode=mode)
    for m in O.METRICS:
        want = g["bins_" + m]
        if want.size == 0:
            assert out[m] is None, m
            continue
        got = out[m]["bins"]
        # restatement is operation-for-operation: allow only last-ulp noise
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14, err_msg=f"{case}/{m}")
        np.testing.assert_allclose(out[m]["band"], g["band_" + m], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(out["COHY"]["cband"], g["cband_COHY"], rtol=1e-12, atol=1e-14)


def test_zero_lag_exact_zeros():
    g = _load("zerolag_dead")
    out, _ = O.compute(list(g["epochs"]), int(g["nfft"]), int(g["lo"]), int(g["hi"]))
    # (0,1) and (0,2) are zero-lag scaled copies of channel 0: the reference's Im
    # flush (spectral.py:227-228) zeroes every phase-lag metric there.  Pair (1,2)
    # (0.7s vs 0.4s) sits on the flush threshold at low-power bins; see DESIGN.md.
    for p in (0, 1):
        for m in ("IMAGCOHY", "PLI", "WPLI", "DSWPLI"):
            assert np.all(out[m]["bins"][p] == 0.0), (m, p)


@pytest.mark.skipif(not (REFERENCE_SRC.parent / "frontend/tests/fixtures/threshold_coh.json").exists(),
                    reason="reference fixtures only present in the build container")
@pytest.mark.parametrize("metric", ["COH", "IMAGCOHY"])
def test_oracle_matches_reference_threshold_fixture(metric):
    """pkg/frontend/tests/fixtures/threshold_{coh,imagcohy}.json hold the normalised
    band-averaged network (pkg/scripts/export_threshold_fixtures.py:47-58)."""
    fx = json.loads((REFERENCE_SRC.parent / f"frontend/tests/fixtures/threshold_{metric.lower()}.json").read_text())
    edges = fx["network"]["edges"]
    want = np.array([e["w"] for e in edges])
    g = _load("sim2024_thresh")
    out, _ = O.compute(list(g["epochs"]), int(g["nfft"]), int(g["lo"]), int(g["hi"]), metrics=(metric,))
    w = out[metric]["band"]
    w = w / np.max(np.abs(w))
    np.testing.assert_allclose(w, want, rtol=1e-12, atol=1e-15)


def test_golden_sim_matches_reference_fixture_file():
    g = _load("sim2024_thresh")
    w = g["band_COH"] / np.max(np.abs(g["band_COH"]))
    p = REFERENCE_SRC.parent / "frontend/tests/fixtures/threshold_coh.json"
    if not p.exists():
        pytest.skip("reference fixtures only present in the build container")
    want = np.array([e["w"] for e in json.loads(p.read_text())["network"]["edges"]])
    np.testing.assert_array_equal(w, want)


def test_oracle_time_domain_matches_reference_golden():
    """COR / XCOR restatements vs the reference's compute_metric outputs (golden)."""
    g = np.load(GOLDEN / "timedomain.npz")
    eps = list(g["epochs"])
    w, dead = O.cor(eps)
    assert np.abs(w - g["cor_w"]).max() <= 1e-12
    assert [f"zero-variance channel {c}" for c in dead] == list(g["cor_warn"])
    for ml, key in ((10, "10"), (None, "all")):
        a, lags = O.xcor(eps, ml)
        assert np.abs(a - g["xcor_w_" + key]).max() <= 1e-12
        assert np.array_equal(lags, g["xcor_lag_" + key])


def test_oracle_bins_and_count_match_reference_golden():
    """accumulate_spectra with column subsets and a count=False back-fill (spectral.py:
    216-261): the oracle's fold replays tests/golden/bins_count.npz (made by the unmodified
    reference, make_golden_bins.py)."""
    g = np.load(GOLDEN / "bins_count.npz")
    spectra = g["spectra"]
    K, C, nb = spectra.shape
    acc = O.Sums(C, nb)
    for i in range(int(g["n_plan"])):
        b = g[f"plan_{i}_bins"]
        bins = None if (b.size == 1 and b[0] == -1) else b
        O.accumulate(acc, spectra[int(g[f"plan_{i}_trial"])], bins=bins, count=bool(g[f"plan_{i}_count"]))
    assert acc.n_trials_accumulated == int(g["n_trials"])
    for m, fn in O.BINS.items():
        np.testing.assert_allclose(fn(acc), g["bins_" + m], rtol=1e-12, atol=1e-12, err_msg=m)
