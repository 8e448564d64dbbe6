"""The incremental online window (csrc/window.cu, plan.IncrementalWindow) against the
oracle over a stream: running sums moved by the entering / leaving trials only must
give, window after window, the reference's metrics over exactly the window's trials
(pipeline.py:304-309 + metrics.py:450-460 re-fold them all)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2303_03279_b200.core import ParameterError
from paper_2303_03279_b200.plan import DevicePlan, IncrementalWindow, WindowGraph, pow2_scale

pytestmark = pytest.mark.gpu
TOL = {"COH": 1e-4, "IMAGCOHY": 1e-4, "PLV": 1e-4, "PLI": 1e-3, "USPLI": 1e-3, "WPLI": 1e-3, "DSWPLI": 1e-3}
SIX = ("COH", "IMAGCOHY", "PLV", "PLI", "USPLI", "WPLI", "DSWPLI")


def _stream(n, N, T, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, N, T))
    x[:, 7] += 0.6 * np.roll(x[:, 3], 2, axis=-1)      # a lagged coupling
    x[9:16, 1] = 0.5 * x[9:16, 0]                       # zero-lag copies in some trials only: the
    x[20:23, 60] = 0.0                                  # guard count enters and leaves the window
    return x.astype(np.float32)


@pytest.mark.parametrize("resync", [256, 4])
@pytest.mark.parametrize("taper", ["hann", None])
def test_incremental_window_matches_oracle(resync, taper):
    win, new, N, T, nfft, lo, hi = 12, 3, 150, 128, 128, 3, 20
    n_up = 13                                          # (12 + 3) / 3 = 5 ring phases, wrapped twice
    x = _stream(win + new * n_up, N, T, seed=17)
    xt = torch.tensor(x, device="cuda")
    scale = pow2_scale(float(np.abs(x).max()), min(T, nfft))
    plan = DevicePlan(N, T, nfft, lo, hi, taper=taper, slot_capacity=win + new, device="cuda", scale=scale)
    iw = IncrementalWindow(plan, win, new, SIX, resync_every=resync)
    iw.prime(xt[:win])
    tp = None if taper is None else np.hanning(T)
    for u in range(1, n_up + 1):
        got = iw.update(xt[win + new * (u - 1): win + new * u])
        if u in (1, 3, 4, 5, 8, 13):
            want, _ = O.compute(list(x[new * u: new * u + win].astype(np.float64)), nfft, lo, hi, SIX, taper=tp)
            for m in SIX:
                e = np.abs(got[m]["bins"].T.cpu().numpy() - want[m]["bins"]).max()
                eb = np.abs(got[m]["band"].cpu().numpy() - want[m]["band"]).max()
                assert max(e, eb) <= TOL[m], f"update {u} {m}: {e:.3g} / {eb:.3g}"
            kp = np.rint(got["PLI"]["bins"].T.cpu().numpy().astype(np.float64) * win)
            assert np.array_equal(kp, np.rint(want["PLI"]["bins"] * win)), f"update {u}: K*PLI"
    assert len(iw._graphs) >= 4


def test_incremental_equals_full_recompute_window():
    """The same stream through WindowGraph (full re-fold per update, the reference's
    rebuild_last semantics) and IncrementalWindow: equal within fp32 summation order."""
    win, new, N, T, nfft, lo, hi = 10, 2, 90, 100, 128, 2, 14
    n_up = 9
    x = torch.tensor(_stream(win + new * n_up, N, T, seed=23), device="cuda")
    scale = pow2_scale(float(x.abs().max()), min(T, nfft))
    pf = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win, device="cuda", scale=scale)
    pi = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=win + new, device="cuda", scale=scale)
    wg = WindowGraph(pf, new, ("PLV", "WPLI"))
    iw = IncrementalWindow(pi, win, new, ("PLV", "WPLI"))
    wg.prime(x[:win])
    iw.prime(x[:win])
    for u in range(1, n_up + 1):
        a = wg.update(x[win + new * (u - 1): win + new * u])
        b = iw.update(x[win + new * (u - 1): win + new * u])
        for m in ("PLV", "WPLI"):
            for part in ("bins", "band"):
                np.testing.assert_allclose(b[m][part].cpu().numpy(), a[m][part].cpu().numpy(), rtol=0,
                                           atol=2e-5, err_msg=f"{m} {part} update {u}")


def test_incremental_window_rejects():
    plan = DevicePlan(20, 64, 64, 1, 5, slot_capacity=10, device="cuda")
    with pytest.raises(ParameterError):
        IncrementalWindow(plan, 10, 2)                  # ring too small for window + n_new
    plan2 = DevicePlan(20, 64, 64, 1, 5, slot_capacity=12, device="cuda")
    with pytest.raises(ParameterError):
        IncrementalWindow(plan2, 10, 2, ("COHY",))      # complex output: full path only
