"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this GPU
pool: profiles/r2_compute_sanitizer_closed.txt).

Every output buffer is a view into a larger allocation whose guard regions are
filled with a sentinel; after the kernels run, the guard regions must be
untouched and -- for row-tile shards -- nothing outside the shard's pair range
may be written.  Shapes cover ragged tiles (N not a multiple of 64), odd and even
trial counts, one and many bins, multitaper, and the spectrum ring's slot range.
"""
import numpy as np
import pytest
import torch

from paper_2303_03279_b200.plan import SEVEN, DevicePlan, pow2_scale, row_tile_range

pytestmark = pytest.mark.gpu
GUARD = 4099          # sentinel elements on each side (odd on purpose)
SENT = 12345.678


def _guarded(n, dtype, dev):
    big = torch.full((n + 2 * GUARD,), SENT, dtype=dtype, device=dev)
    return big, big[GUARD:GUARD + n]


def _check_guards(big, n, what):
    lo, hi = big[:GUARD], big[GUARD + n:]
    assert bool((lo == SENT).all()) and bool((hi == SENT).all()), f"{what}: write outside the buffer"


@pytest.mark.parametrize("N,K,T,nfft,lo,hi,taper", [
    (70, 9, 100, 128, 3, 9, "hann"),         # ragged tile, odd K
    (129, 12, 64, 64, 0, 32, None),           # DC and Nyquist bins, 3 ragged row tiles
    (200, 7, 256, 256, 20, 20, ("dpss", 2.0, 3)),  # one bin, multitaper
    (64, 2, 32, 32, 1, 15, "hann"),           # exactly one tile
])
@pytest.mark.parametrize("shards", [1, 3])
def test_outputs_stay_inside_their_buffers(N, K, T, nfft, lo, hi, taper, shards):
    rng = np.random.default_rng(N + K)
    dev = torch.device("cuda")
    x = torch.tensor(rng.standard_normal((K, N, T)), dtype=torch.float32, device=dev)
    x[:, 1] = 0.5 * x[:, 0]                     # guard-flagged pairs -> fp64 fallback writes
    plan = DevicePlan(N, T, nfft, lo, hi, taper=taper, slot_capacity=K, device=dev,
                      scale=pow2_scale(float(x.abs().max()), min(T, nfft)))
    plan.spectra(x, 0)
    nb = hi - lo + 1
    metrics = SEVEN + ("COHY",)
    slots = torch.arange(K, dtype=torch.int32, device=dev)
    P = N * (N - 1) // 2
    full = plan.pair_metrics(slots, metrics)
    for s in range(shards):
        (rb, re), (p0, p1) = row_tile_range(N, shards, s)
        n = p1 - p0
        if n == 0:              # more shards than row tiles: an empty shard launches nothing
            continue
        outs, bigs = {}, {}
        for m in metrics:
            dt = torch.complex64 if m == "COHY" else torch.float32
            bb, vb = _guarded(nb * n, dt, dev)
            bd, vd = _guarded(n, dt, dev)
            outs[m] = {"bins": vb.view(nb, n), "band": vd}
            bigs[m] = (bb, bd)
        plan.pair_metrics(slots, metrics, outputs=outs, row_tiles=(rb, re), pair_base=p0, pair_count=n)
        torch.cuda.synchronize()
        for m in metrics:
            _check_guards(bigs[m][0], nb * n, f"{m} per-bin shard {s}")
            _check_guards(bigs[m][1], n, f"{m} band shard {s}")
            assert torch.equal(outs[m]["bins"], full[m]["bins"][:, p0:p1]), (m, s)
            assert float((outs[m]["band"] - full[m]["band"][p0:p1]).abs().max()) <= 1e-6, (m, s)
    assert P == sum(row_tile_range(N, shards, s)[1][1] - row_tile_range(N, shards, s)[1][0] for s in range(shards))


def test_spectra_write_only_their_slots():
    """K1 into slots [2, 5) of an 8-slot ring (and a wrapped range [6, 9) -> 6, 7, 0):
    every other slot keeps its sentinel."""
    rng = np.random.default_rng(3)
    N, T, nfft = 90, 200, 256
    plan = DevicePlan(N, T, nfft, 4, 40, taper="hann", slot_capacity=8, device="cuda")
    r64, r32 = plan.ring()
    r64.fill_(complex(SENT, -SENT))
    r32.fill_(complex(SENT, -SENT))
    x = torch.tensor(rng.standard_normal((3, N, T)), device="cuda")
    plan.spectra(x, 2)
    plan.spectra(x, 6)
    torch.cuda.synchronize()
    written = {2, 3, 4, 6, 7, 0}
    for s in range(8):
        untouched = bool((r64[s] == complex(SENT, -SENT)).all()) and bool((r32[s] == complex(SENT, -SENT)).all())
        assert untouched == (s not in written), s
