"""CPU tests: C-ABI library load + exports, host-side logic (tiling, sharding,
domain types, synthetic configs).  No kernel launches (no GPU here)."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_2303_03279_b200 import _lib, synth
from paper_2303_03279_b200.core import (DegenerateTrialCountError, EpochMatrix, FrequencyBand, MetricId,
                                        ParameterError, band_average)


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "csconn.h").read_text()
    names = set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(cs_\w+)\s*\(", header, re.M))
    assert len(names) >= 15
    L = _lib.lib()
    for n in sorted(names):
        assert hasattr(L, n), n
    assert L.cs_version().decode().startswith("csconn")
    assert set(_lib.EXPORTED) <= names


def test_error_mapping_without_gpu():
    L = _lib.lib()
    h = ctypes.c_void_p()
    # argument validation happens before any device work
    st = L.cs_plan_create(ctypes.byref(h), 0, 4, 32, 1, 0, 0, 1, None, 1, 1.0, 0)
    assert st == _lib.CS_EPARAM
    with pytest.raises(ParameterError, match="nfft"):
        _lib.check(st)


@pytest.mark.parametrize("n_nodes", [1, 2, 63, 64, 65, 200, 1000, 10242])
@pytest.mark.parametrize("shards", [1, 2, 3, 4, 8])
def test_row_tile_ranges_partition_pairs(n_nodes, shards):
    from paper_2303_03279_b200.plan import row_tile_range
    P = n_nodes * (n_nodes - 1) // 2
    prev_re, prev_p1 = 0, 0
    nt = (n_nodes + 63) // 64
    work = []
    for s in range(shards):
        (rb, re_), (p0, p1) = row_tile_range(n_nodes, shards, s)
        assert rb == prev_re and p0 == prev_p1 and rb <= re_ and p0 <= p1
        prev_re, prev_p1 = re_, p1
        work.append(sum(nt - r for r in range(rb, re_)))
    assert prev_re == nt and prev_p1 == P
    if nt >= 4 * shards:  # row-granular balance: within ~1.2 rows of tiles of the mean
        assert max(work) - sum(work) / shards <= 1.2 * nt


def test_pair_index_convention():
    from paper_2303_03279_b200.spectral import pair_index, pair_row_slice
    for C in (2, 5, 17):
        pi, pj = pair_index(C)
        p = 0
        for i in range(C):
            sl = pair_row_slice(C, i)
            assert sl.start == p
            for j in range(i + 1, C):
                assert pi[p] == i and pj[p] == j
                p += 1


def test_domain_types():
    assert MetricId.parse(" wpli ") is MetricId.WPLI
    with pytest.raises(ParameterError):
        MetricId.parse("nope")
    with pytest.raises(ParameterError):
        FrequencyBand(5, 4, 1.0)
    b = FrequencyBand.from_hz(8, 13, 1000.0, 1024)
    assert (b.lo_bin, b.hi_bin, b.n_bins) == (8, 13, 6)
    with pytest.raises(ParameterError):
        EpochMatrix(data=np.ones(4), sfreq=1.0)
    with pytest.raises(ParameterError):
        EpochMatrix(data=np.array([[1.0, np.nan]]), sfreq=1.0)
    w = np.arange(12.0).reshape(3, 4)
    np.testing.assert_allclose(band_average(w, FrequencyBand(1, 2, 1.0)), w[:, 1:3].mean(1))
    with pytest.raises(ParameterError):
        band_average(w, FrequencyBand(1, 4, 1.0))
    assert issubclass(DegenerateTrialCountError, ParameterError)


def test_synthetic_configs_match_baseline():
    """bins by the nearest-bin rule and P*B*K update counts."""
    want = {1: (0, 256, 4.55e6), 2: (1, 102, 4.76e8), 3: (7, 68, 1.22e10), 4: (4, 15, 3.14e8),
            5: (8, 13, 3.15e10)}
    for c, (lo, hi, upd) in want.items():
        cfg = synth.CONFIGS[c]
        assert (cfg.lo, cfg.hi) == (lo, hi)
        assert abs(cfg.updates / upd - 1) < 0.01


def test_synthetic_generation_is_node_subset_stable():
    cfg = synth.CONFIGS[2]
    x = synth.generate(cfg, "cpu", nodes=slice(250, 306))
    y = synth.generate(cfg, "cpu", nodes=slice(256, 300))
    assert np.array_equal(x[:, 6:50].numpy(), y.numpy())
    w = synth.generate(synth.CONFIGS[4], "cpu", nodes=slice(0, 8), trials=range(5, 10))
    v = synth.generate(synth.CONFIGS[4], "cpu", nodes=slice(0, 8), trials=range(0, 10))
    assert np.array_equal(w.numpy(), v[5:].numpy())
