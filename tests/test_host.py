"""CPU tests: C-ABI library load + exports, host-side logic (tiling, sharding,
domain types, synthetic configs).  No kernel launches (no GPU here)."""
import ctypes
import re

import numpy as np
import pytest

from conftest import REFERENCE_SRC, ROOT

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


# ---------------------------------------------------------------- network post-processing (core.py:168-243)
def _net(w, n_nodes, cw=None, lags=None):
    from paper_2303_03279_b200.core import ConnectivityNetwork
    return ConnectivityNetwork(MetricId.COH, FrequencyBand(2, 5, 1.0), 3, tuple(range(n_nodes)),
                               np.zeros((n_nodes, 3)), weights=np.asarray(w, dtype=np.float64), complex_weights=cw, lags=lags)


def test_pair_to_ij_inverts_triu_order():
    from paper_2303_03279_b200.core import pair_to_ij
    for n in (2, 3, 5, 64, 1001):
        i, j = np.triu_indices(n, 1)
        a, b = pair_to_ij(np.arange(len(i)), n)
        assert np.array_equal(a, i) and np.array_equal(b, j)


def test_host_threshold_and_normalize_semantics():
    from paper_2303_03279_b200.core import normalize_network, threshold_network
    w = np.array([0.5, -0.9, 0.5, 0.1, -0.5, 0.9])          # n = 4 nodes, 6 edges, ties
    net = normalize_network(_net(w, 4))
    assert net.normalized and np.allclose(net.weights, w / 0.9)
    t = threshold_network(net, 0.5)                          # ceil(3): both 0.9s, then the first 0.5 tie
    assert t.edge_i.tolist() == [0, 0, 2] and t.edge_j.tolist() == [1, 2, 3]
    z = normalize_network(_net(np.zeros(3), 3))
    assert z.normalized and np.all(z.weights == 0)
    with pytest.raises(ParameterError):
        threshold_network(net, 0.0)


@pytest.mark.skipif(not (REFERENCE_SRC / "connstream").exists(), reason="reference not present (GPU box)")
def test_post_processing_matches_reference_functions():
    """Same inputs through the reference's own normalize/threshold/serialize."""
    import sys
    sys.path.insert(0, str(REFERENCE_SRC))
    from connstream import core as RC
    from paper_2303_03279_b200.core import normalize_network, serialize_network, threshold_network
    rng = np.random.default_rng(3)
    n = 23
    P = n * (n - 1) // 2
    w = np.round(rng.standard_normal(P), 2)                  # rounding makes ties
    cw = w + 1j * np.round(rng.standard_normal(P), 2)
    lags = rng.integers(-5, 5, P)
    i, j = np.triu_indices(n, 1)
    ref = RC.ConnectivityNetwork(RC.MetricId.COHY, RC.FrequencyBand(2, 5, 1.0), 3, tuple(range(n)),
                                 np.zeros((n, 3)), i, j, w, complex_weights=cw, lags=lags)
    ours = _net(w, n, cw=cw, lags=lags)
    ours.metric = MetricId.COHY
    for f in (0.05, 0.3, 1.0):
        a = RC.threshold_network(RC.normalize_network(ref), f)
        b = threshold_network(normalize_network(ours), f)
        assert np.array_equal(a.edge_i, b.edge_i) and np.array_equal(a.edge_j, b.edge_j)
        assert np.array_equal(a.weights, b.weights) and np.array_equal(a.complex_weights, b.complex_weights)
        assert np.array_equal(a.lags, b.lags)
        assert RC.serialize_network(a) == serialize_network(b)


def test_network_fields_in_reference_order_and_wire_format():
    """Positional construction in the reference dataclass's field order (core.py:130-141),
    its i < j validation, and the JSON wire format: key order, byte-level round trip
    (core.py:218-273)."""
    import json
    from paper_2303_03279_b200.core import ConnectivityNetwork, deserialize_network, serialize_network
    band = FrequencyBand(1, 4, 2.0)
    net = ConnectivityNetwork(MetricId.IMAGCOHY, band, 5, (0, 1, 2), np.zeros((3, 3)), np.array([0, 0, 1]),
                              np.array([1, 2, 2]), np.array([0.5, -0.25, 0.125]), None, np.array([2, 0, -3]))
    assert net.n_edges == 3 and net.edge_j.tolist() == [1, 2, 2] and net.lags.tolist() == [2, 0, -3]
    raw = serialize_network(net)
    obj = json.loads(raw)
    assert list(obj) == ["metric", "band", "n_trials", "normalized", "nodes", "edges"]
    assert list(obj["edges"][0]) == ["i", "j", "w", "w_im", "lag"] and obj["edges"][2]["lag"] == -3
    back = deserialize_network(raw)
    assert serialize_network(back) == raw
    assert back.metric is MetricId.IMAGCOHY and back.band == band
    assert np.array_equal(back.edge_i, net.edge_i) and np.array_equal(back.weights, net.weights)
    cw = np.array([0.3 + 0.4j, 0.25 + 0j, -0.125j])
    c = ConnectivityNetwork(MetricId.COHY, band, 2, (0, 1, 2), np.zeros((3, 3)), [0, 0, 1], [1, 2, 2],
                            np.abs(cw), complex_weights=cw)
    assert json.loads(serialize_network(c))["edges"][0]["w_im"] == 0.4
    with pytest.raises(ParameterError):
        ConnectivityNetwork(MetricId.COH, band, 1, (0, 1), np.zeros((2, 3)), np.array([1]), np.array([0]),
                            np.array([0.5]))
    with pytest.raises(ParameterError):
        ConnectivityNetwork(MetricId.COH, band, 1, (0, 1), np.zeros((2, 3)), [0], [1], [np.inf])


def test_threshold_count_and_dominance_property():
    """threshold_network keeps ceil(f n) edges and every kept |w| >= every dropped |w|
    (core.py:184-205), ties toward ascending (i, j)."""
    from hypothesis import given, settings, strategies as st
    from paper_2303_03279_b200.core import normalize_network, threshold_network

    @given(st.lists(st.floats(-1, 1, allow_nan=False), min_size=1, max_size=36), st.floats(0.01, 1.0))
    @settings(max_examples=60, deadline=None)
    def check(ws, frac):
        n = 2
        while n * (n - 1) // 2 < len(ws):
            n += 1
        i, j = np.triu_indices(n, 1)
        from paper_2303_03279_b200.core import ConnectivityNetwork
        net = ConnectivityNetwork(MetricId.COH, FrequencyBand(0, 1, 1.0), 1, tuple(range(n)), np.zeros((n, 3)),
                                  i[:len(ws)], j[:len(ws)], np.array(ws))
        kept = threshold_network(net, frac)
        assert kept.n_edges == int(np.ceil(frac * len(ws)))
        ke = set(zip(kept.edge_i.tolist(), kept.edge_j.tolist()))
        dropped = [abs(w) for a, b, w in zip(net.edge_i.tolist(), net.edge_j.tolist(), ws) if (a, b) not in ke]
        if dropped and kept.n_edges:
            assert min(abs(v) for v in kept.weights) >= max(dropped)

    check()
    from paper_2303_03279_b200.core import ConnectivityNetwork
    tie = ConnectivityNetwork(MetricId.COH, FrequencyBand(0, 1, 1.0), 1, tuple(range(4)), np.zeros((4, 3)),
                              *np.triu_indices(4, 1), np.full(6, 0.5))
    t = threshold_network(tie, 0.5)
    assert list(zip(t.edge_i.tolist(), t.edge_j.tolist())) == [(0, 1), (0, 2), (0, 3)]
    with pytest.raises(ParameterError):
        normalize_network(ConnectivityNetwork(MetricId.COH, FrequencyBand(0, 1, 1.0), 1, (0, 1), np.zeros((2, 3)),
                                              np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)))


@pytest.mark.skipif(not (REFERENCE_SRC / "connstream").exists(), reason="reference not present (GPU box)")
def test_domain_validation_matches_reference_types():
    """EpochMatrix / FrequencyBand / MetricId accept and reject the same inputs with the
    same exception type and message as the reference's core.py:25-110."""
    import sys
    sys.path.insert(0, str(REFERENCE_SRC))
    from connstream import core as RC
    from paper_2303_03279_b200 import core as MC
    cases = [dict(data=np.zeros(5), sfreq=1.0), dict(data=np.zeros((2, 5)), sfreq=0.0),
             dict(data=np.full((2, 5), np.inf), sfreq=1.0), dict(data=np.zeros((2, 0)), sfreq=1.0),
             dict(data=np.zeros((0, 5)), sfreq=1.0), dict(data=np.zeros((2, 5)), sfreq=1.0, trial_index=-1),
             dict(data=[[1, 2], [3, 4]], sfreq=1.0), dict(data=np.zeros((2, 5), np.float32), sfreq=1.0),
             dict(data=np.zeros((2, 3, 4)), sfreq=1.0), dict(data=np.zeros((2, 5)), sfreq=1.0, t0_offset=-0.5)]

    def outcome(fn):
        try:
            r = fn()
            return ("ok", r)
        except Exception as ex:  # noqa: BLE001 -- the exception itself is compared
            return (type(ex).__name__, str(ex))

    for c in cases:
        a = outcome(lambda: (lambda e: (e.n_channels, e.n_samples, e.data.dtype.name))(RC.EpochMatrix(**c)))
        b = outcome(lambda: (lambda e: (e.n_channels, e.n_samples, e.data.dtype.name))(MC.EpochMatrix(**c)))
        assert a == b, (c, a, b)
    for args in [(5, 4, 1.0), (-1, 3, 1.0), (0, 0, 1.0), (2, 3, -1.0)]:
        assert outcome(lambda: (lambda f: (f.n_bins, f.lo_hz, f.hi_hz))(RC.FrequencyBand(*args))) == \
            outcome(lambda: (lambda f: (f.n_bins, f.lo_hz, f.hi_hz))(MC.FrequencyBand(*args))), args
    for n in [" coh", "Coh", "wPLI", "cor", "xcor", "bogus", ""]:
        a, b = outcome(lambda: RC.MetricId.parse(n).value), outcome(lambda: MC.MetricId.parse(n).value)
        assert a == b, n
    assert [m.value for m in RC.MetricId] == [m.value for m in MC.MetricId]
    assert [m.value for m in RC.MetricId if m.is_spectral] == [m.value for m in MC.MetricId if m.is_spectral]
