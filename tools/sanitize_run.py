"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck), one
tool per gpurun call (B200_PROFILING.md):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

Covers every kernel family of the path at small sizes: smoke() (K1, node stats,
both preps, K2, K3, fp64 fallback), a cfg1-shaped run (four-step FFT K1, 257
bins incl. DC/Nyquist), multitaper (PLV in K3), IMAGCOHY on the tensor cores,
welch mode, the guard overflow records, the online-window graph, network
post-processing and the time-domain kernels.
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import __graft_entry__ as G
    from paper_2303_03279_b200 import synth
    from paper_2303_03279_b200.plan import DevicePlan, WindowGraph, compute_connectivity, pow2_scale
    G.smoke()
    rng = np.random.default_rng(0)
    c = synth.CONFIGS[1]
    x = synth.generate(c, "cuda")
    compute_connectivity(x, c.nfft, c.lo, c.hi, metrics=c.metrics + ("COHY",), taper=c.taper)
    xm = torch.tensor(rng.standard_normal((6, 70, 300)), device="cuda", dtype=torch.float32)
    compute_connectivity(xm, 512, 5, 40, metrics=("PLV", "PLI", "WPLI", "COH"), taper=("dpss", 2.0, 3))
    compute_connectivity(xm, 512, 5, 40, metrics=("IMAGCOHY",))
    compute_connectivity(torch.tensor(rng.standard_normal((4, 30, 600)), device="cuda"), 256, 2, 60,
                         metrics=("COH", "WPLI"), mode="welch")
    xz = rng.standard_normal((8, 90, 128))
    xz[:, 1:20] = xz[:, :1] * rng.uniform(0.5, 2, 19)[None, :, None]
    os.environ["CSCONN_FLAG_CAP"] = "8"
    try:
        out, plan = compute_connectivity(torch.tensor(xz, device="cuda"), 128, 3, 30,
                                         metrics=("PLI", "USPLI", "WPLI", "DSWPLI", "IMAGCOHY"))
        assert plan.guard_stats()["records"] > 0
    finally:
        del os.environ["CSCONN_FLAG_CAP"]
    xs = torch.tensor(rng.standard_normal((30, 64, 128)), device="cuda", dtype=torch.float32)
    plan = DevicePlan(64, 128, 128, 3, 20, taper="hann", slot_capacity=10, device="cuda",
                      scale=pow2_scale(float(xs.abs().max()), 128))
    wg = WindowGraph(plan, 4, ("PLV", "WPLI"))
    wg.prime(xs[:10])
    for u in range(1, 5):
        wg.update(xs[10 + 4 * (u - 1): 10 + 4 * u])
    from paper_2303_03279_b200 import EpochMatrix, MetricId, compute_metric, normalize_network, threshold_network
    eps = [EpochMatrix(e, 128.0) for e in rng.standard_normal((5, 40, 128))]
    net = compute_metric([EpochMatrix(torch.tensor(e.data, device="cuda"), 128.0) for e in eps],
                         MetricId.parse("COH"), 128)
    threshold_network(normalize_network(net), 0.1)
    compute_metric(eps, MetricId.parse("COR"), 128)
    compute_metric(eps, MetricId.parse("XCOR"), 128, max_lag=8)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
