"""First-divergence classifier on a config-3 crop (SURVEY 8c precision plan #3;
PAPER.md:173): single paths through the render kernels' shade_segment (pt_debug_path_records) against the
fp64 oracle's per-segment records (orc_trace_paths), same Philox draws. Every path either agrees segment
by segment or first differs at a near-edge hit, a near-tie, a near-threshold Fresnel/roulette draw, or an
equirect seam straddle (tools/divergence.py); an unexplained divergence fails. The class histogram is
written to parity.json and gpurun_out/divergence_c3.json."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ptm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_20061_b200 import _build, pt
    _build.build()
    pt.lib()
    return pt


@pytest.mark.parametrize("cfg,crop", [(3, (496, 16, 896, 128)), (2, (500, 8, 448, 128)), (4, (1000, 4, 1800, 128))])
def test_first_divergences_are_explained(ptm, orc, parity_log, cfg, crop):
    import divergence
    res, g, o = divergence.run(cfg, *crop)
    hist = res["histogram"]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"divergence_c{cfg}.json"), "w") as f:
        json.dump(res, f, indent=1)
    n = res["paths"]
    parity_log(f"divergence_c{cfg}_same_fraction", hist["same"] / n, 0.99, higher_is_better=True, histogram=hist)
    assert hist["unexplained"] == 0, [e for e in res["examples"] if e["class"] == "unexplained"][:5]
    assert hist["same"] >= 0.99 * n
