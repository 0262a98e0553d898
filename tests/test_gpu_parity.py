"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the same seeded inputs.

Gates (BASELINE.json north_star):
  * primary-hit primitive ids bit-exact on >= 99.99 % of pixels, any remainder at <= 1e-5 barycentric
    edges (the design makes them 100 % equal: fp32 camera rays are bit-identical, tests run in fp64);
  * NIF: max relative error of exp(y) <= 1e-2 and |dy| <= 1e-3 in log space (SURVEY 8c caution);
  * framebuffer relative RMSE <= 2e-3.
"""
import numpy as np
import pytest

from paper_2305_20061_b200 import scenes

pytestmark = pytest.mark.gpu

REL_RMSE_GATE = 2e-3
NIF_REL_GATE = 1e-2
NIF_LOG_GATE = 1e-3


@pytest.fixture(scope="module")
def ptm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_20061_b200 import _build, pt
    _build.build()
    pt.lib()
    return pt


@pytest.fixture(scope="module")
def blob():
    return scenes.siren_blob(0)


def _uv_cases(n, seed):
    uv = scenes.query_uv(n, seed)
    edge = np.array([[0, 0], [1, 1], [0.5, 0.5], [0, 1], [1, 0], [1e-7, 0.5], [1 - 2 ** -24, 0.25]], np.float32)
    return np.concatenate([edge, uv])[:n] if n >= len(edge) else uv


@pytest.mark.parametrize("n", [1, 127, 128, 129, 1000, 4 * 148 * 128 + 77])
@pytest.mark.parametrize("scale", [1.0, 30.0])
def test_nif_vs_oracle(ptm, orc, parity_log, n, scale):
    import torch
    blob = scenes.siren_blob(0, out_scale=scale)
    nif = ptm.Nif(blob)
    uv = _uv_cases(n, seed=n)
    got = ptm.nif_infer(nif, torch.from_numpy(uv).cuda()).cpu().numpy().astype(np.float64)
    y = orc.nif_eval(blob, uv.astype(np.float64))
    ref = np.exp(y)
    assert np.isfinite(got).all()
    # log-space gate: 1e-3 for the BASELINE network; for the x30 test network the bound of one fp16
    # rounding of the last hidden activations, 2^-11 * max_j sum_k |W5_jk|, exceeds it
    W5 = scenes.nif_layers_from_blob(blob)[4][0]
    log_gate = max(NIF_LOG_GATE, 2.0 ** -11 * np.abs(W5).sum(1).max())
    dy = np.abs(np.log(got) - y).max()
    rel = (np.abs(got - ref) / ref).max()
    parity_log(f"nif_siren_x{scale:g}_n{n}_max_abs_dy", dy, log_gate)
    parity_log(f"nif_siren_x{scale:g}_n{n}_max_rel", rel, NIF_REL_GATE)
    assert dy <= log_gate
    assert rel <= NIF_REL_GATE


def test_nif_bench_size_sampled(ptm, orc, blob):
    """The escaped-queue size of the bench's config-1 frame (about 2.2 M queries; here 2^21 + 333, so the
    last tile is ragged and every CTA runs > 100 tiles in both slots), checked on 4000 sampled rows."""
    import torch
    n = (1 << 21) + 333
    uv = scenes.query_uv(n, 11)
    got = ptm.nif_infer(ptm.Nif(blob), torch.from_numpy(uv).cuda()).cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all() and (got > 0).all()
    idx = np.concatenate([np.linspace(0, n - 1, 3600).astype(np.int64), np.arange(n - 400, n)])
    y = orc.nif_eval(blob, uv[idx].astype(np.float64))
    assert np.abs(np.log(got[idx]) - y).max() <= NIF_LOG_GATE
    assert (np.abs(got[idx] - np.exp(y)) / np.exp(y)).max() <= NIF_REL_GATE


def test_nif_layer_accumulators(ptm, blob):
    """Debug view: every layer's fp32 accumulator against an independent float64 evaluation of the
    same fp16 activations (isolates MMA layout bugs from the sine epilogue)."""
    import torch
    uv = _uv_cases(512, 3)
    nif = ptm.Nif(blob)
    out, dbg = ptm.nif_debug_layers(nif, torch.from_numpy(uv).cuda())
    dbg = dbg.cpu().numpy().astype(np.float64)
    L = scenes.nif_layers_from_blob(blob)
    x = np.stack([2 * uv[:, 0].astype(np.float64) - 1, 2 * uv[:, 1].astype(np.float64) - 1], 1)
    pre = x @ L[0][0].T + L[0][1]
    assert np.abs(dbg[0] - pre).max() < 1e-3 * max(1.0, np.abs(pre).max())
    h = np.sin(dbg[0]).astype(np.float16).astype(np.float64)     # what the kernel feeds forward
    # tolerance: the epilogue's sine (SFU or fp16 polynomial, |err| <= 1.2e-3) plus fp16 rounding of h,
    # propagated through |W|; a layout bug gives O(1) errors
    sin_err = 1.2e-3 + 2.0 ** -11
    for li in (1, 2, 3):
        pre = h @ L[li][0].T + L[li][1]
        tol = sin_err * np.abs(L[li][0]).sum(1).max() + 1e-4
        assert np.abs(dbg[li] - pre).max() < tol, li
        h = np.sin(dbg[li]).astype(np.float16).astype(np.float64)
    y = h @ L[4][0].T + L[4][1]
    assert np.abs(dbg[4][:, :3] - y).max() < sin_err * np.abs(L[4][0]).sum(1).max() + 1e-4


@pytest.fixture(scope="module")
def fr_blob():
    return scenes.fourier_relu_blob(0)


def _fr_features(uv, B):
    p = 2 * np.pi * (uv.astype(np.float64) @ B.T)
    return np.concatenate([np.sin(p), np.cos(p)], 1)


@pytest.mark.parametrize("n", [1, 127, 129, 1000, 4 * 148 * 128 + 77])
def test_fr_nif_vs_oracle(ptm, orc, fr_blob, n):
    """The paper's own HDR-NIF (Fourier features, ReLU, concat skip, YUV->RGB; PT_NIF_FOURIER_RELU)
    on the tcgen05 kernel against oracle.fr_eval, same gates as the SIREN network."""
    import torch
    nif = ptm.Nif(fr_blob, kind=ptm.NIF_FOURIER_RELU)
    uv = _uv_cases(n, seed=n + 5)
    got = ptm.nif_infer(nif, torch.from_numpy(uv).cuda()).cpu().numpy().astype(np.float64)
    y = orc.fr_eval(fr_blob, uv.astype(np.float64))
    assert np.isfinite(got).all() and (got > 0).all()
    assert np.abs(np.log(got) - y).max() <= NIF_LOG_GATE
    assert (np.abs(got - np.exp(y)) / np.exp(y)).max() <= NIF_REL_GATE


def test_fr_nif_layer_accumulators(ptm, fr_blob):
    """Debug view of the paper's NIF: each layer's fp32 accumulator against float64 products of the
    fp16 activations the kernel fed forward (layout check for the 88-wide layer and the concat skip)."""
    import torch
    uv = _uv_cases(640, 11)
    nif = ptm.Nif(fr_blob, kind=ptm.NIF_FOURIER_RELU)
    out, dbg = ptm.nif_debug_layers(nif, torch.from_numpy(uv).cuda())
    dbg = dbg.cpu().numpy().astype(np.float64)
    B, L = scenes.fourier_relu_from_blob(fr_blob)
    g = _fr_features(uv, B)
    # layer 0: features rounded to fp16 (|err| <= 2^-12 on [-1, 1]) + __sincosf of a reduced argument
    feat_err = 2.0 ** -12 + 2e-6
    pre = g @ L[0][0].T + L[0][1]
    assert np.abs(dbg[0] - pre).max() < feat_err * np.abs(L[0][0]).sum(1).max() + 1e-4
    h = np.maximum(dbg[0], 0).astype(np.float16).astype(np.float64)
    acc = lambda W, a: 1e-5 * (np.abs(a) @ np.abs(W).T).max() + 1e-5      # fp32 accumulation
    pre = h @ L[1][0].T + L[1][1]
    assert np.abs(dbg[1][:, :88] - pre).max() < acc(L[1][0], h)
    h1 = np.maximum(dbg[1][:, :88], 0).astype(np.float16).astype(np.float64)
    a = np.concatenate([h1, g], 1)
    pre = a @ L[2][0].T + L[2][1]
    tol = acc(L[2][0], a) + feat_err * np.abs(L[2][0][:, 88:]).sum(1).max()
    assert np.abs(dbg[2] - pre).max() < tol
    h = np.maximum(dbg[2], 0).astype(np.float16).astype(np.float64)
    pre = h @ L[3][0].T + L[3][1]
    assert np.abs(dbg[3] - pre).max() < acc(L[3][0], h)
    h = np.maximum(dbg[3], 0).astype(np.float16).astype(np.float64)
    yuv = h @ L[4][0].T + L[4][1]
    assert np.abs(dbg[4][:, :3] - yuv).max() < acc(L[4][0], h)
    M = np.array(scenes.YUV_TO_RGB)
    y_gpu = np.log(out.cpu().numpy().astype(np.float64))
    assert np.abs(y_gpu - dbg[4][:, :3] @ M.T).max() < 1e-5 * (1 + np.abs(y_gpu).max())


def test_fr_nif_rejects_wrong_size(ptm, fr_blob, blob):
    with pytest.raises(RuntimeError):
        ptm.Nif(blob, kind=ptm.NIF_FOURIER_RELU)
    with pytest.raises(RuntimeError):
        ptm.Nif(fr_blob, kind=ptm.NIF_SIREN)
    with pytest.raises(RuntimeError):
        ptm.Nif(fr_blob, kind=7)


def _primary_check(ptm, orc, sc, W, H, pix, seed=0, sample=0, log=None, name=None):
    prim_g, t_g = ptm.trace_primary(ptm.Scene(sc), W, H, seed, sample)
    prim_g = prim_g.cpu().numpy()[pix]
    t_g = t_g.cpu().numpy()[pix]
    prim_o, t_o, edge = orc.OracleScene(sc).primary(W, H, seed, sample, pix)
    eq = prim_g == prim_o
    frac = eq.mean()
    mism = ~eq
    if log is not None:
        log(name, frac, 0.9999, pixels=int(len(pix)), mismatches=int(mism.sum()), higher_is_better=True)
    assert frac >= 0.9999, f"primary-hit agreement {frac}"
    assert (edge[mism] <= 1e-5).all(), f"mismatches off the edge band: {edge[mism]}"
    hit = prim_o >= 0
    # t: fp32 estimate within its certified interval (exact fp64 only where a tie had to be decided)
    assert np.allclose(t_g[hit & eq], t_o[hit & eq], rtol=1e-5, atol=0)
    return frac


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_primary_hits_full_frame(ptm, orc, parity_log, cfg):
    c = scenes.CONFIGS[cfg]
    sc = scenes.scene_for_config(cfg)
    pix = np.arange(c.n_pix, dtype=np.int64)
    assert _primary_check(ptm, orc, sc, c.width, c.height, pix, log=parity_log,
                          name=f"primary_hits_c{cfg}_full_s0") == 1.0


def test_primary_hits_small_bvh_sampled(ptm, orc, parity_log):
    c = scenes.CONFIGS[3]
    sc = scenes.scene_for_config(3)
    rows = np.arange(0, c.height, 8)
    pix = (rows[:, None] * c.width + np.arange(c.width)[None, :]).reshape(-1).astype(np.int64)
    assert _primary_check(ptm, orc, sc, c.width, c.height, pix, sample=3, log=parity_log,
                          name="primary_hits_c3_rows8_s3") == 1.0


@pytest.fixture(scope="module")
def large_bvh():
    return scenes.scene_for_config(4)


@pytest.mark.parametrize("sample", [0, 3])
def test_primary_hits_large_bvh_sampled(ptm, orc, parity_log, large_bvh, sample):
    """Config 4 (5.08 M triangles of 64 overlapping displaced icospheres seen from 8-15 units: the
    geometry where SURVEY 8c predicts fp32 barycentric error above the 1e-5 band), every 16th pixel of
    samples 0 and 3: the north_star gate (>= 99.99 % equal, any remainder inside the edge band); the
    certified test with its fp64 fallback makes it 100 %."""
    c = scenes.CONFIGS[4]
    pix = np.arange(0, c.n_pix, 16, dtype=np.int64)
    frac = _primary_check(ptm, orc, large_bvh, c.width, c.height, pix, sample=sample, log=parity_log,
                          name=f"primary_hits_c4_every16_s{sample}")
    assert frac == 1.0


@pytest.mark.parametrize("seed", [0, 1])
def test_trace_rays_random_soup_vs_brute_force(ptm, orc, seed):
    import torch
    sc = scenes.random_soup(2000, 64, seed)
    rng = np.random.default_rng(seed)
    n = 20000
    o = rng.uniform(-2, 2, size=(n, 3)).astype(np.float32)
    tgt = rng.uniform(-0.7, 0.7, size=(n, 3)).astype(np.float32)
    d = (tgt - o).astype(np.float32)
    d[:100] = np.eye(3, dtype=np.float32)[rng.integers(0, 3, 100)]       # axis-aligned rays
    prim_g, t_g = ptm.trace_rays(ptm.Scene(sc), torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda())
    prim_o, t_o, _, _ = orc.OracleScene(sc).closest_hit(o.astype(np.float64), d.astype(np.float64), brute=True)
    assert np.array_equal(prim_g.cpu().numpy(), prim_o)
    hit = prim_o >= 0
    assert np.allclose(t_g.cpu().numpy()[hit], t_o[hit], rtol=1e-5, atol=1e-5)


def test_furnace_empty_scene_exact(ptm):
    img = ptm.render(ptm.Scene(scenes.empty_scene()), None, 37, 23, 3, 4, seed=1, env_rgb=(0.3, 0.7, 1.9))
    assert np.array_equal(img, np.broadcast_to(np.array([0.3, 0.7, 1.9], np.float32), img.shape))


def test_furnace_lambert_sphere(ptm, orc):
    rho = (0.25, 0.5, 0.75)
    sc = scenes.single_sphere_scene(kind=scenes.LAMBERT, albedo=rho)
    W = H = 48
    spp = 8
    img = ptm.render(ptm.Scene(sc), None, W, H, spp, 4, seed=7, env_rgb=(1, 1, 1)).reshape(-1, 3).astype(np.float64)
    k = (img[:, 0] - 1) * spp / (rho[0] - 1)
    assert np.allclose(k, np.round(k), atol=1e-4)
    ref, _ = orc.OracleScene(sc).render(W, H, 4, 7, s0=0, s1=spp)
    assert np.allclose(img, ref / spp, rtol=0, atol=1e-6)


def _rel_rmse(a, b):
    return float(np.sqrt(((a - b) ** 2).sum() / (b ** 2).sum()))


def test_render_config0_full_vs_oracle(ptm, orc, blob, parity_log):
    c = scenes.CONFIGS[0]
    sc = scenes.scene_for_config(0)
    img = ptm.render(ptm.Scene(sc), ptm.Nif(blob), c.width, c.height, c.spp, c.max_depth, seed=c.seed)
    ref, _ = orc.OracleScene(sc).render(c.width, c.height, c.max_depth, c.seed, s0=0, s1=c.spp, nif_blob=blob)
    ref = ref.reshape(c.height, c.width, 3) / c.spp
    rel = _rel_rmse(img, ref)
    parity_log("frame_rel_rmse_c0_full", rel, REL_RMSE_GATE)
    assert rel <= REL_RMSE_GATE


def test_render_config1_rows_vs_oracle(ptm, orc, blob, parity_log):
    """Config 1 at full size in the bench launch configuration; oracle on every 16th row."""
    c = scenes.CONFIGS[1]
    sc = scenes.scene_for_config(1)
    img = ptm.render(ptm.Scene(sc), ptm.Nif(blob), c.width, c.height, c.spp, c.max_depth, seed=c.seed)
    rows = np.arange(0, c.height, 16)
    pix = (rows[:, None] * c.width + np.arange(c.width)[None, :]).reshape(-1).astype(np.int64)
    ref, _ = orc.OracleScene(sc).render(c.width, c.height, c.max_depth, c.seed, pix=pix, s0=0, s1=c.spp,
                                        nif_blob=blob)
    got = img.reshape(-1, 3)[pix]
    rel = _rel_rmse(got, ref / c.spp)
    parity_log("frame_rel_rmse_c1_rows16", rel, REL_RMSE_GATE)
    assert rel <= REL_RMSE_GATE


def test_render_deterministic_and_wave_invariant(ptm, blob):
    import torch
    c = scenes.CONFIGS[0]
    s = ptm.Scene(scenes.scene_for_config(0))
    nif = ptm.Nif(blob)
    a = ptm.render(s, nif, c.width, c.height, 4, 4, seed=5)
    b = ptm.render(s, nif, c.width, c.height, 4, 4, seed=5)
    assert np.array_equal(a, b)
    acc = torch.zeros(c.width * c.height * 3, device="cuda")
    for first in range(4):            # one sample per wave, four calls
        ptm.render_samples(s, nif, c.width, c.height, first, 1, 4, 5, acc, wave_samples=1)
    torch.cuda.synchronize()
    d = acc.cpu().numpy().reshape(a.shape) / 4
    assert np.allclose(d, a, rtol=1e-6, atol=1e-7)


def _rows_pix(c, n_rows):
    rows = np.linspace(0, c.height - 1, n_rows).astype(np.int64)
    return (rows[:, None] * c.width + np.arange(c.width)[None, :]).reshape(-1).astype(np.int64)


@pytest.mark.parametrize("cfg,n_rows", [(2, 12), (3, 6), (4, 4)])
def test_render_full_size_rows_vs_oracle(ptm, orc, blob, parity_log, cfg, n_rows):
    """Configs 2-4 at full resolution and full spp (config 4: 5.08 M triangles, constant env);
    the oracle evaluates evenly spaced full rows of the same frame."""
    c = scenes.CONFIGS[cfg]
    sc = scenes.scene_for_config(cfg)
    nif = ptm.Nif(blob) if c.use_nif else None
    img = ptm.render(ptm.Scene(sc), nif, c.width, c.height, c.spp, c.max_depth, seed=c.seed,
                     env_rgb=None if c.use_nif else c.env_rgb)
    pix = _rows_pix(c, n_rows)
    ref, _ = orc.OracleScene(sc).render(c.width, c.height, c.max_depth, c.seed, pix=pix, s0=0, s1=c.spp,
                                        nif_blob=blob if c.use_nif else None, env_rgb=c.env_rgb)
    got = img.reshape(-1, 3)[pix].astype(np.float64)
    rel = _rel_rmse(got, ref / c.spp)
    parity_log(f"frame_rel_rmse_c{cfg}_{n_rows}rows", rel, REL_RMSE_GATE)
    assert rel <= REL_RMSE_GATE, rel


@pytest.mark.parametrize("W,H,spp,depth", [(1, 1, 1, 1), (7, 3, 1, 1), (33, 17, 3, 2), (64, 64, 5, 12)])
def test_render_edge_sizes(ptm, orc, blob, W, H, spp, depth):
    """Odd/tiny frames, single sample, depth 1 (direct only) and a deep cap: exact agreement in the
    direct-only case (primary hits are bit-exact, NIF within its gate), rel-RMSE otherwise."""
    sc = scenes.box_scene()
    img = ptm.render(ptm.Scene(sc), ptm.Nif(blob), W, H, spp, depth, seed=11)
    ref, _ = orc.OracleScene(sc).render(W, H, depth, 11, s0=0, s1=spp, nif_blob=blob)
    ref = ref.reshape(H, W, 3) / spp
    assert np.isfinite(img).all()
    assert _rel_rmse(img, ref) <= REL_RMSE_GATE
    if depth == 1:
        assert np.allclose(img, ref, rtol=1e-2, atol=1e-6)


def test_invalid_arguments_raise(ptm, blob):
    s = ptm.Scene(scenes.box_scene())
    with pytest.raises(ptm.PtError):
        ptm.render(s, ptm.Nif(blob), 0, 4, 1, 1)
    with pytest.raises(ptm.PtError):
        ptm.render(s, ptm.Nif(blob), 4, 4, 1, 0)
    with pytest.raises(ptm.PtError):
        ptm.Nif(blob[:-1])


def test_render_closed_box_no_escapes(ptm, orc, blob):
    """Camera inside a closed box: no path escapes, so the NIF queue is empty in every wave (the NIF
    kernels launch with a zero row count and must only drain their prologue). The frame equals the
    oracle's (emitter light only), and is bit-identical whichever NIF is attached."""
    sc = scenes.box_scene()
    h = 0.5
    front = scenes._quad((-h, -h, h), (-h, h, h), (h, h, h), (h, -h, h), 0)      # -z, closes the box
    sc.tris = np.concatenate([sc.tris, front])
    sc.camera = scenes._camera((0.0, 0.0, 0.4), (0.0, 0.0, -0.5), (0.0, 1.0, 0.0), 60.0)
    W, H, spp, depth = 24, 16, 4, 6
    S = ptm.Scene(sc)
    img = ptm.render(S, ptm.Nif(blob), W, H, spp, depth, seed=3)
    gst = S.stats()
    assert gst["escaped"] == 0
    # traversal counters are a counting-build feature (pt.h): -1 in the product library
    assert (gst["node_visits"], gst["prim_tests"], gst["fp64_rechecks"]) == (-1, -1, -1)
    ref, st = orc.OracleScene(sc).render(W, H, depth, 3, s0=0, s1=spp, nif_blob=blob)
    assert st["escaped"] == 0
    assert _rel_rmse(img, ref.reshape(H, W, 3) / spp) <= REL_RMSE_GATE
    others = [ptm.Nif(scenes.fourier_relu_blob(0), kind=ptm.NIF_FOURIER_RELU),
              ptm.Nif(scenes.fourier_relu_family_blob(64, 2, seed=1), kind=ptm.NIF_FR_FAMILY, hidden=64, layers=2),
              ptm.Nif(scenes.fourier_relu_family_blob(1024, 8, seed=1), kind=ptm.NIF_FR_FAMILY, hidden=1024,
                      layers=8)]
    for nif in others:
        assert np.array_equal(ptm.render(ptm.Scene(sc), nif, W, H, spp, depth, seed=3), img)


def test_render_identical_without_programmatic_dependent_launch(ptm, blob, tmp_path):
    """The wave's kernels chained with programmatic dependent launch (griddepcontrol) produce exactly the
    frame of plain stream-ordered launches (PT_NO_PDL=1, read once per process: a child process)."""
    import os
    import subprocess
    import sys
    c = scenes.CONFIGS[0]
    img = ptm.render(ptm.Scene(scenes.scene_for_config(0)), ptm.Nif(blob), c.width, c.height, c.spp, c.max_depth,
                     seed=c.seed)
    out = tmp_path / "nopdl.npy"
    code = ("import numpy as np; from paper_2305_20061_b200 import pt, scenes; c = scenes.CONFIGS[0]; "
            "img = pt.render(pt.Scene(scenes.scene_for_config(0)), pt.Nif(scenes.siren_blob(0)), c.width, c.height, "
            f"c.spp, c.max_depth, seed=c.seed); np.save(r'{out}', img)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, PT_NO_PDL="1"),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert np.array_equal(np.load(out), img)


def test_render_rows_equals_full_frame_rows(ptm, blob):
    """pt_render_rows (the multi-GPU row-block split, reading R19) renders exactly the full frame's rows:
    the same Philox counters (full-frame pixel index) and the same per-pixel sample order, so the rows are
    bit-identical and every other row of the accumulator is left untouched."""
    import torch
    c = scenes.CONFIGS[0]
    S = ptm.Scene(scenes.scene_for_config(0))
    N = ptm.Nif(blob)
    full = torch.zeros(c.width * c.height * 3, device="cuda")
    ptm.render_samples(S, N, c.width, c.height, 0, c.spp, c.max_depth, 9, full, wave_samples=c.spp)
    for r0, r1 in ((0, 64), (5, 6), (17, 43), (60, 64)):
        part = torch.full((c.width * c.height * 3,), -1.0, device="cuda")
        part.view(c.height, c.width, 3)[r0:r1] = 0.0
        ptm.render_rows(S, N, c.width, c.height, r0, r1, 0, c.spp, c.max_depth, 9, part, wave_samples=c.spp)
        torch.cuda.synchronize()
        p3 = part.view(c.height, c.width, 3).cpu().numpy()
        f3 = full.view(c.height, c.width, 3).cpu().numpy()
        assert np.array_equal(p3[r0:r1], f3[r0:r1])
        assert (p3[:r0] == -1).all() and (p3[r1:] == -1).all()
    with pytest.raises(ptm.PtError):
        ptm.render_rows(S, N, c.width, c.height, 10, 10, 0, 1, 2, 0, full)


def test_concurrent_streams_match_sequential(ptm, blob):
    """Library scratch shared across calls (the NIF query queue of pt_nif_infer, the pooled wave state of
    the renders) is ordered by events across streams: two streams issuing interleaved NIF
    queries and renders of two scene handles produce exactly the sequential results."""
    import torch
    nif = ptm.Nif(blob)
    uv1 = torch.from_numpy(scenes.query_uv(300_000, 21)).cuda()
    uv2 = torch.from_numpy(scenes.query_uv(200_000, 22)).cuda()
    ref1 = ptm.nif_infer(nif, uv1).clone()
    ref2 = ptm.nif_infer(nif, uv2).clone()
    c = scenes.CONFIGS[0]
    S1, S2 = ptm.Scene(scenes.scene_for_config(0)), ptm.Scene(scenes.box_scene(seed=3))
    fr1 = torch.zeros(c.width * c.height * 3, device="cuda")
    fr2 = torch.zeros(c.width * c.height * 3, device="cuda")
    ptm.render_samples(S1, nif, c.width, c.height, 0, 4, 6, 1, fr1)
    ptm.render_samples(S2, nif, c.width, c.height, 0, 4, 6, 2, fr2)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    o1 = torch.empty_like(ref1)
    o2 = torch.empty_like(ref2)
    g1 = torch.zeros_like(fr1)
    g2 = torch.zeros_like(fr2)
    for _ in range(3):
        g1.zero_()
        g2.zero_()
        torch.cuda.synchronize()
        ptm.nif_infer(nif, uv1, out=o1, stream=sa)
        ptm.nif_infer(nif, uv2, out=o2, stream=sb)
        ptm.render_samples(S1, nif, c.width, c.height, 0, 4, 6, 1, g1, stream=sa)
        ptm.render_samples(S2, nif, c.width, c.height, 0, 4, 6, 2, g2, stream=sb)
        torch.cuda.synchronize()
        assert torch.equal(o1, ref1) and torch.equal(o2, ref2)
        assert torch.equal(g1, fr1) and torch.equal(g2, fr2)


@pytest.mark.parametrize("n_tiles", [1, 149, 148 * 2 + 77, 148 * 3, 148 * 4 + 147, 148 * 5 + 1, 148 * 6 + 100, 148 * 8])
def test_nif_schedule_rounds(ptm, orc, blob, n_tiles):
    """The SIREN kernel runs three 128-row tiles per CTA round (tiles b + s * grid, s < 3) with the layer
    groups rotating over two accumulator regions, two epilogue teams and two issuers; a CTA's last round
    holds 1, 2 or 3 tiles. Query counts whose tile counts end every CTA on each of those cases (and a
    ragged last tile): sampled rows (the first and last tile in full) against the oracle, and the whole
    output bit-identical across two launches (a barrier-protocol race would show as a difference)."""
    import torch
    n = n_tiles * 128 - 37
    uv = scenes.query_uv(n, 11)
    nif = ptm.Nif(blob)
    q = torch.from_numpy(uv).cuda()
    a = ptm.nif_infer(nif, q).cpu().numpy()
    b = ptm.nif_infer(nif, q).cpu().numpy()
    assert np.array_equal(a, b)
    rng = np.random.default_rng(n_tiles)
    idx = np.unique(np.concatenate([np.arange(min(128, n)), np.arange(max(0, n - 128), n),
                                    rng.integers(0, n, size=min(n, 1536))]))
    y = orc.nif_eval(blob, uv[idx].astype(np.float64))
    got = a[idx].astype(np.float64)
    assert np.isfinite(got).all()
    assert np.abs(np.log(got) - y).max() <= NIF_LOG_GATE
    assert (np.abs(got - np.exp(y)) / np.exp(y)).max() <= NIF_REL_GATE


def test_render_async_matches_render(ptm, blob):
    """pt_render_async on two streams with two scene handles (the overlapped read-back an application
    uses) returns the frames pt_render returns, bit for bit."""
    import torch
    c = scenes.CONFIGS[1]
    sc = scenes.scene_for_config(1)
    W, H, spp = 96, 64, 4
    nif = ptm.Nif(blob)
    S1, S2 = ptm.Scene(sc), ptm.Scene(sc)
    ref1 = ptm.render(S1, nif, W, H, spp, c.max_depth, seed=5)
    ref2 = ptm.render(S1, nif, W, H, spp, c.max_depth, seed=6)
    b1 = torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)
    b2 = torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ptm.render_async(S1, nif, W, H, spp, c.max_depth, 5, b1.numpy(), stream=s1)
    ptm.render_async(S2, nif, W, H, spp, c.max_depth, 6, b2.numpy(), stream=s2)
    s1.synchronize()
    s2.synchronize()
    assert np.array_equal(b1.numpy().reshape(H, W, 3), ref1)
    assert np.array_equal(b2.numpy().reshape(H, W, 3), ref2)


@pytest.mark.parametrize("cfg", [0, 3])
def test_wave_buffer_layouts_bit_identical(ptm, blob, cfg):
    """Sample sums accumulated with waves of 1 and 3 samples (sample-major wave buffer, 8 x 4 tiles) and
    of 4 / 32 samples (a pixel's samples per first-bounce warp, pixel-major buffer, float4 accumulate)
    are bit-identical: every layout adds a pixel's samples in the same order."""
    import torch
    c = scenes.CONFIGS[cfg]
    W, H, spp = (c.width, c.height, 4) if cfg == 0 else (320, 64, 32)
    s = ptm.Scene(scenes.scene_for_config(cfg))
    nif = ptm.Nif(blob)
    outs = []
    for k in (1, 3, spp):
        acc = torch.zeros(W * H * 3, device="cuda")
        ptm.render_samples(s, nif, W, H, 0, spp, c.max_depth, 7, acc, wave_samples=k)
        torch.cuda.synchronize()
        outs.append(acc.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


def test_nif_empty_query_all_kinds(ptm, blob):
    """Zero queries are a no-op for every NIF kind (SIREN, the paper's NIF, a family member in fp16 and
    fp8), and a one-row query right after still matches a fresh handle's result."""
    import torch
    nets = [ptm.Nif(blob), ptm.Nif(scenes.fourier_relu_blob(0), kind=ptm.NIF_FOURIER_RELU),
            ptm.Nif(scenes.fourier_relu_family_blob(128, 4, seed=1), kind=ptm.NIF_FR_FAMILY, hidden=128, layers=4),
            ptm.Nif(scenes.fourier_relu_family_blob(128, 4, seed=1), kind=ptm.NIF_FR_FAMILY, hidden=128, layers=4,
                    fp8=True)]
    uv0 = torch.zeros((0, 2), dtype=torch.float32, device="cuda")
    uv1 = torch.tensor([[0.3, 0.7]], dtype=torch.float32, device="cuda")
    for nif in nets:
        out = ptm.nif_infer(nif, uv0)
        assert tuple(out.shape) == (0, 3)
        a = ptm.nif_infer(nif, uv1).cpu().numpy()
        assert np.isfinite(a).all() and (a > 0).all()
