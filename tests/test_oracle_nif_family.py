"""Pins for the oracle's evaluation of the paper's NIF family of the size sweep ("hidden
size H (128) and number of dense-relu layers L (4) can be varied", Fig. nrf-vs-blender H64 L2 / H256 L4 /
H1024 L8; reading R23).

(i) the concat-layer rule and the parameter counts the paper/SURVEY quote ("97 KiB" for H128 L4,
PAPER.md:165; 387 KiB and 14.0 MiB for H256 L4 and H1024 L8); (ii) for every sweep member
a hand-built single-path network whose signal crosses the concat skip at the reading's layer has a
closed form (catches the skip position, feature order, transposes, ReLU, the colour matrix); (iii) the
(128, 4) member equals the separately pinned orc_fr_eval on a random network."""
import math

import numpy as np
import pytest

from paper_2305_20061_b200 import scenes


def test_concat_layer_rule(orc):
    # largest odd 0-based index below L/2, else 0 (written out by hand)
    want = {1: 0, 2: 0, 3: 1, 4: 1, 5: 1, 6: 1, 7: 3, 8: 3, 9: 3, 10: 3}
    for L, c in want.items():
        assert orc.fr_concat_layer(L) == c == scenes.fr_concat_layer(L), L


def test_family_sizes():
    kib = {hl: scenes.fr_family_halves(*hl) * 2 / 1024 for hl in scenes.NIF_SWEEP}
    assert scenes.fr_family_halves(128, 4) == scenes.FR_N_HALVES == 50051
    assert abs(kib[(128, 4)] - 97.8) < 0.05                   # "97 KiB" (incl. B)
    assert abs(kib[(256, 4)] - 387.5) < 0.05                  # 387 KiB
    assert abs(kib[(1024, 8)] / 1024 - 14.02) < 0.01          # 14.0 MiB


def _chain_blob(H, L, w=None, bias=None, cos_w=3.0):
    """Single active path: sin feature 5 -> unit 3 of layer 0 -> ... ; the layer after the concat
    also reads cos feature 5 from its concat column. Returns (blob, closed-form function of (u, v))."""
    c = scenes.fr_concat_layer(L)
    dims = scenes.fr_family_layers(H, L)
    B = np.zeros((20, 2))
    B[5] = (1.25, -0.5)
    Ws = [np.zeros((o, i)) for i, o in dims]
    bs = [np.zeros(o) for i, o in dims]
    units = [3 + 2 * l for l in range(L)]               # active unit of layer l (always < H - 40)
    Ws[0][units[0], 5] = 2.0                             # sin feature 5
    bs[0][units[0]] = 0.25
    wl = [None] + [(w if w is not None else (-1.5 if l % 2 else 0.75)) for l in range(1, L)]
    bl = [None] + [(bias if bias is not None else (1.0 if l % 2 else 0.125)) for l in range(1, L)]
    cos_col = (H - 40) + 20 + 5                          # cos feature 5 in the concat input
    for l in range(1, L):
        Ws[l][units[l], units[l - 1]] = wl[l]
        bs[l][units[l]] = bl[l]
        if l == c + 1:
            Ws[l][units[l], cos_col] = cos_w
    Ws[L][0, units[L - 1]] = 1.0                         # Y
    Ws[L][2, units[L - 1]] = 0.5                         # V
    bs[L][:] = (0.125, 0.25, 0.0)
    parts = [B.reshape(-1)]
    for W, b in zip(Ws, bs):
        parts += [W.reshape(-1), b]
    blob = np.concatenate(parts).astype(np.float16).view(np.uint16)

    def closed(u, v):
        relu = lambda z: max(z, 0.0)
        p = 2 * math.pi * (1.25 * u - 0.5 * v)
        x = relu(2.0 * math.sin(p) + 0.25)
        for l in range(1, L):
            z = wl[l] * x + bl[l]
            if l == c + 1:
                z += cos_w * math.cos(p)
            x = relu(z)
        Y, U, V = 0.125 + x, 0.25, 0.5 * x
        return np.array([Y + 1.13983 * V, Y - 0.39465 * U - 0.58060 * V, Y + 2.03211 * U])

    return blob, closed


@pytest.mark.parametrize("H,L", scenes.NIF_SWEEP + [(128, 6), (64, 3)])
def test_single_path_closed_form(orc, H, L):
    blob, closed = _chain_blob(H, L)
    assert blob.size == scenes.fr_family_halves(H, L)
    uv = np.array([[0.1, 0.7], [0.35, 0.2], [0.9, 0.9], [0.0, 0.5], [0.6, 0.05], [0.27, 0.81]])
    y = orc.fr_eval_hl(H, L, blob, uv)
    for (u, v), yy in zip(uv, y):
        assert np.abs(yy - closed(u, v)).max() < 1e-12


def test_h128_l4_member_equals_pinned_fr_eval(orc):
    blob = scenes.fourier_relu_blob(3)
    uv = np.random.default_rng(5).random((300, 2))
    assert np.array_equal(orc.fr_eval_hl(128, 4, blob, uv), orc.fr_eval(blob, uv))


def test_family_blob_generator_is_seeded():
    a = scenes.fourier_relu_family_blob(64, 2, seed=1)
    b = scenes.fourier_relu_family_blob(64, 2, seed=1)
    c = scenes.fourier_relu_family_blob(64, 2, seed=2)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    h = a.view(np.float16).astype(np.float64)
    assert np.isfinite(h).all()


@pytest.mark.parametrize("H,L", [(64, 2), (128, 4)])
def test_render_fr_empty_scene_is_the_nif_of_the_camera_rays(orc, H, L):
    """Empty scene: every sample escapes at its camera ray, so the render is exactly exp of the NIF at
    equirect(d) for the oracle's fp32 camera ray d (one NIF evaluation per sample, no other term)."""
    blob = scenes.fourier_relu_family_blob(H, L, seed=4)
    sc = orc.OracleScene(scenes.empty_scene())
    W, Hh, seed = 12, 8, 5
    pix = np.arange(W * Hh)
    out, st = sc.render_fr(H, L, blob, W, Hh, 4, seed, pix=pix, s0=0, s1=2)
    want = np.zeros((W * Hh, 3))
    for s in range(2):
        d = orc.camera_rays(sc.scene.camera, W, Hh, seed, s, pix).astype(np.float64)
        want += np.exp(orc.fr_eval_hl(H, L, blob, orc.equirect(d)))
    assert st["escaped"] == W * Hh * 2
    assert np.abs(out - want).max() <= 1e-12 * np.abs(want).max()


def test_e4m3_rounding(orc):
    """OCP e4m3, round to nearest even, saturating at 448: hand-computed cases (ties go to the even
    code), and agreement with torch's float8_e4m3fn conversion (a library routine) inside the range."""
    import torch
    cases = {0.0: 0.0, 1.0: 1.0, 1.0625: 1.0, 1.1875: 1.25, 1.125: 1.125, 448.0: 448.0, 500.0: 448.0,
             2.0 ** -9: 2.0 ** -9, 2.0 ** -10: 0.0, 3 * 2.0 ** -11: 2.0 ** -9, 232.0: 224.0, 248.0: 256.0,
             -0.3: -0.3125}
    for x, want in cases.items():
        assert orc.e4m3_round(x) == want, x
    xs = np.random.default_rng(1).uniform(-440, 440, 5000) * np.random.default_rng(2).choice([1e-3, 1e-1, 1], 5000)
    ref = torch.from_numpy(xs).float().to(torch.float8_e4m3fn).double().numpy()
    assert np.array_equal(np.array([orc.e4m3_round(float(np.float32(x))) for x in xs]), ref)


def test_fp8_oracle_on_representable_chain_equals_fp16(orc):
    """With B = 0 (features sin 0 = 0, cos 0 = 1) and weights/biases whose every partial result is an
    e4m3 value, the fp8 evaluation performs no rounding at all and equals the fp16 one exactly."""
    for H, L in [(64, 2), (256, 4)]:
        blob, _ = _chain_blob(H, L, w=1.0, bias=0.25, cos_w=0.5)   # activations 0.25, 0.5, 1.25, 1.5 ...
        h = blob.view(np.float16).copy()
        h[:40] = 0                                         # B = 0
        blob0 = h.view(np.uint16)
        uv = np.random.default_rng(3).random((8, 2))
        a = orc.fr_eval_hl_fp8(H, L, blob0, uv)
        b = orc.fr_eval_hl(H, L, blob0, uv)
        assert np.array_equal(a, b), (H, L)


def test_fp8_oracle_rounds_hidden_activations(orc):
    """One unit whose pre-activation is 1.0625 (a tie between e4m3 1.0 and 1.125): the fp8 model feeds
    1.0 forward, the fp16 model 1.0625 (closed form through the output Y)."""
    H, L = 64, 2
    dims = scenes.fr_family_layers(H, L)
    Ws = [np.zeros((o, i)) for i, o in dims]
    bs = [np.zeros(o) for i, o in dims]
    bs[0][3] = 1.0625                                      # h0[3] = relu(1.0625), exact in fp16
    Ws[1][5, 3] = 1.0
    Ws[2][0, 5] = 1.0                                      # Y = h1[5]
    parts = [np.zeros(40)]
    for W, b in zip(Ws, bs):
        parts += [W.reshape(-1), b]
    blob = np.concatenate(parts).astype(np.float16).view(np.uint16)
    uv = np.array([[0.3, 0.6]])
    y8 = orc.fr_eval_hl_fp8(H, L, blob, uv)[0]
    y16 = orc.fr_eval_hl(H, L, blob, uv)[0]
    assert y16[0] == 1.0625 and y8[0] == 1.0 and y8[1] == 1.0 and y8[2] == 1.0


@pytest.mark.parametrize("H,L", [(64, 2), (128, 4)])
def test_render_fr_fp8_empty_scene_is_the_fp8_nif(orc, H, L):
    """As the fp16 case: with the fp8 model (reading R24) the empty-scene render is exactly exp of
    fr_eval_hl_fp8 at each camera ray's equirect coordinates."""
    blob = scenes.fourier_relu_family_blob(H, L, seed=4)
    sc = orc.OracleScene(scenes.empty_scene())
    W, Hh, seed = 12, 8, 5
    pix = np.arange(W * Hh)
    out, st = sc.render_fr(H, L, blob, W, Hh, 4, seed, pix=pix, s0=0, s1=2, fp8=True)
    want = np.zeros((W * Hh, 3))
    for s in range(2):
        d = orc.camera_rays(sc.scene.camera, W, Hh, seed, s, pix).astype(np.float64)
        want += np.exp(orc.fr_eval_hl_fp8(H, L, blob, orc.equirect(d)))
    assert st["escaped"] == W * Hh * 2
    assert np.abs(out - want).max() <= 1e-12 * np.abs(want).max()
    out16, _ = sc.render_fr(H, L, blob, W, Hh, 4, seed, pix=pix, s0=0, s1=2)
    assert not np.array_equal(out, out16)                     # the flag reaches the evaluation
