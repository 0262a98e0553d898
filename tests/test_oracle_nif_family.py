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


def _chain_blob(H, L):
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
    wl = [None] + [(-1.5 if l % 2 else 0.75) for l in range(1, L)]
    bl = [None] + [(1.0 if l % 2 else 0.125) for l in range(1, L)]
    cos_col = (H - 40) + 20 + 5                          # cos feature 5 in the concat input
    for l in range(1, L):
        Ws[l][units[l], units[l - 1]] = wl[l]
        bs[l][units[l]] = bl[l]
        if l == c + 1:
            Ws[l][units[l], cos_col] = 3.0
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
                z += 3.0 * math.cos(p)
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
