"""Pins for the oracle's evaluation of the paper's own HDR-NIF (reading R4):
Fourier features [sin(2 pi B x), cos(2 pi B x)] -> ReLU 128 -> ReLU 88 (+ concat of the 40 features)
-> ReLU 128 -> ReLU 128 -> linear 3 (YUV, log) -> fixed BT.601 YUV->RGB.

(i) zero network = M b4; (ii) a hand-built single-frequency network whose signal passes through the
concat skip has a closed form (catches feature order, skip position, transposes, the colour matrix);
(iii) the full network agrees with torch.float64 (independent nn.functional.linear / relu)."""
import math

import numpy as np
import torch

from paper_2305_20061_b200 import scenes


def _blob(B, layers):
    parts = [np.asarray(B, dtype=np.float64).reshape(-1)]
    for W, b in layers:
        parts += [np.asarray(W, dtype=np.float64).reshape(-1), np.asarray(b, dtype=np.float64)]
    h = np.concatenate(parts).astype(np.float16)
    assert h.size == scenes.FR_N_HALVES
    return h.view(np.uint16)


def _zeros():
    return [(np.zeros((o, i)), np.zeros(o)) for i, o in scenes.FR_LAYERS]


def test_blob_size_and_params():
    blob = scenes.fourier_relu_blob(0)
    assert blob.size == 50051
    n_params = sum(o * i + o for i, o in scenes.FR_LAYERS)
    assert n_params == 50011 and abs(n_params * 2 / 1024 - 97.67) < 0.01    # "97 KiB"


def test_zero_net_is_colour_matrix_of_b4(orc):
    L = _zeros()
    b4 = np.array([0.5, -0.25, 0.125])
    L[4] = (np.zeros((3, 128)), b4)
    y = orc.fr_eval(_blob(np.ones((20, 2)), L), np.random.default_rng(0).random((50, 2)))
    want = scenes.YUV_TO_RGB @ b4.astype(np.float16).astype(np.float64)
    assert np.abs(y - want).max() < 1e-15


def test_single_frequency_through_concat_skip(orc):
    B = np.zeros((20, 2)); B[3] = (1.5, -0.75)                 # frequency row 3
    L = _zeros()
    W0 = np.zeros((128, 40)); W0[7, 3] = 2.0                   # unit 7 reads sin feature 3
    b0 = np.zeros(128); b0[7] = 0.25
    W1 = np.zeros((88, 128)); W1[11, 7] = 1.5                  # h1[11] = relu(1.5 h0[7])
    W2 = np.zeros((128, 128)); W2[30, 11] = -1.0; W2[31, 88 + 20 + 3] = 3.0   # h1[11] and cos feature 3
    b2 = np.zeros(128); b2[30] = 2.0
    W3 = np.zeros((128, 128)); W3[40, 30] = 0.5; W3[41, 31] = 1.0
    W4 = np.zeros((3, 128)); W4[0, 40] = 1.0; W4[2, 41] = 0.5  # Y <- unit 40, V <- unit 41
    b4 = np.array([0.125, 0.25, 0.0])
    L = [(W0, b0), (W1, np.zeros(88)), (W2, b2), (W3, np.zeros(128)), (W4, b4)]
    uv = np.array([[0.1, 0.7], [0.35, 0.2], [0.9, 0.9], [0.0, 0.5]])
    y = orc.fr_eval(_blob(B, L), uv)
    relu = lambda z: max(z, 0.0)
    for (u, v), yy in zip(uv, y):
        p = 2 * math.pi * (1.5 * u - 0.75 * v)
        h0 = relu(2.0 * math.sin(p) + 0.25)
        h1 = relu(1.5 * h0)
        h2a, h2b = relu(2.0 - h1), relu(3.0 * math.cos(p))
        Y, U, V = 0.125 + 0.5 * h2a, 0.25, 0.5 * h2b
        want = scenes.YUV_TO_RGB @ np.array([Y, U, V])
        assert np.abs(yy - want).max() < 1e-14


def test_full_network_matches_torch_float64(orc):
    blob = scenes.fourier_relu_blob(0)
    B, L = scenes.fourier_relu_from_blob(blob)
    uv = scenes.query_uv(2048, 4).astype(np.float64)
    x = torch.tensor(uv)
    p = 2 * math.pi * (x @ torch.tensor(B).T)
    g = torch.cat([torch.sin(p), torch.cos(p)], 1)
    lin = lambda a, i: torch.nn.functional.linear(a, torch.tensor(L[i][0]), torch.tensor(L[i][1]))
    h = torch.relu(lin(g, 0))
    h = torch.relu(lin(h, 1))
    h = torch.relu(lin(torch.cat([h, g], 1), 2))
    h = torch.relu(lin(h, 3))
    ref = (lin(h, 4) @ torch.tensor(scenes.YUV_TO_RGB).T).numpy()
    assert np.abs(orc.fr_eval(blob, uv) - ref).max() < 1e-12
