"""Pins for the oracle's HDR-NIF (BASELINE.json SIREN; readings R1-R3):
y = W5 h4 + b5 with h1 = sin(W1' x0 + b1'), h_{k+1} = sin(W'_{k+1} h_k + b'_{k+1}), x0 = (2u-1, 2v-1).

(i) a zero network reduces to exp(b5); (ii) a hand-built single-path chain network with asymmetric
(non-diagonal) weights has a closed form and catches transposed operands and dropped biases;
(iii) the full SIREN agrees with torch.float64's independent nn.functional.linear implementation."""
import math

import numpy as np
import torch

from paper_2305_20061_b200 import scenes


def _blob_from_layers(layers):
    parts = []
    for W, b in layers:
        parts.append(np.asarray(W, dtype=np.float64).reshape(-1))
        parts.append(np.asarray(b, dtype=np.float64))
    h = np.concatenate(parts).astype(np.float16)
    assert h.size == scenes.NIF_N_HALVES
    return h.view(np.uint16)


def _zero_layers():
    return [(np.zeros((o, i)), np.zeros(o)) for i, o in scenes.NIF_LAYERS]


def test_blob_layout_and_size():
    blob = scenes.siren_blob(0)
    assert blob.dtype == np.uint16 and blob.size == 50307 and blob.nbytes == 100614
    L = scenes.nif_layers_from_blob(blob)
    assert [W.shape for W, _ in L] == [(128, 2), (128, 128), (128, 128), (128, 128), (3, 128)]
    # w0 = 30 folded into layers 1-4: hidden weights bounded by 30 * sqrt(6/128)/30
    assert np.abs(L[1][0]).max() <= math.sqrt(6 / 128) * 1.001
    assert np.abs(L[0][0]).max() <= 30 * 0.5 * 1.001


def test_zero_net_is_exp_b5(orc):
    layers = _zero_layers()
    layers[4] = (np.zeros((3, 128)), np.array([0.5, -1.25, 2.0]))
    uv = np.random.default_rng(0).random((100, 2))
    y = orc.nif_eval(_blob_from_layers(layers), uv)
    assert np.array_equal(y, np.broadcast_to([0.5, -1.25, 2.0], y.shape))


def test_chain_net_closed_form(orc):
    a, bx, c = 0.75, -1.5, 0.3125        # layer 1, unit 0: sin(a*x + bx*y + c)
    w2, w3, w4 = 1.25, -0.875, 2.0       # unit 0 -> unit 1 -> unit 2 -> unit 3 (off-diagonal)
    b2 = 0.125                           # a hidden bias on the chain
    w5 = [0.0, 1.5, -0.5]                # output channels read unit 3 (channel 0 reads nothing)
    b5 = [0.25, -0.125, 0.0625]
    L = _zero_layers()
    W1 = np.zeros((128, 2)); W1[0] = (a, bx); b1 = np.zeros(128); b1[0] = c
    W2 = np.zeros((128, 128)); W2[1, 0] = w2; bb2 = np.zeros(128); bb2[1] = b2
    W3 = np.zeros((128, 128)); W3[2, 1] = w3
    W4 = np.zeros((128, 128)); W4[3, 2] = w4
    W5 = np.zeros((3, 128)); W5[:, 3] = w5
    L = [(W1, b1), (W2, bb2), (W3, np.zeros(128)), (W4, np.zeros(128)), (W5, np.array(b5))]
    uv = np.array([[0.1, 0.9], [0.5, 0.5], [0.0, 0.0], [0.999, 0.25]])
    y = orc.nif_eval(_blob_from_layers(L), uv)
    for (u, v), yy in zip(uv, y):
        x, z = 2 * u - 1, 2 * v - 1
        h = math.sin(w4 * math.sin(w3 * math.sin(w2 * math.sin(a * x + bx * z + c) + b2)))
        want = [b5[k] + w5[k] * h for k in range(3)]
        assert np.abs(yy - want).max() < 1e-15


def _torch_siren(blob, uv):
    L = scenes.nif_layers_from_blob(blob)
    x = torch.tensor(np.stack([2 * uv[:, 0] - 1, 2 * uv[:, 1] - 1], 1), dtype=torch.float64)
    for W, b in L[:4]:
        x = torch.sin(torch.nn.functional.linear(x, torch.tensor(W), torch.tensor(b)))
    W, b = L[4]
    return torch.nn.functional.linear(x, torch.tensor(W), torch.tensor(b)).numpy()


def test_full_siren_matches_torch_float64(orc):
    for scale in (1.0, 30.0):
        blob = scenes.siren_blob(0, out_scale=scale)
        uv = scenes.query_uv(4096, seed=1).astype(np.float64)
        y = orc.nif_eval(blob, uv)
        ref = _torch_siren(blob, uv)
        assert np.abs(y - ref).max() < 1e-12
    # the BASELINE network is nearly constant (SURVEY 8c caution): radiance ~ 0.9 .. 1.2
    env = np.exp(orc.nif_eval(scenes.siren_blob(0), scenes.query_uv(4096, 2).astype(np.float64)))
    assert 0.7 < env.min() and env.max() < 1.5
