"""Pins of the decoder oracle (oracle/decoder.py) against what the paper, SPEC and independent
library routines fix."""
import numpy as np
import pytest
import torch
from scipy.signal import correlate2d

from oracle import decoder as D


def _pyr(H, W, n, F, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return [rng.normal(0, scale, (F + 1, h, w)) for (h, w) in D.layer_dims(H, W, n)]


def test_layer_dims_and_param_layout():
    assert D.layer_dims(1080, 1920, 4) == [(1080, 1920), (540, 960), (270, 480), (135, 240)]
    assert D.layer_dims(9, 7, 3) == [(9, 7), (5, 4), (3, 2)]
    # SPEC.md:311 "for F=4, n=4, total decoder parameters < 120k"
    assert D.param_count(4, 4, 3) < 120_000
    lay = dict(D.param_layout(4, 4, 27))
    assert lay["Wf3"] == (32, 5, 3, 3) and lay["Wf0"] == (32, 37, 3, 3) and lay["Wb1"] == (32, 37)
    assert lay["Wo"] == (27, 32)


def test_conv3x3_equals_library_correlation():
    """Zero-padded 3x3 cross-correlation summed over input channels == scipy correlate2d."""
    rng = np.random.default_rng(1)
    x = rng.normal(size=(3, 7, 9))
    w = rng.normal(size=(2, 3, 3, 3))
    got = D.conv3x3(x, w)
    ref = np.stack([sum(correlate2d(x[c], w[o, c], mode="same", boundary="fill") for c in range(3))
                    for o in range(2)])
    assert np.allclose(got, ref, atol=1e-12)
    # and a single tap lands where it should: w only at (dy, dx) = (+1, -1) shifts the image
    w1 = np.zeros((1, 1, 3, 3))
    w1[0, 0, 2, 0] = 1.0
    s = D.conv3x3(x[:1], w1)[0]
    assert np.array_equal(s[:-1, 1:], x[0, 1:, :-1]) and np.all(s[-1] == 0) and np.all(s[:, 0] == 0)


@pytest.mark.parametrize("h,w,H,W", [(4, 5, 8, 10), (3, 3, 5, 6), (1, 2, 1, 3), (68, 120, 135, 240)])
def test_upsample_equals_torch_bilinear(h, w, H, W):
    """Bilinear 2x with half-pixel centres == torch interpolate(align_corners=False), cropped."""
    y = np.random.default_rng(2).normal(size=(3, h, w))
    ref = torch.nn.functional.interpolate(torch.from_numpy(y)[None], scale_factor=2, mode="bilinear",
                                          align_corners=False)[0].numpy()[:, :H, :W]
    assert np.allclose(D.upsample2x(y, H, W), ref, atol=1e-12)


def test_decode_equals_torch_reference_net():
    """The whole decoder against an independent torch (float64) evaluation of the same network:
    conv2d(padding=1), interpolate, ELU, sigmoid, 1x1 convs."""
    F, n, out_ch, H, W = 3, 3, 3, 13, 11
    pyr = _pyr(H, W, n, F, 3)
    prm = D.init_params(F, n, out_ch, seed=4, gate_bias=0.3)
    prm = prm + np.random.default_rng(5).normal(0, 0.1, prm.shape).astype(np.float32)   # nonzero biases
    p = D.unpack(prm, F, n, out_ch)
    tt = lambda a: torch.from_numpy(np.asarray(a, np.float64))  # noqa: E731
    y = None
    for l in range(n - 1, -1, -1):
        P = tt(pyr[l])[None]
        if y is not None:
            up = torch.nn.functional.interpolate(y, scale_factor=2, mode="bilinear", align_corners=False)
            P = torch.cat([up[:, :, :P.shape[2], :P.shape[3]], P], 1)
        f = torch.nn.functional.conv2d(P, tt(p[f"Wf{l}"]), tt(p[f"bf{l}"]), padding=1)
        g = torch.nn.functional.conv2d(P, tt(p[f"Wg{l}"]), tt(p[f"bg{l}"]), padding=1)
        b = torch.nn.functional.conv2d(P, tt(p[f"Wb{l}"])[:, :, None, None])
        y = torch.nn.functional.elu(f) * torch.sigmoid(g) + b
    ref = torch.nn.functional.conv2d(y, tt(p["Wo"])[:, :, None, None], tt(p["bo"]))[0].numpy()
    got = D.decode(pyr, prm, F, n, out_ch)
    assert got.shape == (out_ch, H, W)
    assert np.allclose(got, ref, atol=1e-11)


def test_closed_gate_gives_zero():
    """gate biases -20 (sigmoid ~ 0), bypass zeroed -> output ~ 0 (< 1e-6)."""
    F, n, out_ch = 4, 3, 3
    prm = D.init_params(F, n, out_ch, seed=6)
    p = D.unpack(prm, F, n, out_ch)
    flat = []
    for name, shape in D.param_layout(F, n, out_ch):
        v = p[name].copy()
        if name.startswith("bg"):
            v[:] = -20.0
        if name.startswith("Wb"):
            v[:] = 0.0
        flat.append(v.reshape(-1))
    out = D.decode(_pyr(16, 12, n, F, 7, scale=0.2), np.concatenate(flat), F, n, out_ch)
    assert np.abs(out).max() < 1e-6


def test_zero_input_zero_bias_is_exactly_zero():
    """all raster channels zero and all biases zero -> output exactly 0."""
    F, n, out_ch = 2, 4, 27
    prm = D.init_params(F, n, out_ch, seed=8, gate_bias=0.0)
    pyr = [np.zeros_like(a) for a in _pyr(20, 18, n, F, 9)]
    assert np.array_equal(D.decode(pyr, prm, F, n, out_ch), np.zeros((out_ch, 20, 18)))


def test_receptive_field_of_a_coarse_pixel():
    """n = 3, one nonzero pixel in the coarsest layer -> the output's support lies in
    that pixel's receptive neighbourhood: 3x3 conv -> +-1 at layer 2, bilinear 2x doubles and
    widens by one, another +-1 per conv on the way down."""
    F, n, out_ch, H, W = 2, 3, 3, 40, 40
    pyr = [np.zeros((F + 1, h, w)) for (h, w) in D.layer_dims(H, W, n)]
    pyr[2][0, 5, 6] = 1.0
    prm = D.init_params(F, n, out_ch, seed=10, gate_bias=0.0)      # zero biases: zero stays zero
    out = D.decode(pyr, prm, F, n, out_ch)
    ys, xs = np.nonzero(np.abs(out).sum(0) > 0)
    assert ys.size > 0

    def grow(lo, hi):                                            # layer l+1 interval -> layer l
        return 2 * lo - 1, 2 * hi + 2
    ylo, yhi, xlo, xhi = 5 - 1, 5 + 1, 6 - 1, 6 + 1               # conv at layer 2
    for _ in range(2):                                           # upsample + conv, twice
        ylo, yhi = grow(ylo, yhi)
        xlo, xhi = grow(xlo, xhi)
        ylo, yhi, xlo, xhi = ylo - 1, yhi + 1, xlo - 1, xhi + 1
    assert ys.min() >= ylo and ys.max() <= yhi and xs.min() >= xlo and xs.max() <= xhi


def test_open_gate_passes_elu_of_features():
    """gate biases +20 (sigmoid ~ 1), feature path = identity-like centre tap, bypass
    zero -> each layer's y = ELU(x) on the passed channels."""
    F, n, out_ch, H, W = 3, 1, 3, 6, 5
    C = F + 1
    pyr = _pyr(H, W, n, F, 11)
    p = {name: np.zeros(shape) for name, shape in D.param_layout(F, n, out_ch)}
    for c in range(C):
        p["Wf0"][c, c, 1, 1] = 1.0
    p["bg0"][:] = 20.0
    p["Wo"][np.arange(3), np.arange(3)] = 1.0
    flat = np.concatenate([p[name].reshape(-1) for name, _ in D.param_layout(F, n, out_ch)])
    out = D.decode(pyr, flat, F, n, out_ch)
    ref = D.elu(pyr[0][:3]) / (1.0 + np.exp(-20.0))
    assert np.allclose(out, ref, atol=1e-14)


def test_fp16_operands_and_magnitudes():
    """fp16 operand rounding moves the output by at most ~2^-10 of the magnitude bound, and the
    magnitude bound dominates the output."""
    F, n, out_ch, H, W = 4, 3, 3, 24, 20
    pyr = _pyr(H, W, n, F, 12, scale=0.5)
    prm = D.init_params(F, n, out_ch, seed=13)
    a = D.decode(pyr, prm, F, n, out_ch)
    b = D.decode(pyr, prm, F, n, out_ch, fp16_operands=True)
    m = D.magnitudes(pyr, prm, F, n, out_ch)
    assert np.all(np.abs(a) <= m + 1e-12)
    assert np.all(np.abs(a - b) <= 2e-3 * m)
    assert np.abs(a - b).max() > 0
