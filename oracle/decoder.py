"""Oracle of the gated-convolution decoder over the image pyramid.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): plain numpy, float64, no blocking or fusion.

What it computes (Sec. 3.3 "Neural Network" and Fig. ``fig:conv``, with the
readings SPEC.md:264-317 fixes where the paper is silent -- DESIGN.md readings D1-D8):

  "a single gated convolution in each layer with a self-bypass connection and a feature size of
   32.  Additionally, we include a bilinear upsampling operation for all layers except the final
   one, merging the output with the subsequent level."

  for l = n-1 (coarsest) .. 0:
      x_l = P_l                                   (l = n-1; the F+1 pyramid channels)
      x_l = concat(U(y_{l+1})[:H_l, :W_l], P_l)   (l < n-1; 32 + F + 1 channels)         D3, D4
      f   = conv3x3(x_l; Wf_l) + bf_l,  g = conv3x3(x_l; Wg_l) + bg_l                    D1, D2
      y_l = ELU(f) * sigmoid(g) + Wb_l x_l        (gated conv [yu2019free] + 1x1 bypass) D5, D6
  out = Wo y_0 + bo                               (1x1 projection to 3 / 27 channels)    D7

U = bilinear 2x upsampling, half-pixel centres (align_corners=False), edge-clamped; the result
is cropped to the finer layer's ceil-size (D4).  conv3x3 is a zero-padded cross-correlation.

The parameters travel as ONE flat float32 vector, layer by layer (l = 0 .. n-1), each layer
``Wf [32][C_l][3][3], bf [32], Wg [32][C_l][3][3], bg [32], Wb [32][C_l]`` with
C_l = F + 1 for the coarsest layer and 32 + F + 1 otherwise (input channel order: the 32
upsampled channels first, then the pyramid's F features and its opacity channel), then
``Wo [out][32], bo [out]`` (``param_layout``).

``decode(..., fp16_operands=True)`` rounds every convolution operand (x_l and the Wf / Wg / Wb
weights) to IEEE half before the float64 arithmetic: the precision the tensor-core kernels
compute in (D8).  ``magnitudes`` propagates |.| bounds for the tolerance.
"""
import math

import numpy as np

HIDDEN = 32


def layer_dims(H, W, n):
    """[(H_l, W_l)] with H_l = ceil(H / 2^l) (reading Q8)."""
    return [(-(-H // (1 << l)), -(-W // (1 << l))) for l in range(n)]


def in_channels(F, n, l):
    return F + 1 if l == n - 1 else HIDDEN + F + 1


def param_layout(F, n, out_ch):
    """[(name, shape)] in the order of the flat parameter vector."""
    lay = []
    for l in range(n):
        C = in_channels(F, n, l)
        lay += [(f"Wf{l}", (HIDDEN, C, 3, 3)), (f"bf{l}", (HIDDEN,)), (f"Wg{l}", (HIDDEN, C, 3, 3)),
                (f"bg{l}", (HIDDEN,)), (f"Wb{l}", (HIDDEN, C))]
    lay += [("Wo", (out_ch, HIDDEN)), ("bo", (out_ch,))]
    return lay


def param_count(F, n, out_ch):
    return sum(int(np.prod(s)) for _, s in param_layout(F, n, out_ch))


def unpack(params, F, n, out_ch):
    out, o = {}, 0
    flat = np.asarray(params, np.float64).reshape(-1)
    for name, shape in param_layout(F, n, out_ch):
        k = int(np.prod(shape))
        out[name] = flat[o:o + k].reshape(shape)
        o += k
    assert o == flat.size, "parameter vector size mismatch"
    return out


def split_pyramid(flat, H, W, n, F):
    """Planar layers [(F+1, H_l, W_l)] of a flat pyramid (the rasterizer's output layout)."""
    layers, o = [], 0
    for (h, w) in layer_dims(H, W, n):
        k = (F + 1) * h * w
        layers.append(np.asarray(flat[o:o + k], np.float64).reshape(F + 1, h, w))
        o += k
    return layers


def conv3x3(x, w):
    """Zero-padded 3x3 cross-correlation: out[o, y, x] = sum_{c, dy, dx} w[o, c, dy+1, dx+1]
    x[c, y+dy, x+dx] (x outside the image = 0)."""
    C, H, W = x.shape
    xp = np.zeros((C, H + 2, W + 2))
    xp[:, 1:H + 1, 1:W + 1] = x
    out = np.zeros((w.shape[0], H, W))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            out += np.tensordot(w[:, :, dy + 1, dx + 1], xp[:, 1 + dy:1 + dy + H, 1 + dx:1 + dx + W], axes=([1], [0]))
    return out


def upsample2x(y, H, W):
    """Bilinear 2x upsampling with half-pixel centres (output i samples input (i + 0.5) / 2 - 0.5,
    clamped to the edge), cropped to (H, W)."""
    C, h, w = y.shape

    def axis(n_out, n_in):
        src = np.maximum((np.arange(n_out) + 0.5) / 2.0 - 0.5, 0.0)
        i0 = np.minimum(np.floor(src).astype(np.int64), n_in - 1)
        i1 = np.minimum(i0 + 1, n_in - 1)
        lam = src - i0
        return i0, i1, lam

    y0, y1, ly = axis(2 * h, h)
    x0, x1, lx = axis(2 * w, w)
    rows = y[:, y0, :] * (1 - ly)[None, :, None] + y[:, y1, :] * ly[None, :, None]
    up = rows[:, :, x0] * (1 - lx)[None, None, :] + rows[:, :, x1] * lx[None, None, :]
    return up[:, :H, :W]


def elu(v):
    return np.where(v > 0, v, np.expm1(np.minimum(v, 0.0)))


def sigmoid(v):
    return 1.0 / (1.0 + np.exp(-v))


def _f16(a):
    return np.asarray(a, np.float64).astype(np.float16).astype(np.float64)


def decode(pyr_layers, params, F, n, out_ch, fp16_operands=False, return_hidden=False):
    """pyr_layers: [(F+1, H_l, W_l)] (split_pyramid).  Returns out (out_ch, H, W) float64
    (and the hidden outputs [y_0 .. y_{n-1}] when return_hidden)."""
    p = unpack(params, F, n, out_ch)
    q = _f16 if fp16_operands else (lambda a: a)
    ys = [None] * n
    y = None
    for l in range(n - 1, -1, -1):
        P = np.asarray(pyr_layers[l], np.float64)
        _, H, W = P.shape
        x = P if y is None else np.concatenate([upsample2x(y, H, W), P], 0)
        x = q(x)
        f = conv3x3(x, q(p[f"Wf{l}"])) + p[f"bf{l}"][:, None, None]
        g = conv3x3(x, q(p[f"Wg{l}"])) + p[f"bg{l}"][:, None, None]
        y = elu(f) * sigmoid(g) + np.tensordot(q(p[f"Wb{l}"]), x, axes=([1], [0]))
        ys[l] = y
    out = np.tensordot(p["Wo"], y, axes=([1], [0])) + p["bo"][:, None, None]
    return (out, ys) if return_hidden else out


def magnitudes(pyr_layers, params, F, n, out_ch):
    """Per-element |.| bounds of the same computation (|x|, |W|, |b| everywhere; ELU and
    sigmoid bounded by their Lipschitz / range properties: |ELU(f)| <= |f|, sigmoid <= 1):
    the tolerance scale of GPU-vs-oracle comparisons."""
    p = unpack(params, F, n, out_ch)
    y = None
    for l in range(n - 1, -1, -1):
        P = np.abs(np.asarray(pyr_layers[l], np.float64))
        _, H, W = P.shape
        x = P if y is None else np.concatenate([upsample2x(y, H, W), P], 0)
        f = conv3x3(x, np.abs(p[f"Wf{l}"])) + np.abs(p[f"bf{l}"])[:, None, None]
        g = conv3x3(x, np.abs(p[f"Wg{l}"])) + np.abs(p[f"bg{l}"])[:, None, None]
        # |ELU(f) sigmoid(g)| <= |f|; an error dg in g moves it by <= |ELU(f)| |dg| / 4 <= |f| |g| / 4
        y = f * (1.0 + g / 4.0) + np.tensordot(np.abs(p[f"Wb{l}"]), x, axes=([1], [0]))
    return np.tensordot(np.abs(p["Wo"]), y, axes=([1], [0])) + np.abs(p["bo"])[:, None, None]


def init_params(F, n, out_ch, seed=0, gate_bias=1.0):
    """SPEC.md:300 initialisation: Kaiming-uniform kernels (fan-in = C k^2), zero biases, gate
    biases +1 (mostly open gates) -- seeded, float32."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shape in param_layout(F, n, out_ch):
        if name.startswith("W"):
            fan_in = int(np.prod(shape[1:]))
            bound = math.sqrt(6.0 / fan_in)
            parts.append(rng.uniform(-bound, bound, shape).reshape(-1))
        elif name.startswith("bg"):
            parts.append(np.full(shape, gate_bias).reshape(-1))
        else:
            parts.append(np.zeros(shape).reshape(-1))
    return np.concatenate(parts).astype(np.float32)
