"""GPU parity of the gated-convolution decoder (trips_decode, tcgen05 implicit-GEMM convolutions)
against oracle/decoder.py.

Tolerances (D8): the kernels round every convolution operand to fp16 (x_l, weights) and
accumulate in fp32.  Against the oracle evaluated with the same fp16 operand rounding the
remaining differences are fp32 accumulation / activation rounding plus the rare fp16 rounding
flip of an operand whose fp32 and fp64 values straddle a half-precision rounding boundary:
|gpu - oracle_fp16| <= 1e-3 M.  Against the exact (fp64) decoder: |gpu - oracle| <= 4e-3 M, where
M is the oracle's per-element magnitude bound (|x|, |W|, |b| propagated)."""
import numpy as np
import pytest
import torch

from oracle import decoder as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def run_case(dev, W, H, n, F, out_ch, seed, gate_bias=1.0, pyr_scale=0.5):
    from paper_2401_06003_b200 import Decoder, Rasterizer
    r = Rasterizer(W, H, n, F, max_points=16, device=dev)
    dec = Decoder(r, out_ch)
    rng = np.random.default_rng(seed)
    pyr = rng.normal(0.0, pyr_scale, r.pyramid_floats).astype(np.float32)
    prm = D.init_params(F, n, out_ch, seed=seed + 1, gate_bias=gate_bias)
    assert prm.size == dec.param_count == D.param_count(F, n, out_ch)
    prm = prm + rng.normal(0.0, 0.05, prm.size).astype(np.float32)        # nonzero biases everywhere
    got = dec(torch.from_numpy(prm).to(dev), torch.from_numpy(pyr).to(dev))
    torch.cuda.synchronize()
    got = got.cpu().numpy().astype(np.float64)
    layers = D.split_pyramid(pyr, H, W, n, F)
    ref16 = D.decode(layers, prm, F, n, out_ch, fp16_operands=True)
    ref = D.decode(layers, prm, F, n, out_ch)
    mag = D.magnitudes(layers, prm, F, n, out_ch)
    assert got.shape == (out_ch, H, W) and np.isfinite(got).all()
    e16 = np.abs(got - ref16)
    assert np.all(e16 <= 1e-3 * mag), f"max err vs fp16-operand oracle {e16.max():.3e} (ratio {(e16 / mag).max():.3e})"
    e = np.abs(got - ref)
    assert np.all(e <= 4e-3 * mag), f"max err vs exact oracle {e.max():.3e} (ratio {(e / mag).max():.3e})"
    return got, ref


def test_decoder_c1_geometry(dev):
    run_case(dev, 64, 64, 4, 4, 3, seed=1)


@pytest.mark.parametrize("W,H,n,F,out_ch", [(100, 77, 3, 1, 27), (130, 200, 1, 8, 3), (257, 35, 2, 4, 3),
                                            (16, 9, 5, 2, 5)])
def test_decoder_odd_shapes(dev, W, H, n, F, out_ch):
    """Widths that are not multiples of the 128-pixel tile (partial tiles, TMA zero fill), a
    single layer (no upsampling), F = 1 and 8, the SH-sized output (27), layers narrower than
    the tile and a 1-pixel-wide coarsest layer."""
    run_case(dev, W, H, n, F, out_ch, seed=W + H)


def test_decoder_closed_gate_and_zero_input(dev):
    """SPEC.md:285 / 295 on the GPU: all-zero pyramid and zero biases -> exactly 0."""
    from paper_2401_06003_b200 import Decoder, Rasterizer
    r = Rasterizer(96, 40, 3, 4, max_points=16, device=dev)
    dec = Decoder(r, 3)
    prm = torch.from_numpy(D.init_params(4, 3, 3, seed=3, gate_bias=0.0)).to(dev)
    out = dec(prm, torch.zeros(r.pyramid_floats, device=dev))
    torch.cuda.synchronize()
    assert torch.count_nonzero(out).item() == 0


def test_decoder_full_hd(dev):
    """The bench's frame: 1920 x 1080, 4 layers, F = 4, 3 output channels, every pixel."""
    got, ref = run_case(dev, 1920, 1080, 4, 4, 3, seed=7)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 1e-3


def test_decoder_argument_errors(dev):
    from paper_2401_06003_b200 import Decoder, Rasterizer
    from paper_2401_06003_b200 import _abi as A
    r = Rasterizer(32, 32, 2, 4, max_points=16, device=dev)
    with pytest.raises(A.TripsError):
        Decoder(r, 0)
    with pytest.raises(A.TripsError):
        Decoder(r, 33)
    dec = Decoder(r, 3)
    with pytest.raises(ValueError):
        dec(torch.zeros(dec.param_count + 1, device=dev), torch.zeros(r.pyramid_floats, device=dev))
    with pytest.raises(A.TripsError):
        A.trips_decode(r.plan, dec.ws.data_ptr() + 4, 0, 3, 0, 0, None)
