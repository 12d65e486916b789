"""The device float32 array power (csrc/rb_svml_powf.cuh) equals NumPy's
``np.power`` bit for bit (NumPy routes float32 array powers through its
bundled SVML powf)."""

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def device_pow(x, y):
    import torch

    from paper_1407_7737_b200 import _lib
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(y, x.shape), np.float32)).cuda()
    out = torch.empty_like(xt)
    _lib.check(_lib.load().rb_np_powf(xt.data_ptr(), yt.data_ptr(), out.data_ptr(), xt.numel(),
                                      torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy()


@pytest.mark.parametrize("y", [0.2, -0.5, 0.25, 2.5, 6.0])
def test_scalar_exponents_bit_exact(y):
    rng = np.random.default_rng(int(abs(y) * 100))
    x = np.exp(rng.uniform(np.log(1e-6), np.log(1e6), 2_000_000)).astype(np.float32)
    want = np.power(x, np.float32(y))
    got = device_pow(x, np.float32(y))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_powers_exponent_tables_bit_exact():
    rng = np.random.default_rng(5)
    for d in (2, 10, 30, 50, 100):
        e = (2.0 + 4.0 * np.arange(d, dtype=np.float32) / max(d - 1, 1)).astype(np.float32)
        x = np.abs(rng.uniform(-200, 200, (20000, d))).astype(np.float32)
        want = np.abs(x) ** e
        got = device_pow(x, np.broadcast_to(e, x.shape))
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_zero_base():
    x = np.zeros(4, np.float32)
    assert np.array_equal(device_pow(x, np.float32(0.2)), np.zeros(4, np.float32))
