"""GPU tests of ABI features around the hot path: the device-memory hook
(fed_options.dev_alloc / dev_free, here PyTorch's caching allocator) and the
wait bound option."""
import numpy as np
import pytest

from fed_inputs import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1909_03355_b200.build import build
    build()


@pytest.mark.parametrize("resident", [-1, 1])
def test_torch_allocator_hook(resident):
    import torch
    from paper_1909_03355_b200 import fed
    p = make_config(5, n=20)
    a = fed.Fed.from_problem(p, precision=32, dt=2.0e-3, resident=resident)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    b = fed.Fed.from_problem(p, precision=32, dt=2.0e-3, resident=resident, torch_alloc=True)
    grown = torch.cuda.memory_allocated() - before
    ib = b.info()
    assert ib["device_bytes"] > 0 and grown >= ib["device_bytes"]   # every buffer came from torch's pool
    a.step(40)
    b.step(40)
    np.testing.assert_array_equal(a.temperature(), b.temperature())  # same kernels, same arithmetic
    b.close()
    assert torch.cuda.memory_allocated() == before                   # and went back to it
    a.close()


def test_wait_timeout_option_accepted():
    from paper_1909_03355_b200 import fed
    p = make_config(2, n=8, steps=10)
    g = fed.Fed.from_problem(p, precision=64, wait_timeout_s=30.0, resident=1)
    g.step(10)
    assert g.info()["step"] == 10
    with pytest.raises(fed.FedError):
        fed.Fed.from_problem(p, precision=64, wait_timeout_s=float("nan"))
