"""turbo_memcpy_sm (include/turbo.h): the serving loop's host <-> device copies done by the SMs.
Not a step of the method; checked byte for byte against the source, both directions, aligned and
unaligned sizes and offsets, device <-> device included."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_00172_b200 import build, turbo
    build.build()
    turbo.load()


@pytest.mark.parametrize("n", [1, 15, 16, 17, 4096, 36288, 41407, 3 << 20])
@pytest.mark.parametrize("off", [0, 1, 7])
def test_memcpy_sm_roundtrip(n, off):
    import torch
    from paper_2207_00172_b200 import turbo
    g = torch.Generator().manual_seed(n + off)
    src = torch.randint(0, 256, (n + off,), dtype=torch.uint8, generator=g).pin_memory()
    dev = torch.zeros(n + off, dtype=torch.uint8, device="cuda")
    turbo.memcpy_sm(dev[off:], src[off:])                     # host -> device
    dev2 = torch.zeros_like(dev)
    turbo.memcpy_sm(dev2[off:], dev[off:])                    # device -> device
    back = torch.zeros(n + off, dtype=torch.uint8).pin_memory()
    turbo.memcpy_sm(back[off:], dev2[off:])                   # device -> host
    torch.cuda.synchronize()
    assert torch.equal(back[off:], src[off:])
    assert int(back[:off].sum()) == 0 and int(dev[:off].sum()) == 0


def test_memcpy_sm_errors():
    import ctypes
    from paper_2207_00172_b200 import turbo
    lib = turbo.load()
    assert lib.turbo_memcpy_sm(None, None, 0, None) == turbo.TURBO_OK
    assert lib.turbo_memcpy_sm(None, ctypes.c_void_p(16), 8, None) != turbo.TURBO_OK
