"""Peer-memory payload exchange (csrc/kg_peer.cu) through the C ABI on one
GPU: the rank's own region stands in for every peer (P copies of one region
pointer), so publish -> gather must return P bit-identical copies of the
payload, alternate the two slots round by round, and a gather with no
publish must time out through the flags instead of hanging. The 2/4-rank
bitwise check against the single-process run is tools/dist_check.py."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_02791_b200 import _lib  # noqa: E402


def make_region(n):
    lib = _lib.require_cuda()
    region, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
    _lib.check(lib.kg_peer_alloc(lib.kg_peer_region_bytes(n), ctypes.byref(region), handle), "kg_peer_alloc")
    return lib, region.value


@pytest.mark.parametrize("n", [1, 1000, 1001, 65_600])
def test_publish_gather_rounds(n):
    lib, region = make_region(n)
    P = 3
    regions_dev = torch.tensor([region] * P, dtype=torch.int64, device="cuda")
    seq = torch.zeros(3, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = _lib.stream_handle()
    try:
        for r in range(5):
            local = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(r))
            out = torch.full((P, n), float("nan"), device="cuda")
            _lib.call("kg_peer_publish", local.data_ptr(), region, n, seq.data_ptr(), st)
            _lib.call("kg_peer_gather", regions_dev.data_ptr(), P, n, out.data_ptr(), seq.data_ptr(),
                      flags.data_ptr(), st)
            torch.cuda.synchronize()
            assert int(flags.item()) == 0
            assert seq.tolist() == [r + 1, 0, 0]
            for p in range(P):
                assert torch.equal(out[p], local)
    finally:
        lib.kg_peer_close(region, 1)


def test_gather_without_publish_times_out():
    n = 64
    lib, region = make_region(n)
    regions_dev = torch.tensor([region], dtype=torch.int64, device="cuda")
    seq = torch.zeros(3, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.zeros((1, n), device="cuda")
    try:
        _lib.call("kg_peer_gather", regions_dev.data_ptr(), 1, n, out.data_ptr(), seq.data_ptr(), flags.data_ptr(),
                  _lib.stream_handle())
        torch.cuda.synchronize()
        assert int(flags.item()) & 16     # KG_FLAG_PEER_TIMEOUT
    finally:
        lib.kg_peer_close(region, 1)
