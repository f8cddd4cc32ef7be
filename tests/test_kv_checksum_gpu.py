"""K6 migration checksum on the GPU (emm_kv_checksum) against the C oracle,
and as the verification of a real paged copy."""
import numpy as np
import pytest
import torch

from oracle import hashes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,slots,row_elems,n", [(2, 64, 512, 40), (28, 3000, 512, 2500),
                                                 (3, 10, 8, 10), (1, 5, 4096, 0)])
def test_kv_checksum_matches_oracle(L, slots, row_elems, n):
    from paper_2507_10069_b200 import dataplane
    g = torch.Generator(device="cuda").manual_seed(L * 7 + n)
    planes = torch.randn(L, 2, slots, row_elems, device="cuda", generator=g).bfloat16()
    rows = torch.randperm(slots, device="cuda", generator=g)[:n].to(torch.int32)
    got = int(dataplane.kv_checksum(planes, rows, n).item()) & (2 ** 64 - 1)
    want = hashes.kv_checksum(planes.view(torch.int16).cpu().numpy(), rows.cpu().numpy(), n)
    assert got == want
    got_id = int(dataplane.kv_checksum(planes, None, min(n, slots)).item()) & (2 ** 64 - 1)
    assert got_id == hashes.kv_checksum(planes.view(torch.int16).cpu().numpy(), None,
                                        min(n, slots))


def test_checksum_verifies_a_paged_copy_and_catches_corruption():
    from paper_2507_10069_b200 import dataplane
    L, slots, row = 4, 2000, 512
    g = torch.Generator(device="cuda").manual_seed(9)
    pool = torch.randn(L, 2, slots, row, device="cuda", generator=g).bfloat16()
    src_rows = torch.randperm(slots, device="cuda", generator=g)[:1500].to(torch.int32)
    dst = torch.zeros(L, 2, 1600, row, device="cuda", dtype=torch.bfloat16)
    dst_rows = torch.randperm(1600, device="cuda", generator=g)[:1500].to(torch.int32)
    dataplane.kv_copy_rows(pool, src_rows, dst, dst_rows, 1500)
    a = dataplane.kv_checksum(pool, src_rows, 1500).item()
    b = dataplane.kv_checksum(dst, dst_rows, 1500).item()
    assert a == b
    dst[2, 1, dst_rows[77].item(), 3] += 1.0
    assert dataplane.kv_checksum(dst, dst_rows, 1500).item() != a
