"""GPU payload wire codec (message.cpp:53-99 on device buffers) against the
oracle encoder, plus round trips and the reference's FormatError cases
(test_message.cpp:37-73)."""
import numpy as np
import pytest
import torch

from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def osp():
    from paper_2306_16926_b200 import osp as m
    m.lib()
    return m


def test_encode_matches_oracle_and_round_trips(osp):
    rng = np.random.default_rng(8)
    for trial in range(20):
        L = int(rng.integers(1, 40))
        counts = rng.integers(1, 3000, L)
        M = int(counts.sum())
        vals = rng.uniform(-1e6, 1e6, M).astype(np.float32)
        ids = sorted(rng.choice(L, size=int(rng.integers(0, L + 1)), replace=False).tolist())
        part = osp.Partition(counts)
        dv = torch.as_tensor(vals, device="cuda")
        kind, it = int(rng.integers(0, 8)), int(rng.integers(0, 2**32))
        enc = osp.encode_payload(part, dv, ids, kind, it)
        want = oracle.encode_payload(kind, it, counts, vals, ids)
        assert bytes(enc.cpu().numpy().tobytes()) == want
        back = torch.zeros_like(dv)
        k2, it2, ids2 = osp.decode_payload(part, enc, back)
        assert (k2, it2) == (kind, it) and list(ids2) == ids
        got = back.cpu().numpy()
        for i in ids:
            off = int(counts[:i].sum())
            assert np.array_equal(got[off:off + counts[i]].view(np.uint32),
                                  vals[off:off + counts[i]].view(np.uint32))


def test_decode_rejects_truncation_and_trailing_bytes(osp):
    part = osp.Partition([2])
    v = torch.tensor([1.0, 2.0], device="cuda")
    enc = osp.encode_payload(part, v, [0], 6, 0)
    out = torch.zeros(2, device="cuda")
    with pytest.raises(osp.FormatError):
        osp.decode_payload(part, enc[:-1].contiguous(), out)
    padded = torch.cat([enc, torch.zeros(1, dtype=torch.uint8, device="cuda")])
    with pytest.raises(osp.FormatError):
        osp.decode_payload(part, padded, out)
    with pytest.raises(osp.FormatError):
        osp.decode_payload(part, torch.tensor([1, 2], dtype=torch.uint8, device="cuda"), out)
    with pytest.raises(osp.ShapeError):
        osp.decode_payload(osp.Partition([3]), enc, torch.zeros(3, device="cuda"))
