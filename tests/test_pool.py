"""Host logic of pipeline.Pool (the persistent graph-array slots of
HotPath.build): views of one cached buffer per key, grown with
headroom, reused while the size fits.  CPU tensors stand in for device ones."""
import torch

from paper_2402_15106_b200.pipeline import Pool


def test_pool_views_reuse_and_growth():
    p = Pool(torch.device("cpu"))
    a = p.empty("x", (10, 4), torch.float32)
    assert a.shape == (10, 4) and a.dtype == torch.float32
    a.fill_(1.0)
    b = p.empty("x", (5, 4), torch.float32)  # fits: same storage
    assert b.data_ptr() == a.data_ptr()
    assert torch.equal(b, torch.ones(5, 4))
    c = p.empty("y", 7, torch.int64)  # another key: its own buffer
    assert c.shape == (7,) and c.data_ptr() != a.data_ptr()
    big = p.empty("x", (1000, 4), torch.float32)  # grows (new buffer, 25 % headroom)
    assert big.shape == (1000, 4)
    assert p.bufs["x"].numel() >= 1000 * 4 * 4 * 1.25
    again = p.empty("x", (1100, 4), torch.float32)  # inside the headroom: no new buffer
    assert again.data_ptr() == big.data_ptr()


def test_pool_dtypes_and_empty_shapes():
    p = Pool(torch.device("cpu"))
    h = p.empty("h", (3, 16), torch.bfloat16)
    assert h.shape == (3, 16) and h.dtype == torch.bfloat16
    z = p.empty("z", (0, 16), torch.int32)
    assert z.shape == (0, 16) and z.numel() == 0
    i = p.empty("i", 5, torch.int32)
    i.copy_(torch.arange(5, dtype=torch.int32))
    assert p.empty("i", 3, torch.int32).tolist() == [0, 1, 2]
