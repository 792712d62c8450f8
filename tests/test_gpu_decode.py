"""GPU check of rtgs_decode_rgbd (P:232 input pre-processing): the planar float32 frame is, bit for
bit, rgb * float32(1/255) and raw * float32(1/scale) (the plain definition, evaluated by numpy)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W,scale", [(48, 64, 5000.0), (61, 83, 6553.5), (1, 3, 1000.0)])
def test_decode_bitexact(H, W, scale):
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    rng = np.random.default_rng(H * W)
    rgb = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    raw = rng.integers(0, 65536, (H, W), dtype=np.uint16)
    raw[0, 0] = 0
    col = torch.empty((3, H, W), dtype=torch.float32, device="cuda")
    dep = torch.empty((H, W), dtype=torch.float32, device="cuda")
    P.decode_rgbd(torch.as_tensor(rgb, device="cuda"), torch.as_tensor(raw.view(np.int16), device="cuda"), scale,
                  col, dep)
    torch.cuda.synchronize()
    want_c = np.moveaxis(rgb.astype(np.float32) * (np.float32(1) / np.float32(255)), -1, 0)
    want_d = raw.astype(np.float32) * (np.float32(1) / np.float32(scale))
    np.testing.assert_array_equal(col.cpu().numpy(), want_c)
    np.testing.assert_array_equal(dep.cpu().numpy(), want_d)
    assert dep.cpu().numpy()[0, 0] == 0.0
