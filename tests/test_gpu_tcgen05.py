"""Unit test of the tcgen05 correlation kernel (TMA + UMMA fp16 + TMEM top-k
epilogue) against a plain PyTorch fp32 reference of the same op:
c = fp16(R) . fp16(s D)^T / s with exact fp16 products and fp32 sums (s = 2^8
over the largest atom norm's power of two: the dictionary operand's scale)."""

import numpy as np
import pytest
import torch

from paper_1511_05174_b200 import _native as N
from paper_1511_05174_b200 import device as D

pytestmark = pytest.mark.gpu


def reference_topk(rows, atoms):
    scale = 2.0 ** (8 - int(np.floor(np.log2(np.linalg.norm(atoms, axis=1).max()))))
    r = torch.from_numpy(rows).cuda().to(torch.float16).float()
    d = (torch.from_numpy(atoms).cuda() * scale).to(torch.float16).float() / scale
    c = (r @ d.T).abs()
    vals, idx = torch.sort(c, dim=1, descending=True)
    return c.cpu().numpy(), vals.cpu().numpy(), idx.cpu().numpy()


@pytest.mark.parametrize("p,n,t,cap", [(25, 6, 10, 0), (300, 64, 256, 0), (1000, 256, 2048, 0),
                                       (1000, 256, 2048, 1), (700, 256, 1000, 2),
                                       (300, 1024, 512, 0), (129, 33, 130, 1)])
def test_corr_topk_matches_torch(p, n, t, cap):
    rng = np.random.default_rng(p + n + t)
    atoms = rng.standard_normal((t, n))
    atoms /= np.linalg.norm(atoms, axis=1, keepdims=True)
    rows = rng.standard_normal((p, n)).astype(np.float32)
    dd = D.DeviceDictionary(atoms)
    rd = torch.from_numpy(rows).cuda()
    idx = torch.empty((p, 8), dtype=torch.int32, device="cuda")
    val = torch.empty((p, 8), dtype=torch.float32, device="cuda")
    drop = torch.empty((p,), dtype=torch.float32, device="cuda")
    N.check(N.load().cdb_debug_corr_topk(dd.handle, N.ptr(rd), p, N.ptr(idx), N.ptr(val),
                                         N.ptr(drop), cap, None))
    c, vals, order = reference_topk(rows, atoms.astype(np.float32))
    idx, val, drop = idx.cpu().numpy(), val.cpu().numpy(), drop.cpu().numpy()
    tol = 1e-4 * np.abs(c).max(axis=1) + 1e-6
    for r in range(p):
        kept = idx[r][idx[r] >= 0]
        # values reported are the kernel's |c| truncated to 2^-15 relative
        assert np.all(np.abs(val[r][: len(kept)] - c[r, kept]) <= tol[r] + 4e-5 * c[r, kept])
        # everything not kept is below the smallest kept value and <= drop
        rest = np.setdiff1d(np.arange(t), kept)
        if rest.size:
            assert c[r, rest].max() <= drop[r] * (1 + 1e-4) + tol[r]
        # the true top entries are kept unless tied within tolerance of drop
        top = order[r, : min(8, t)]
        missing = np.setdiff1d(top, kept)
        for j in missing:
            assert c[r, j] <= drop[r] * (1 + 1e-4) + tol[r]
