"""K5/K6 parity: the fused row pass of the iterations
through lsrn_debug_rowpass, against the plain fp64 definition on the same inputs:
    z_new = c1 z + c2 sx (Y t),  acc += ca z_new,  out = [sx Y^T z_new ; ||z_new||^2].
Shapes cover every kernel plan: one CTA per row slice (2 CTAs per SM, register
tile kept or not), 2- and 3-CTA clusters for rows wider than 4096 doubles, the
8-byte fallback for odd leading dimensions, ragged row tiles."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    c = lsrn.Context()
    yield c
    c.close()


@pytest.mark.parametrize("R,C,pad", [(3000, 100, 0), (5001, 2000, 0), (999, 33, 1), (777, 4096, 0),
                                     (700, 4100, 0), (333, 10000, 0), (150, 20000, 0), (90, 17001, 1), (120, 30000, 0),
                                     (64, 8193, 2)])
def test_rowpass_vs_definition(ctx, R, C, pad):
    g = torch.Generator().manual_seed(R + C)
    Yfull = torch.randn(R, C + pad, generator=g, dtype=torch.float64)
    Y = Yfull[:, :C]
    t = torch.randn(C, generator=g, dtype=torch.float64)
    z = torch.randn(R, generator=g, dtype=torch.float64)
    acc = torch.randn(R, generator=g, dtype=torch.float64)
    c1, c2, ca, sx = 0.7, -1.3, 0.4, 0.9
    Yd = Yfull.cuda()[:, :C]
    zd, accd, td = z.cuda(), acc.cuda(), t.cuda()
    out, _ = ctx.debug_rowpass(Yd, td, zd, (c1, c2, ca), sx=sx, acc=accd)
    Yn, tn = Y.numpy(), t.numpy()
    zn = c1 * z.numpy() + c2 * sx * (Yn @ tn)
    accn = acc.numpy() + ca * zn
    wn = sx * (Yn.T @ zn)
    scale_z = np.abs(c1 * z.numpy()) + np.abs(c2 * sx) * (np.abs(Yn) @ np.abs(tn))
    assert np.max(np.abs(zd.cpu().numpy() - zn) / scale_z) <= 1e-14
    assert np.max(np.abs(accd.cpu().numpy() - accn) / (np.abs(acc.numpy()) + np.abs(ca) * scale_z)) <= 1e-14
    scale_w = np.abs(sx) * (np.abs(Yn).T @ np.abs(zn))
    o = out.cpu().numpy()
    assert np.max(np.abs(o[:C] - wn) / scale_w) <= 1e-13
    assert abs(o[C] - zn @ zn) <= 1e-13 * (zn @ zn)


def test_rowpass_deterministic(ctx):
    g = torch.Generator().manual_seed(5)
    Y = torch.randn(500, 10000, generator=g, dtype=torch.float64).cuda()
    t = torch.randn(10000, generator=g, dtype=torch.float64).cuda()
    z0 = torch.randn(500, generator=g, dtype=torch.float64).cuda()
    outs = []
    for _ in range(2):
        z = z0.clone()
        out, _ = ctx.debug_rowpass(Y, t, z, (0.5, 1.0, 0.0))
        outs.append((out.cpu(), z.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
