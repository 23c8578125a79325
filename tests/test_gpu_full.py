"""Parity at BASELINE.json's full sizes (C2, C3, C4), where the CPU oracle is
too slow: size-independent properties of the result and an independent FP64
factorization on the same device (cuSOLVER through torch: potrf + potri for
one matrix, getrf/getri for the batch) as the comparison.

Tolerances (north_star): normwise max|X - R| / max|R| <= 1e-10 * cond(A);
residual ||I - A X||_1 / (n ||A||_1 ||X||_1 eps) = O(1) (< 10); the result is
bitwise symmetric and bitwise reproducible run to run.
"""

import numpy as np
import pytest
import torch

import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if _native.device_count() < 1:
        pytest.fail("no B200 visible: the GPU tests must run on the GPU box")


def spd_device(n, shift=1.0, seed=0):
    """A = G G^T / n + shift I, G iid N(0,1) (torch Philox on the device), bitwise symmetric."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    a = torch.matmul(g, g.T)
    del g
    a.div_(n)
    a.diagonal().add_(shift)
    return torch.tril(a) + torch.tril(a, -1).T


def run_device(a, nb, cfg):
    n = a.shape[0]
    t = n // nb
    ctx = _native.Context(n, nb)
    s = P.gen_inversion(t, cfg)
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
    assert plan.rc == 0, plan.msg
    outs = []
    for _ in range(2):
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, ms = plan.run()
        assert rc == 0, plan.msg
        x = torch.empty_like(a)
        ctx.get_dense_device(x.data_ptr(), n, _native.DENSE_SYMMETRIZE)
        outs.append(x)
    plan.close()
    ctx.close()
    return outs


def residual_cols(a, x, cols):
    n = a.shape[0]
    r = a @ x[:, cols]
    r[cols, torch.arange(len(cols), device="cuda")] -= 1.0
    return float(r.abs().sum(0).max() / (n * a.abs().sum(0).max() * x.abs().sum(0).max() * EPS))


@pytest.mark.parametrize("n,nb,cfg", [
    (8192, 256, P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True)),    # BASELINE config 2
    (32768, 512, P.VariantConfig(P.Placement.OUT_OF_PLACE, "DDU", True)),   # config 3, the bench default
])
def test_full_size_inversion_properties_and_cusolver(n, nb, cfg):
    a = spd_device(n)
    x, x2 = run_device(a, nb, cfg)
    assert torch.equal(x, x2)  # bitwise reproducible
    cols = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(1))[:256]
    assert torch.equal(x[cols, :], x[:, cols].T)  # bitwise symmetric (sampled rows / columns)
    assert residual_cols(a, x, cols) < 10
    del x2
    torch.cuda.empty_cache()
    ref = torch.cholesky_inverse(torch.linalg.cholesky(a))  # cuSOLVER potrf + potri, FP64
    cond = float(a.abs().sum(0).max() * ref.abs().sum(0).max())  # 1-norm condition number of A
    rel = float((x - ref).abs().max() / ref.abs().max())
    assert rel <= 1e-10 * cond


def test_full_size_steps_vs_cusolver():
    """BASELINE config 2's per-step entry points at full size: L = POTRF(A),
    L^-1 = TRTRI(L), A^-1 = LAUUM(L^-1) against cuSOLVER's factor / inverses."""
    n, nb = 8192, 256
    t = n // nb
    a = spd_device(n)
    l_ref = torch.linalg.cholesky(a)
    linv_ref = torch.linalg.solve_triangular(l_ref, torch.eye(n, dtype=torch.float64, device="cuda"), upper=False)
    ctx = _native.Context(n, nb)

    def step(stream, src):
        plan = _native.Plan(ctx, stream.table(), t, np.zeros(0, np.int64))
        ctx.put_dense_device(src.data_ptr(), n)
        rc, err, _ = plan.run()
        assert rc == 0, plan.msg
        plan.close()
        out = torch.empty_like(src)
        ctx.get_dense_device(out.data_ptr(), n, _native.DENSE_LOWER)
        return torch.tril(out)

    lo = step(P.gen_step1(t, "U"), a)
    assert float((lo - l_ref).abs().max() / l_ref.abs().max()) < 1e-12
    li = step(P.gen_step2(t, "D", P.Placement.OUT_OF_PLACE), lo)
    assert float((li - linv_ref).abs().max() / linv_ref.abs().max()) < 1e-11
    ai = step(P.gen_step3(t, "U", P.Placement.OUT_OF_PLACE), li)
    ref = torch.tril(linv_ref.T @ linv_ref)
    assert float((ai - ref).abs().max() / ref.abs().max()) < 1e-11
    ctx.close()


@pytest.mark.parametrize("engine", ["cta", "pipe"])
def test_full_size_batched_c4_vs_cusolver(engine):
    """BASELINE config 4 (8192 x n=256) through the fused engine: bitwise
    symmetric and reproducible, normwise against cuSOLVER's batched inverse."""
    B, n = 8192, 256
    gen = torch.Generator(device="cuda").manual_seed(0)
    g = torch.randn(B, n, n, dtype=torch.float64, device="cuda", generator=gen)
    a = torch.bmm(g, g.transpose(1, 2)) / n
    del g
    a.diagonal(dim1=1, dim2=2).add_(1.0)
    a = torch.tril(a) + torch.tril(a, -1).transpose(1, 2)
    fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    xs = []
    prev = _native.batch_engine(engine)
    for _ in range(2):
        x = torch.empty_like(a)
        _native.batch_small_launch(a.data_ptr(), x.data_ptr(), B, n, n * n, st, fail.data_ptr())
        torch.cuda.synchronize()
        assert int(fail.item()) == -1
        xs.append(x)
    _native.batch_engine(prev)
    x = xs[0]
    assert torch.equal(x, xs[1])
    assert torch.equal(x, x.transpose(1, 2))
    ref = torch.linalg.inv(a)
    cond = a.abs().sum(1).amax(1) * ref.abs().sum(1).amax(1)  # per-matrix 1-norm condition numbers
    rel = (x - ref).abs().amax(dim=(1, 2)) / ref.abs().amax(dim=(1, 2))
    assert bool((rel <= 1e-10 * cond).all())
    k = torch.arange(0, B, 97, device="cuda")
    r = torch.bmm(a[k], x[k]) - torch.eye(n, dtype=torch.float64, device="cuda")
    res = r.abs().sum(1).amax(1) / (n * a[k].abs().sum(1).amax(1) * x[k].abs().sum(1).amax(1) * EPS)
    assert float(res.max()) < 10
