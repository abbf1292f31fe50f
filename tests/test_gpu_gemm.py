"""The library's GEMMs (csrc/gemm_tc.cu tcgen05 + TMA, csrc/gemm_simt.cu
CUDA-core) against a plain PyTorch fp32 reference of the same op.

Operands are bf16 (exact in fp32), so the fp32 reference differs from the
tensor-core result only by accumulation order: fp32 outputs must agree to
1e-4 of max|ref| and bf16 outputs to one bf16 rounding (1e-2).  Covered: every
transpose combination, M / N / K tails, the engine's shapes at the bench
configuration, the fused bias / ReLU / residual / beta epilogues, the
channel-batched (TriangleMultiplication) form and the split-K path."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


def _tc_count():
    from paper_2207_05477_b200 import _lib
    return _lib.lib().evo_gemm_tc_launches()


def _operands(M, N, K, ta, tb, dt=torch.bfloat16, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((K, M) if ta else (M, K), device="cuda", generator=g).to(dt)
    b = torch.randn((N, K) if tb else (K, N), device="cuda", generator=g).to(dt)
    ref = (a.float().t() if ta else a.float()) @ (b.float().t() if tb else b.float())
    return a, b, ref


def _err(x, ref):
    return float((x.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))


SHAPES = [
    # (M, N, K): engine shapes at the bench configuration ...
    (32768, 1024, 256), (32768, 256, 256), (65536, 512, 128), (65536, 128, 128),
    (32768, 64, 256), (65536, 128, 1024), (32768, 256, 1024), (32768, 256, 64),
    # ... and tails in every dimension
    (1000, 192, 72), (129, 64, 16), (77, 320, 200), (256, 8, 64),
]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_gemm_nn_nt_matches_torch(M, N, K, out):
    from paper_2207_05477_b200 import ops
    odt = torch.bfloat16 if out == "bf16" else torch.float32
    for tb in (False, True):
        a, b, ref = _operands(M, N, K, False, tb)
        c = torch.empty((M, N), device="cuda", dtype=odt)
        ops.gemm(a, b, c, tb=tb)
        assert _err(c, ref) <= (1e-2 if out == "bf16" else 1e-4), (tb, _err(c, ref))


@pytest.mark.parametrize("M,N,K", [(256, 1024, 32768), (1024, 256, 32768), (128, 512, 65536),
                                   (1024, 128, 65536), (256, 64, 32768), (200, 136, 5000)])
def test_gemm_weight_gradient_split_k(M, N, K):
    """ta=True, K = tokens: the split-K path, fp32 out, with and without beta."""
    from paper_2207_05477_b200 import ops
    a, b, ref = _operands(M, N, K, True, False)
    c = torch.empty((M, N), device="cuda")
    n0 = _tc_count()
    ops.gemm(a, b, c, ta=True)
    assert _tc_count() > n0
    assert _err(c, ref) <= 1e-4
    c0 = torch.randn_like(c)
    c1 = c0.clone()
    ops.gemm(a, b, c1, ta=True, beta=1.0)
    assert _err(c1, ref + c0) <= 1e-4
    # deterministic: the same call gives the same bits
    c2 = torch.empty_like(c)
    ops.gemm(a, b, c2, ta=True)
    assert torch.equal(c, c2)


@pytest.mark.parametrize("ta,tb", [(True, True), (True, False)])
def test_gemm_transposed_a(ta, tb):
    from paper_2207_05477_b200 import ops
    for (M, N, K) in [(128, 8192, 8192), (300, 200, 500), (64, 64, 64)]:
        a, b, ref = _operands(M, N, K, ta, tb)
        c = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
        ops.gemm(a, b, c, ta=ta, tb=tb)
        assert _err(c, ref) <= 1e-2, (M, N, K, ta, tb)


@pytest.mark.parametrize("M,N,K", [(32768, 256, 256), (32768, 1024, 256), (65536, 128, 1024), (1000, 136, 72)])
def test_gemm_bias_epilogues(M, N, K):
    from paper_2207_05477_b200 import ops
    a, b, ref = _operands(M, N, K, False, False)
    bias = torch.randn(N, device="cuda")
    res = torch.randn((M, N), device="cuda").to(torch.bfloat16)
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    n0 = _tc_count()
    ops.gemm_bias(a, b, out, bias, res=res)
    assert _tc_count() > n0
    assert _err(out, ref + bias + res.float()) <= 1e-2
    ops.gemm_bias(a, b, out, bias, relu=True)
    assert _err(out, torch.relu(ref + bias)) <= 1e-2
    out32 = torch.empty((M, N), device="cuda")
    res32 = torch.randn((M, N), device="cuda")
    ops.gemm_bias(a.float(), b.float(), out32, bias, res=res32)   # fp32: CUDA-core kernel
    assert _err(out32, ref + bias + res32) <= 1e-4


def test_gemm_strided_output_and_beta_accumulate():
    """Column-sliced output (ld > N) and beta=1 accumulation into fp32 (dzl +=)."""
    from paper_2207_05477_b200 import ops
    M, N, K = 4096, 128, 512
    a, b, ref = _operands(M, N, K, False, True)
    big = torch.zeros((M, 3 * N), device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, big[:, N:2 * N], tb=True)
    assert _err(big[:, N:2 * N], ref) <= 1e-2
    assert big[:, :N].abs().max() == 0 and big[:, 2 * N:].abs().max() == 0
    acc = torch.randn((M, N), device="cuda")
    expect = acc + ref
    ops.gemm(a, b, acc, tb=True, beta=1.0)
    assert _err(acc, expect) <= 1e-4


@pytest.mark.parametrize("ta,tb", [(False, True), (True, False), (False, False)])
def test_gemm_batched_trimul_form(ta, tb):
    """The channel-batched contractions of TriangleMultiplication: batch of
    R x R matrices at stride R*R (channel-major), bf16 out."""
    from paper_2207_05477_b200 import ops
    R, ch = 256, 16
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((ch, R, R), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn((ch, R, R), device="cuda", generator=g).to(torch.bfloat16)
    O = torch.empty((ch, R, R), device="cuda", dtype=torch.bfloat16)
    ops.gemm_batched(A[0], B[0], O[0], ch, R * R, R * R, R * R, ta=ta, tb=tb)
    Af = A.float().transpose(1, 2) if ta else A.float()
    Bf = B.float().transpose(1, 2) if tb else B.float()
    assert _err(O, Af @ Bf) <= 1e-2


def test_gemm_fp32_is_true_fp32():
    """fp32 operands use FFMA (no TF32): a product TF32 would round is exact."""
    from paper_2207_05477_b200 import ops
    # 1 + 2^-12 needs 12 mantissa bits (TF32 keeps 10); every partial sum
    # k (1 + 2^-12), k <= 8, is exact in fp32
    a = torch.full((64, 8), 1.0 + 2 ** -12, device="cuda")
    b = torch.ones((8, 64), device="cuda")
    c = torch.empty((64, 64), device="cuda")
    ops.gemm(a, b, c)
    assert torch.all(c == 8 * (1.0 + 2 ** -12))


@pytest.mark.parametrize("M,N,K", [(8, 128, 65536), (8, 256, 32768), (100, 36, 4100)])
def test_gemm_fp32_split_k(M, N, K):
    """The embedding weight gradients (fp32, 8 x C outputs, K = tokens) take
    the CUDA-core kernel's split-K path; deterministic and true fp32."""
    from paper_2207_05477_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((K, M), device="cuda", generator=g)
    b = torch.randn((K, N), device="cuda", generator=g)
    ref = a.double().t() @ b.double()
    c = torch.empty((M, N), device="cuda")
    ops.gemm(a, b, c, ta=True)
    assert float((c.double() - ref).abs().max() / ref.abs().max()) <= 1e-5
    c2 = torch.full_like(c, 1.0)
    ops.gemm(a, b, c2, ta=True, beta=1.0)
    assert float((c2.double() - ref - 1.0).abs().max() / ref.abs().max()) <= 1e-5
    c3 = torch.empty_like(c)
    ops.gemm(a, b, c3, ta=True)
    assert torch.equal(c, c3)


@pytest.mark.parametrize("M,N,K", [(4096, 1024, 256), (8192, 512, 128), (1000, 384, 64)])
def test_gemm_relu_mask_epilogue(M, N, K):
    """D = (h > 0) * (A B^T): the transition's ReLU backward in the GEMM
    epilogue (the mask tile fetched by TMA like a residual) == fp32 torch,
    masked entries exactly zero."""
    from paper_2207_05477_b200 import ops
    torch.manual_seed(M + N)
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    h = torch.relu(torch.randn(M, N, device="cuda")).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.full((N,), 7.0, device="cuda")
    ops.gemm_relu_mask(a, b, h, out, tb=True, colsum=cs)
    ref = (a.float() @ b.float().t()) * (h.float() > 0)
    assert torch.all(out[h == 0] == 0)
    err = (out.float() - ref).abs().max() / ref.abs().max()
    assert err <= 1e-2, float(err)
    # the epilogue's column sums are those of the stored bf16 values
    want = out.double().sum(0).float()
    assert float((cs - want).abs().max() / want.abs().max()) <= 1e-5
    acc = cs.clone()
    ops.gemm_relu_mask(a, b, h, out, tb=True, colsum=acc, accumulate=True)
    assert float((acc - 2 * cs).abs().max() / cs.abs().max()) <= 1e-6
