"""The tcgen05 GEMM core against a torch fp32 reference (bf16 inputs)."""

import pytest

torch = pytest.importorskip("torch")

from paper_2504_19442_b200 import _lib  # noqa: E402
from paper_2504_19442_b200.pipelines import gemm  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-2  # relative Frobenius error vs fp32 (BASELINE.json north_star)


def rel_fro(x, ref):
    return (x.float() - ref).norm().item() / max(ref.norm().item(), 1e-30)


@pytest.fixture(autouse=True)
def _default_cfg():
    yield
    _lib.check(_lib.load().sh_set_tile_config(0, 0))


@pytest.mark.parametrize("bn,cg", [(512, 2), (256, 2), (224, 2), (128, 2), (256, 1), (128, 1)])
@pytest.mark.parametrize("m,n,k", [(256, 256, 64), (512, 512, 512), (1024, 768, 1024),
                                   (384, 320, 200), (1000, 520, 136), (1024, 1536, 8448)])
def test_gemm_matches_fp32(bn, cg, m, n, k):
    _lib.check(_lib.load().sh_set_tile_config(bn, cg))
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
    c = gemm(a, b)
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    assert rel_fro(c, ref) < TOL


def test_gemm_exact_small_integers():
    # integer-valued bf16 operands with |sum| < 256 are exact end to end
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randint(-3, 4, (512, 256), device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randint(-1, 2, (256, 384), device="cuda", generator=g).to(torch.bfloat16)
    c = gemm(a, b).float()
    ref = a.float() @ b.float()
    assert ref.abs().max() < 256
    assert torch.equal(c, ref)


def test_gemm_fp16():
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(768, 512, device="cuda", generator=g).half()
    b = torch.randn(512, 640, device="cuda", generator=g).half()
    c = gemm(a, b)
    assert rel_fro(c, a.float() @ b.float()) < TOL


def test_gemm_large_llama_shape():
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.randn(2048, 8192, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(8192, 3584, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    c = gemm(a, b)
    assert rel_fro(c, a.float() @ b.float()) < TOL


@pytest.mark.parametrize("sk", ["0", "1"])
@pytest.mark.parametrize("m,n,k", [(2560, 2048, 1024), (2560, 2048, 136), (2304, 2304, 2048)])
def test_gemm_stream_k_tail(monkeypatch, sk, m, n, k):
    # 80+ tiles on 74 CTA pairs: the stream-K tail splits tiles by k-block and
    # the finishing cluster adds the fp32 partials of the others
    monkeypatch.setenv("SHB_SK", sk)
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
    for _ in range(3):  # repeated launches reuse the workspace (epoch-tagged flags)
        c = gemm(a, b)
    assert rel_fro(c, a.float() @ b.float()) < TOL


@pytest.mark.parametrize("dyn,wave", [("0", "0"), ("1", "0"), ("0", "1")])
def test_gemm_stream_k_exact_integers(monkeypatch, dyn, wave):
    # dyn=1: data-parallel tiles handed out by the atomic counter (opt-in);
    # wave=1: wave lockstep of the data-parallel tiles (opt-in)
    monkeypatch.setenv("SHB_SK", "1")
    monkeypatch.setenv("SHB_DYN", dyn)
    monkeypatch.setenv("SHB_WAVE", wave)
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randint(-2, 3, (2560, 1024), device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randint(-1, 2, (1024, 2048), device="cuda", generator=g).to(torch.bfloat16)
    ref = a.float() @ b.float()
    assert ref.abs().max() < 256
    assert torch.equal(gemm(a, b).float(), ref)
