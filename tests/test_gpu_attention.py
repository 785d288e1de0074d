"""GPU parity of AG-KV fused with Q.K^T (BASELINE config 3)."""

import numpy as np
import pytest
import torch

from tests._devices import devices_for

from oracle import attention as OA
from oracle import collectives as OC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _ctx(world, **kw):
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    args = dict(block_m=256, block_n=256, group_m=4, num_gemm_sms=0, num_comm_sms=0,
                devices=devices_for(world))
    args.update(kw)
    return WorkloadContext(topology=build_topology(world, 1), **args)


@pytest.mark.parametrize("world,sl,hq,hkv,d", [(1, 64, 2, 1, 16), (2, 100, 4, 2, 8), (4, 96, 8, 2, 128),
                                               (8, 128, 8, 1, 64), (2, 33, 2, 2, 5)])
@pytest.mark.parametrize("bn", [128, 256])
def test_ag_kv_scores_exact(world, sl, hq, hkv, d, bn):
    from paper_2605_02953_b200.attention import ag_kv_scores
    rng = np.random.default_rng(world * 1000 + sl + d)
    q = [rng.integers(-8, 8, (sl, hq, d)) for _ in range(world)]
    k = [rng.integers(-8, 8, (sl, hkv, d)) for _ in range(world)]
    run = ag_kv_scores(q, k, _ctx(world, block_n=bn))
    want = OA.ref_ag_kv_scores(q, k, hkv)
    for r in range(world):
        assert run.outputs[r].shape == (hq, sl, sl * world)
        assert np.array_equal(run.outputs[r], want[r]), r


@pytest.mark.parametrize("world", [1, 4, 8])
def test_ag_kv_scores_bf16_tolerance(world):
    from paper_2605_02953_b200.attention import ag_kv_scores
    rng = np.random.default_rng(world)
    sl, hq, hkv, d = 256, 8, 2, 128
    q = [torch.from_numpy(rng.standard_normal((sl, hq, d)).astype(np.float32)).to(torch.bfloat16).cuda()
         for _ in range(world)]
    k = [torch.from_numpy(rng.standard_normal((sl, hkv, d)).astype(np.float32)).to(torch.bfloat16).cuda()
         for _ in range(world)]
    run = ag_kv_scores(q, k, _ctx(world))
    want = OA.ref_ag_kv_scores([x.float().cpu().numpy() for x in q], [x.float().cpu().numpy() for x in k], hkv)
    for r in range(world):
        assert run.outputs[r].dtype == torch.bfloat16
        assert OC.compare(run.outputs[r].float().cpu().numpy(), want[r]) <= 2e-2


def test_ag_kv_scores_validation():
    from paper_2605_02953_b200.attention import ag_kv_scores
    rng = np.random.default_rng(0)
    q = [rng.integers(-8, 8, (8, 3, 8)) for _ in range(2)]
    k = [rng.integers(-8, 8, (8, 2, 8)) for _ in range(2)]
    with pytest.raises(ValueError):
        ag_kv_scores(q, k, _ctx(2))  # 3 query heads over 2 kv heads
    with pytest.raises(ValueError):
        ag_kv_scores(q[:1], k, _ctx(2))


# -- fused AG-KV flash-attention forward ------------------------------


@pytest.mark.parametrize("world,sl,hq,hkv", [(1, 128, 1, 1), (1, 256, 2, 1), (2, 128, 4, 2),
                                             (4, 256, 8, 1), (8, 128, 8, 8),
                                             (1, 512, 2, 1), (2, 512, 4, 2), (4, 1024, 8, 2)])
# TF_ATTN_PAIR=1: CTA-pair kernel, two query tiles per CTA (s_local % 512 == 0);
# TF_ATTN_PAIR=2: CTA-pair kernel, one query tile per CTA and S double-buffered (s_local % 256 == 0)
@pytest.mark.parametrize("pair", ["0", "1", "2"])
def test_ag_kv_attention_vs_oracle(world, sl, hq, hkv, pair, monkeypatch):
    monkeypatch.setenv("TF_ATTN_PAIR", pair)
    from paper_2605_02953_b200.attention import ag_kv_attention
    rng = np.random.default_rng(world * 7 + sl + hq)
    d = 128
    mk = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16).cuda()
    q = [mk(sl, hq, d) for _ in range(world)]
    k = [mk(sl, hkv, d) for _ in range(world)]
    v = [mk(sl, hkv, d) for _ in range(world)]
    run = ag_kv_attention(q, k, v, _ctx(world))
    want = OA.ref_ag_kv_attention([x.float().cpu().numpy() for x in q], [x.float().cpu().numpy() for x in k],
                                  [x.float().cpu().numpy() for x in v], hkv, d ** -0.5)
    for r in range(world):
        got = run.outputs[r].float().cpu().numpy()
        assert np.isfinite(got).all()
        assert OC.compare(got, want[r]) <= 2e-2, r


@pytest.mark.parametrize("pair", ["0", "2"])
def test_ag_kv_attention_peaked_scores_rescaling(pair, monkeypatch):
    """Large, growing logits force the online-softmax rescale path every tile."""
    monkeypatch.setenv("TF_ATTN_PAIR", pair)
    from paper_2605_02953_b200.attention import ag_kv_attention
    rng = np.random.default_rng(11)
    world, sl, hq, hkv, d = 2, 256, 2, 1, 128
    q = [torch.from_numpy(rng.standard_normal((sl, hq, d)).astype(np.float32) * 3).to(torch.bfloat16).cuda()
         for _ in range(world)]
    ramp = np.linspace(0.2, 4.0, sl * world).astype(np.float32)
    kk = rng.standard_normal((sl * world, hkv, d)).astype(np.float32) * ramp[:, None, None]
    k = [torch.from_numpy(kk[r * sl:(r + 1) * sl]).to(torch.bfloat16).cuda() for r in range(world)]
    v = [torch.from_numpy(rng.standard_normal((sl, hkv, d)).astype(np.float32)).to(torch.bfloat16).cuda()
         for _ in range(world)]
    run = ag_kv_attention(q, k, v, _ctx(world))
    want = OA.ref_ag_kv_attention([x.float().cpu().numpy() for x in q], [x.float().cpu().numpy() for x in k],
                                  [x.float().cpu().numpy() for x in v], hkv, d ** -0.5)
    for r in range(world):
        assert OC.compare(run.outputs[r].float().cpu().numpy(), want[r]) <= 2e-2
