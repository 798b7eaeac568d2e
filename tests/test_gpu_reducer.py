"""BucketwiseReducer (Algorithm 1 on a real model's gradients) at world size 1.

The reducer's result must equal sync_bucketwise over the model's flat
gradient with the reducer's own bucket layout (gradsync.py:148-162): within
1e-5 relative with an fp32 comm buffer, within one bf16 rounding with the
bf16 comm buffer.  B (and c/sqrt(B)) is fixed before the first backward.
"""

import copy

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import ClipConfig  # noqa: E402
from paper_2402_02447_b200.reducer import BucketwiseReducer  # noqa: E402


def model(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(
        torch.nn.Linear(64, 300), torch.nn.GELU(), torch.nn.Linear(300, 512), torch.nn.GELU(),
        torch.nn.Linear(512, 257), torch.nn.GELU(), torch.nn.Linear(257, 10)).cuda()


def batch(seed=1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(96, 64, device="cuda", generator=g), torch.randint(0, 10, (96,), device="cuda", generator=g)


def ref_grads(m, x, y, scale=1.0):
    m = copy.deepcopy(m)
    loss = torch.nn.functional.cross_entropy(m(x), y) * scale
    loss.backward()
    return torch.cat([p.grad.reshape(-1) for p in m.parameters()]).double().cpu().numpy()


@pytest.mark.parametrize("comm,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2.0 ** -8)])
@pytest.mark.parametrize("scale", [1.0, 1e-4])  # above and below the per-bucket limit
def test_reducer_matches_sync_bucketwise(comm, tol, scale):
    m = model()
    x, y = batch()
    flat_ref = ref_grads(m, x, y, scale)
    r = BucketwiseReducer(m.parameters(), ClipConfig(0.5, "bucket_wise"), bucket_cap_mb=0.1, comm_dtype=comm)
    assert len(r.layout) >= 3 and r.limit == 0.5 / np.sqrt(len(r.layout))  # B fixed before iteration 0
    for step in range(3):  # repeated steps: counters re-armed, grads zeroed in place
        r.zero_grad()
        loss = torch.nn.functional.cross_entropy(m(x), y) * scale
        loss.backward()
        r.finish()
        got = r.flat.double().cpu().numpy()
        ref = O.sync_bucketwise(flat_ref[None, :], r.layout, 0.5)
        assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), step
        # every parameter's .grad is its slice of the averaged, clipped flat gradient
        assert all(p.grad.data_ptr() >= r.flat.data_ptr() for p in m.parameters())
    assert r.fired_order[0] == len(r.layout) - 1  # backward fires the last bucket first
    norms = r.norms.cpu().numpy()
    np.testing.assert_allclose(norms, O.bucket_norms(flat_ref, r.layout), rtol=1e-6)


def test_reducer_unused_parameter_and_nonfinite():
    m = model()
    extra = torch.nn.Linear(8, 8).cuda()  # never used in forward: its bucket fires in finish()
    params = list(m.parameters()) + list(extra.parameters())
    r = BucketwiseReducer(params, ClipConfig(1.0, "bucket_wise"), bucket_cap_mb=0.2, comm_dtype=torch.float32)
    x, y = batch()
    loss = torch.nn.functional.cross_entropy(m(x), y)
    loss.backward()
    r.finish()
    assert torch.count_nonzero(extra.weight.grad) == 0 and sorted(r.fired_order) == list(range(len(r.layout)))
    r.zero_grad()
    loss = torch.nn.functional.cross_entropy(m(x), y) * float("inf")
    loss.backward()
    with pytest.raises(ValueError, match="non-finite"):
        r.finish()


@pytest.mark.parametrize("mode", ["bucketwise", "reducer", "presort"])
def test_train_step_modes_small_bert(mode):
    """The bench's training modes on a small BERT at world size 1: the DDP hook with B predicted
    before iteration 0 (must equal DDP's rebuilt count), the reducer (Algorithm 1, bf16 comm) and
    the reducer fed by the per-step batch former (K2 + native draws + LocalPresort/K3)."""
    pytest.importorskip("transformers")
    from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths
    from paper_2402_02447_b200.train_step import bert_large_step_bench

    small = dict(vocab_size=1024, hidden_size=128, num_hidden_layers=2, num_attention_heads=2,
                 intermediate_size=256, max_position_embeddings=128)
    lens = generate_lengths(LengthDistribution(), 50_000, 3)
    import torch.distributed as dist

    try:
        r = bert_large_step_bench(mode, steps=2, warmup=2, batch=8, seq=128, bucket_cap_mb=1, lengths=lens,
                                  model_config=small)
    finally:
        if dist.is_initialized():  # the step bench initialised a world-size-1 NCCL group
            dist.destroy_process_group()
    assert np.isfinite(r["loss"]) and r["samples_per_s"] > 0
    if mode == "bucketwise":
        assert r["buckets_iter0"]["predicted"] == r["buckets_iter0"]["ddp"]
        assert r["buckets_after_rebuild"]["predicted"] == r["buckets_after_rebuild"]["ddp"]
    else:
        assert r["buckets"] >= 2
