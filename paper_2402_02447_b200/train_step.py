"""BERT-large training step with the three clip disciplines.

MLPerf BERT phase-2 shape: seq 512, local batch 48, bf16 autocast, fp32
master gradients in DDP's 25 MiB buckets, AdamW.  Modes:
  * ``stock``      — DDP allreduce, no clipping (speed ceiling);
  * ``after``      — DDP allreduce, then global-norm clip of the mean
                     (clip after allreduce, gradsync.py:131-134 semantics);
  * ``bucketwise`` — the paper's method: DDP comm hook clips each bucket at
                     c/sqrt(B) with K1 before its allreduce
                     (sync_bucketwise, gradsync.py:148-162; Algorithm 1).
Synthetic token ids and random-init weights (no network).  Returns
samples/s over the timed steps (CUDA events, max over ranks).
"""

from __future__ import annotations

import math
import os

import torch
import torch.distributed as dist

from .ddp import bucketwise_clip_hook, make_hook_state
from .gradsync import ClipConfig

BERT_LARGE = dict(vocab_size=30528, hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                  intermediate_size=4096, max_position_embeddings=512)


def _batch(batch: int, seq: int, device, gen):
    ids = torch.randint(0, BERT_LARGE["vocab_size"], (batch, seq), device=device, generator=gen)
    labels = torch.where(torch.rand(batch, seq, device=device, generator=gen) < 0.15, ids, torch.full_like(ids, -100))
    return {
        "input_ids": ids,
        "attention_mask": torch.ones_like(ids),
        "token_type_ids": torch.zeros_like(ids),
        "labels": labels,
        "next_sentence_label": torch.randint(0, 2, (batch,), device=device, generator=gen),
    }


def bert_large_step_bench(mode: str = "bucketwise", steps: int = 5, warmup: int = 2, batch: int = 48,
                          seq: int = 512, clip: float = 1.0, bucket_cap_mb: int = 25) -> dict:
    from torch.nn.parallel import DistributedDataParallel as DDP
    from transformers import BertConfig, BertForPreTraining

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29600 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", torch.cuda.current_device()))
    dev = torch.device("cuda", torch.cuda.current_device())
    world = dist.get_world_size()
    torch.manual_seed(1234)
    cfg = BertConfig(**BERT_LARGE)
    cfg._attn_implementation = "sdpa"
    model = BertForPreTraining(cfg).to(dev)
    ddp = DDP(model, device_ids=[dev.index], bucket_cap_mb=bucket_cap_mb, gradient_as_bucket_view=True)
    state = None
    if mode == "bucketwise":
        n_params = sum(p.numel() for p in model.parameters())
        guess = max(1, math.ceil(n_params * 4 / (bucket_cap_mb * 1024 * 1024)))
        state = make_hook_state(ClipConfig(clip, "bucket_wise"), guess)
        ddp.register_comm_hook(state, bucketwise_clip_hook)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + dist.get_rank())
    data = _batch(batch, seq, dev, gen)

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = ddp(**data).loss
        loss.backward()
        if mode == "after":
            torch.nn.utils.clip_grad_norm_(model.parameters(), clip)
        opt.step()
        opt.zero_grad(set_to_none=False)
        return loss

    for _ in range(warmup):
        step()
    if state is not None:  # DDP rebuilt its buckets after iteration 1: fix B = c/sqrt(B)'s B
        state.set_num_buckets(max(state.norms) + 1 if state.norms else 1)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        loss = step()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out = {"mode": mode, "ms_per_step": ms, "samples_per_s": world * batch / (ms * 1e-3), "world": world,
           "batch_per_gpu": batch, "seq": seq, "loss": float(loss), "params": sum(p.numel() for p in model.parameters())}
    if state is not None:
        out["buckets"] = state.num_buckets
    del ddp, model, opt
    torch.cuda.empty_cache()
    return out
