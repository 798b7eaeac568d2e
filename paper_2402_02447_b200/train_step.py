"""BERT-large training step with the three clip disciplines.

MLPerf BERT phase-2 shape: seq 512, local batch 48, bf16 autocast, fp32
master gradients in 25 MiB buckets, AdamW.  Modes:
  * ``stock``      — DDP allreduce, no clipping (speed ceiling);
  * ``after``      — DDP allreduce, then global-norm clip of the mean
                     (clip after allreduce, gradsync.py:131-134 semantics);
  * ``bucketwise`` — DDP comm hook clips each DDP bucket at c/sqrt(B) with K1
                     before its fp32 allreduce; B is DDP's rebuilt bucket
                     count, predicted before iteration 0 from DDP's own
                     assignment rule (first bucket 1 MiB, then 25 MiB, in
                     backward order);
  * ``reducer``    — the paper's Algorithm 1 without DDP: ``BucketwiseReducer``
                     (own 25 MiB layout, B known up front, K1 clip + cast into
                     a bf16 comm buffer as each bucket's gradients land,
                     ncclAllReduce on a side stream, overlapped with backward);
  * ``presort``    — ``reducer`` fed by the paper's batch former every step:
                     per-rank stratified draws (NativeDraws, strata.py:113-161)
                     from a K2-stratified rank shard of the 10M Wikipedia-like
                     corpus, the node's local presort (LocalPresort: all-gather
                     + K3, balance.py:158-184), the dealt samples' lengths as
                     the attention masks (config 4 of BASELINE.json).
Synthetic token ids and random-init weights (no network).  Returns
samples/s over the timed steps (CUDA events, max over ranks).
"""

from __future__ import annotations

import math
import os
import time

import torch
import torch.distributed as dist

import numpy as np

from .ddp import bucketwise_clip_hook, make_hook_state
from .gradsync import ClipConfig
from .reducer import BucketwiseReducer

BERT_LARGE = dict(vocab_size=30528, hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                  intermediate_size=4096, max_position_embeddings=512)


def _batch(batch: int, seq: int, device, gen, vocab: int = BERT_LARGE["vocab_size"]):
    ids = torch.randint(0, vocab, (batch, seq), device=device, generator=gen)
    labels = torch.where(torch.rand(batch, seq, device=device, generator=gen) < 0.15, ids, torch.full_like(ids, -100))
    return {
        "input_ids": ids,
        "attention_mask": torch.ones_like(ids),
        "token_type_ids": torch.zeros_like(ids),
        "labels": labels,
        "next_sentence_label": torch.randint(0, 2, (batch,), device=device, generator=gen),
    }


def ddp_bucket_counts(ddp, ready_order=None) -> int:
    """B of DDP's bucket layout, from DDP's own assignment rule
    (torch.distributed._compute_bucket_assignment_by_size with the size limits DDP passes it).
    ready_order None: iteration 0's layout (registration order; with find_unused_parameters=False
    DDP puts everything in ONE bucket for iteration 0).  Otherwise: the layout DDP rebuilds
    before iteration 1 from the order gradients became ready in iteration 0."""
    import sys

    first = dist._DEFAULT_FIRST_BUCKET_BYTES if ddp.bucket_bytes_cap_default else ddp.bucket_bytes_cap
    caps = list(getattr(ddp, "bucket_bytes_cap_list", None) or [])
    if ready_order is None:
        params = [p for p in ddp.module.parameters() if p.requires_grad]
        if caps:
            limits = caps
        elif getattr(ddp, "static_graph", False) or not ddp.find_unused_parameters:
            limits = [sys.maxsize]
        else:
            limits = [first, ddp.bucket_bytes_cap] if ddp.bucket_bytes_cap_default else [ddp.bucket_bytes_cap]
    else:
        params = list(ready_order)
        limits = caps or [first, ddp.bucket_bytes_cap]
    buckets, _ = dist._compute_bucket_assignment_by_size(params, limits, [False] * len(params))
    return len(buckets)


class PresortBatches:
    """The paper's batch former on the device path, one local batch per step for this rank.

    Rank r of a Topology(1, gpus) node owns the contiguous shard r of the corpus;
    its strata come from K2 (stratify_lengths), each step draws ``lb`` samples
    with seed derive_seed(seed, r, step) (NativeDraws, bit-exact draw_batch),
    LocalPresort all-gathers the node's draws and deals them with K3, and the
    rank's dealt lengths become the batch's attention mask.
    """

    def __init__(self, lengths: np.ndarray, local_batch: int, seq: int, seed: int = 2402):
        from .presort_dist import LocalPresort
        from .seqdata import Topology
        from .strata import NativeDraws, allocate_counts, stratify_lengths

        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        n = lengths.size // self.world
        off = self.rank * n
        shard = np.ascontiguousarray(lengths[off:off + n], dtype=np.int32)
        ds = stratify_lengths(shard)  # K2
        o = np.concatenate([[0], np.cumsum(ds.counts)])
        ids = ds.ids.cpu().numpy().astype(np.int64) + off
        self.nd = NativeDraws([ids[o[k]:o[k + 1]] for k in range(len(ds.counts))], ds.boundaries)
        self.counts = allocate_counts(ds.probs, local_batch).counts
        self.lengths = lengths
        self.d_lengths = torch.from_numpy(np.ascontiguousarray(lengths, dtype=np.int32)).cuda()
        self.lp = LocalPresort(Topology(1, self.world), local_batch, int(lengths.max()), int(lengths.size - 1),
                               deferred_check=True)
        self.seed, self.seq, self.step_i = seed, seq, 0
        self.pos = torch.arange(seq, device="cuda")
        # pinned staging ring: the H2D of step t is truly asynchronous, and slot t is rewritten
        # only after its copy has run (event), so the host never waits on the GPU queue
        self.ring = [torch.empty((2, local_batch), dtype=torch.int32).pin_memory() for _ in range(4)]
        self.ring_ev = [None] * len(self.ring)

    def next(self):
        from .strata import derive_seed

        ids = self.nd.draw(self.counts, derive_seed(self.seed, self.rank, self.step_i))
        slot = self.step_i % len(self.ring)
        self.step_i += 1
        if self.ring_ev[slot] is not None:
            self.ring_ev[slot].synchronize()
        h = self.ring[slot].numpy()
        h[0] = ids
        h[1] = self.lengths[ids]
        d = self.ring[slot].to("cuda", non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.ring_ev[slot] = ev
        mine, tokens = self.lp.step(d[0], d[1])
        lens = self.d_lengths[mine.long()].clamp(max=self.seq)
        return (self.pos[None, :] < lens[:, None]).long(), tokens


def bert_large_step_bench(mode: str = "bucketwise", steps: int = 5, warmup: int = 2, batch: int = 48,
                          seq: int = 512, clip: float = 1.0, bucket_cap_mb: int = 25, lengths=None,
                          model_config: dict | None = None) -> dict:
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
    cfg = BertConfig(**(model_config or BERT_LARGE))
    cfg._attn_implementation = "sdpa"
    model = BertForPreTraining(cfg).to(dev)
    state = reducer = loader = None
    predicted = None
    if mode in ("stock", "after", "bucketwise"):
        ddp = DDP(model, device_ids=[dev.index], bucket_cap_mb=bucket_cap_mb, gradient_as_bucket_view=True)
        if mode == "bucketwise":
            params = [p for p in model.parameters() if p.requires_grad]
            predicted = ddp_bucket_counts(ddp)  # iteration 0's B, before it runs
            state = make_hook_state(ClipConfig(clip, "bucket_wise"), predicted)
            ddp.register_comm_hook(state, bucketwise_clip_hook)
            ready: list = []  # gradient-ready order of iteration 0 = DDP's rebuilt bucket order
            recorders = [p.register_post_accumulate_grad_hook(lambda q: ready.append(q)) for p in params]
    elif mode in ("reducer", "presort"):
        ddp = model
        reducer = BucketwiseReducer(model.parameters(), ClipConfig(clip, "bucket_wise"), bucket_cap_mb=bucket_cap_mb)
        if mode == "presort":
            if lengths is None:
                from .seqdata import LengthDistribution, generate_lengths

                lengths = generate_lengths(LengthDistribution(), 10_000_000, 2402)
            loader = PresortBatches(lengths, batch, seq)
    else:
        raise ValueError(f"unknown mode {mode!r}")
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + dist.get_rank())
    data = _batch(batch, seq, dev, gen, cfg.vocab_size)

    def step():
        if loader is not None:  # this step's presorted local batch: its lengths mask the tokens
            mask, _tok = loader.next()
            data["attention_mask"] = mask
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = ddp(**data).loss
        loss.backward()
        if reducer is not None:
            reducer.finish(check_finite=False)  # flags checked once after the timed loop
        if mode == "after":
            torch.nn.utils.clip_grad_norm_(model.parameters(), clip)
        opt.step()
        if reducer is not None:
            reducer.zero_grad()
        else:
            opt.zero_grad(set_to_none=False)
        return loss

    actual = actual0 = rebuilt = None
    for i in range(warmup):
        step()
        if state is not None and i == 0:
            # DDP rebuilds its buckets before iteration 1: set B for the rebuilt layout now
            actual0 = max(state.norms) + 1 if state.norms else 1
            for h in recorders:
                h.remove()
            rebuilt = ddp_bucket_counts(ddp, ready)
            state.set_num_buckets(rebuilt)
            state.norms.clear()
    if state is not None:
        actual = max(state.norms) + 1 if state.norms else 1
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
           "batch_per_gpu": batch, "seq": seq, "loss": float(loss.detach()), "params": sum(p.numel() for p in model.parameters())}
    if state is not None:
        out["buckets"] = state.num_buckets
        out["buckets_iter0"] = {"predicted": predicted, "ddp": actual0}
        out["buckets_after_rebuild"] = {"predicted": rebuilt, "ddp": actual}
    if reducer is not None:
        if bool(reducer.nonfinite.any()):
            raise ValueError("gradient has non-finite components")
        out["buckets"] = len(reducer.layout)
        out["comm_dtype"] = str(reducer.comm.dtype).replace("torch.", "")
        reducer.remove()
    if loader is not None:
        # the batch former alone (host draws + H2D + all-gather + K3 + mask), per step
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            loader.next()
        torch.cuda.synchronize()
        out["batch_former_ms_per_step"] = (time.perf_counter() - t0) / 20 * 1e3
        # the same step with this step's padding mask held fixed (no batch former): the mask, not
        # the former, is what changes the attention kernels' cost
        fixed = data["attention_mask"].clone()
        loader_saved, loader = loader, None
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        a.record()
        for _ in range(steps):
            step()
        b.record()
        torch.cuda.synchronize()
        out["same_mask_without_former_ms_per_step"] = a.elapsed_time(b) / steps
        loader = loader_saved
        del fixed
        loader.lp.check()
        out["batch_former"] = "K2 strata + NativeDraws + LocalPresort (all-gather + K3) every step"
    del ddp, model, opt, reducer, loader
    torch.cuda.empty_cache()
    return out
