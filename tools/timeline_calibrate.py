"""Timeline calibration on B200.

    torchrun --nproc-per-node N tools/timeline_calibrate.py [--out profiles/r01_timeline]

Measures, on BERT-large (``train_step`` shape: seq 512, batch 48/GPU, bf16
autocast, DDP 25 MiB buckets), the per-bucket durations the reference's
two-stream pipeline model takes (``TimelinePlan``, timeline.py:28-73):

* ``t_comp[b]``  backward compute that produces bucket b: CUDA events in a
                 timing comm hook (the hook fires, in stream order, once the
                 bucket's gradients are complete);
* ``t_clip[b]``  the K1 clip of bucket b (events around it in the hook);
* ``t_comm[b]``  the NCCL allreduce of bucket b, timed standalone at N ranks;
* ``t_gclip``    the global clip of ``clip_grad_norm_`` (after_allreduce);
* ``t_nred``     a one-scalar allreduce (the global-norm reduce).

It writes ``<out>.toml`` in the reference's plan format (``load_plan``,
timeline.py:228-248; ``ddpsim timeline --plan <out>.toml`` reads it), then
compares the model's per-mode prediction (``schedule``, timeline.py:97-152,
restated below) with the MEASURED backward + synchronisation time of the same
step under each mode (``<out>.json``).  Times are in milliseconds.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


# ----------------------------------------------------------------- model (timeline.py:97-161)
def schedule_total(t_comp, t_comm, t_clip, t_gclip, t_nred, mode: str) -> float:
    B = len(t_comp)
    order = range(B - 1, -1, -1)  # bucket B first
    ready = [0.0] * B
    t = 0.0
    # same float operation order as the reference (bits match its totals)
    if mode == "bucket_wise":
        for b in order:
            t = t + t_comp[b]
            t = t + t_clip[b]
            ready[b] = t
    elif mode == "after_allreduce":
        for b in order:
            t = t + t_comp[b]
            ready[b] = t
    else:  # before_allreduce
        for b in order:
            t = t + t_comp[b]
        t = t + t_nred
        t = t + t_gclip
        ready = [t] * B
    end = 0.0
    first_end = None
    for b in order:
        end = max(ready[b], end) + t_comm[b]
        if b == 0:
            first_end = end
    total = first_end  # bucket 1 is communicated last
    if mode == "after_allreduce":
        total += t_gclip
    return total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01_timeline")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    if "LOCAL_RANK" not in os.environ:
        os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29871")
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)

    from torch.nn.parallel import DistributedDataParallel as DDP
    from transformers import BertConfig, BertForPreTraining

    from paper_2402_02447_b200.ddp import bucketwise_clip_hook, make_hook_state
    from paper_2402_02447_b200.gradsync import ClipConfig
    from paper_2402_02447_b200.train_step import BERT_LARGE, _batch

    torch.manual_seed(1234)
    cfg = BertConfig(**BERT_LARGE)
    cfg._attn_implementation = "sdpa"
    model = BertForPreTraining(cfg).to(dev)
    ddp = DDP(model, device_ids=[local], bucket_cap_mb=25, gradient_as_bucket_view=True)
    state = make_hook_state(ClipConfig(1.0, "bucket_wise"), 37)
    rec = {"on": False, "events": [], "mode": "bucket_wise"}

    def timing_hook(st, bucket):
        if rec["mode"] == "after_allreduce":  # stock DDP comm: plain average, no per-bucket clip
            buf = bucket.buffer()
            return dist.all_reduce(buf, op=dist.ReduceOp.AVG, async_op=True).get_future().then(
                lambda f: f.value()[0])
        if rec["on"]:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        fut = bucketwise_clip_hook(st, bucket)
        if rec["on"]:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()  # after K1, on the compute stream (the allreduce runs on NCCL's)
            rec["events"].append((bucket.index(), bucket.buffer().numel(), e0, e1))
        return fut

    ddp.register_comm_hook(state, timing_hook)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + rank)
    data = _batch(48, 512, dev, gen)

    def step(mode, timed=False):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = ddp(**data).loss
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        loss.backward()
        if mode == "after_allreduce":
            torch.nn.utils.clip_grad_norm_(model.parameters(), 1.0)
        ev[1].record()
        model.zero_grad(set_to_none=False)
        return ev

    for _ in range(3):  # DDP rebuilds its buckets after iteration 1
        step("bucket_wise")
    state.set_num_buckets(max(state.norms) + 1)
    B = state.num_buckets

    # --- per-bucket compute / clip from the hook (bucket_wise mode)
    t_comp = [0.0] * B
    t_clip = [0.0] * B
    sizes = [0] * B
    n = args.steps
    for _ in range(n):
        rec["on"], rec["events"] = True, []
        ev = step("bucket_wise")
        rec["on"] = False
        torch.cuda.synchronize()
        prev = ev[0]
        # DDP bucket index 0 is ready first (the last layers); timeline bucket
        # b = B - 1 - index (bucket B is produced first, timeline.py:103-104)
        for idx, numel, e0, e1 in sorted(rec["events"], key=lambda x: x[0]):
            b = B - 1 - idx
            t_comp[b] += prev.elapsed_time(e0) / n
            t_clip[b] += e0.elapsed_time(e1) / n
            sizes[b] = numel
            prev = e1
    # --- per-bucket allreduce, standalone at this world size (fp32 in place, avg)
    op = dist.ReduceOp.AVG
    t_comm = []
    for b in range(B):
        x = torch.randn(sizes[b], device=dev)
        for _ in range(3):
            dist.all_reduce(x, op=op)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(10):
            dist.all_reduce(x, op=op)
        e[1].record()
        torch.cuda.synchronize()
        t_comm.append(e[0].elapsed_time(e[1]) / 10)
    # --- global clip and the norm reduce
    for _ in range(2):
        step("bucket_wise")
    torch.cuda.synchronize()
    # clip_grad_norm_ issues ~400 small launches: timed eagerly it measures the
    # CPU, not the GPU (in the real step those launches hide behind the
    # backward queue), so its GPU time is taken from a CUDA-graph replay
    params = [p for p in model.parameters() if p.grad is not None]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        torch.nn.utils.clip_grad_norm_(params, 1.0)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        torch.nn.utils.clip_grad_norm_(params, 1.0)
    graph.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(10):
        graph.replay()
    e[1].record()
    torch.cuda.synchronize()
    t_gclip = e[0].elapsed_time(e[1]) / 10
    del graph
    s = torch.ones(1, device=dev)
    e[0].record()
    for _ in range(20):
        dist.all_reduce(s)
    e[1].record()
    torch.cuda.synchronize()
    t_nred = e[0].elapsed_time(e[1]) / 20

    # --- measured backward + sync per mode (event pair around backward [+ clip])
    measured = {}
    for mode in ("bucket_wise", "after_allreduce"):
        rec["mode"] = mode
        step(mode)
        tot = 0.0
        for _ in range(n):
            ev = step(mode)
            torch.cuda.synchronize()
            tot += ev[0].elapsed_time(ev[1]) / n
        measured[mode] = tot
    t = torch.tensor([measured["bucket_wise"], measured["after_allreduce"]], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    measured = {"bucket_wise": float(t[0]), "after_allreduce": float(t[1])}

    if rank == 0:
        plan = {"t_comp": t_comp, "t_comm": t_comm, "t_clip": t_clip, "t_gclip": t_gclip, "t_nred": t_nred}
        out = Path(args.out)
        out.parent.mkdir(parents=True, exist_ok=True)
        with open(out.with_suffix(".toml"), "w") as f:
            f.write(f"# BERT-large on {world} x B200, measured (ms); ddpsim timeline --plan reads this\n")
            for k, v in plan.items():
                if isinstance(v, list):
                    f.write(f"{k} = [{', '.join(f'{x:.6f}' for x in v)}]\n")
                else:
                    f.write(f"{k} = {v:.6f}\n")
        pred = {m: schedule_total(t_comp, t_comm, t_clip, t_gclip, t_nred, m)
                for m in ("bucket_wise", "after_allreduce", "before_allreduce")}
        res = {"world": world, "buckets": B, "units": "ms",
               "sum_t_comp": sum(t_comp), "sum_t_clip": sum(t_clip), "sum_t_comm": sum(t_comm),
               "t_gclip": t_gclip, "t_nred": t_nred,
               "predicted": pred, "measured": measured,
               "rel_err": {m: (pred[m] - measured[m]) / measured[m] for m in measured},
               "note": "measured = backward (+ clip_grad_norm_ for after_allreduce) including DDP's wait "
                       "for the last allreduce, CUDA events on the compute stream, max over ranks; bucket_wise "
                       "runs the K1 clip hook, after_allreduce a plain average hook; predicted = "
                       "timeline.schedule (timeline.py:97-152) on the measured plan"}
        out.with_suffix(".json").write_text(json.dumps(res, indent=1))
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
