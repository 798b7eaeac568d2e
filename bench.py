"""Benchmark: clip+allreduce GB/s (H1, BERT-large synthetic gradients) + presort keys/s (H2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by the driver under torchrun (one rank per GPU, NCCL).  Rank 0
prints ONE JSON line.  Headline (`value`): whole-job fp32 gradient GB/s
through the bucket-wise clip — at N=1 one fused K1 launch over the 52
buckets (nothing to reduce), at N>1 one K1 launch per 25 MiB bucket in
backward order + an NCCL average of that bf16 bucket on a side stream —
inputs resident in HBM (1.34 GB per rank > 126 MB L2, so no flush is
needed).  `e2e`: the same metric through the public API
(`GradientState`+`sync_bucketwise`, or `BucketwiseSync` at N>1) from pinned
host gradients to a host result.  `presort`: stratified local presort of 10M
Wikipedia-like lengths over 8 rank shards (K2 partition of every shard + K3
sort/deal of a whole epoch of Topology(1,8) node-step pools), rank 0.
`--impl reference` times the oracle port of the reference CPU path
(oracle/ddp_oracle.py; /root/reference is not on the GPU box) on the host.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BOUNDS = (128, 256, 384, 512)
CORPUS_N, CORPUS_SEED, SHARDS, GPN = 10_000_000, 2402, 8, 8


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- dist
def dist_init(n_gpus: int):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# --------------------------------------------------------------------- H1 (ours)
def ncu_traffic(kernel_key: str):
    """dram read+write bytes per launch of `kernel_key` from the committed ncu summary, if any."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text()).get(kernel_key)
    return None if d is None else d.get("dram_bytes_per_launch")


def bench_clip(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200 import synthetic
    from paper_2402_02447_b200.ddp import BucketwiseSync

    dim = synthetic.BERT_LARGE_DIM
    g, layout, scales = synthetic.bert_grads(dim, rank=rank)
    nb = len(layout)
    cfg = B.ClipConfig(1.0, "bucket_wise")
    limit = 1.0 / math.sqrt(nb)  # c / sqrt(B), gradsync.py:155
    comm = torch.empty(dim, dtype=torch.bfloat16, device="cuda")
    compute = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(nb)]
    order = list(reversed(range(nb)))  # backward order, gradsync.py:157
    segs = [(layout[b][0], layout[b][0], layout[b][1] - layout[b][0]) for b in order]
    clip = B.BucketClipper()

    if world == 1:
        # all buckets resident: one fused launch over the 52 buckets (sync_bucketwise path)
        launch_all = clip.prepare(g, comm, segs, limit)

        def step():
            launch_all()
        mode = "one fused K1 launch over all 52 buckets (no allreduce at N=1)"
        launches_per_step = 1
    else:
        from paper_2402_02447_b200.ddp import FusedBucketSync

        def capture(fn):
            """Capture fn(stream) once into a CUDA graph; return (replay, note)."""
            try:
                cap = torch.cuda.Stream()
                cap.wait_stream(compute)
                with torch.cuda.stream(cap):
                    fn(cap)
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=cap):
                    fn(cap)
                torch.cuda.synchronize()
                return graph.replay, "CUDA graph"
            except Exception as e:  # capture unsupported: stay eager, say so
                torch.cuda.synchronize()
                return (lambda: fn(compute)), f"eager (graph capture failed: {str(e)[:100]})"

        # (a) NCCL path: per bucket K1 on the compute stream + ncclAllReduce(avg, bf16) on a side stream
        bsync = BucketwiseSync(layout, cfg, comm_dtype=torch.bfloat16)

        def nccl_step(s_):
            bsync.sync_native(g, stream=s_)
            s_.wait_stream(bsync.side)

        nccl_replay, nccl_note = capture(nccl_step)
        # (b) fused path: one kernel per rank clips and reduces every bucket over NVLink peer memory
        fused_replay, fused_note = None, "unavailable"
        if args.comm == "fused":
            try:
                fsync = FusedBucketSync(layout, cfg)
                fused_replay, fused_note = capture(lambda s_: fsync.sync(g, stream=s_))
            except Exception as e:
                fused_note = f"unavailable: {str(e)[:120]}"
        if fused_replay is not None:
            step = fused_replay
            mode = (f"fused K1 + allreduce per bucket over NVLink ({fsync.transport}: "
                    f"{'NVSwitch multimem reduce' if fsync.transport == 'nvls' else 'two-shot peer memory'}), "
                    f"one kernel per rank ({fused_note})")
            launches_per_step = 1
        else:
            step = nccl_replay
            mode = f"per-bucket K1 + ncclAllReduce(avg, bf16) on a side stream ({nccl_note}); fused: {fused_note}"
            launches_per_step = nb
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU loaded ~0.6 s so the sampler sees clocks under load, then time
        tl = time.perf_counter()
        while time.perf_counter() - tl < 0.6:
            step()
            torch.cuda.synchronize()
        barrier(world)
        t0.record(compute)
        for _ in range(args.steps):
            step()
        t1.record(compute)
        torch.cuda.synchronize()
        barrier(world)
        sustained_copy = None
        if world == 1:
            # the copy peak in the same (power-capped) state: MEASURED_PEAKS' method (copy_ of
            # 1 Gi bf16 elements, read + write bytes), right after the timed steps
            src = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
            dst = torch.empty_like(src)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = None
            for _ in range(5):
                c0.record(compute)
                dst.copy_(src)
                c1.record(compute)
                torch.cuda.synchronize()
                best = min(best or 1e9, c0.elapsed_time(c1))
            sustained_copy = 2 * src.numel() * 2 / (best * 1e-3) / 1e9
            del src, dst
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)

    # dominant kernel alone: the fused launch over all buckets, CUDA events on its stream
    launch_all = clip.prepare(g, comm, segs, limit)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        launch_all()
    torch.cuda.synchronize()
    k0.record(compute)
    for _ in range(args.steps):
        launch_all()
    k1.record(compute)
    torch.cuda.synchronize()
    kb_ms = k0.elapsed_time(k1) / args.steps
    # per-bucket launches (DDP-hook shape), captured once in a CUDA graph
    pb = {}
    try:
        gside = torch.cuda.Stream()
        gside.wait_stream(compute)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gside):
            gclip = B.BucketClipper(stream=gside)
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=gside):
                for s_ in segs:
                    gclip.prepare(g, comm, [s_], limit)()
        torch.cuda.synchronize()
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        k0.record(compute)
        for _ in range(args.steps):
            graph.replay()
        k1.record(compute)
        torch.cuda.synchronize()
        pb_ms = k0.elapsed_time(k1) / args.steps
        pb = {"us_per_step": pb_ms * 1e3, "us_per_launch": pb_ms * 1e3 / nb,
              "achieved_gbs": dim * 6 / (pb_ms * 1e-3) / 1e9, "launches": nb, "cuda_graph": True}
    except Exception as e:  # graph capture unavailable: report, do not fail the bench
        pb = {"error": str(e)[:200]}

    pk = peaks()
    alg_bytes = dim * (4 + 2)  # fp32 read + bf16 write per element
    kb_gbs = alg_bytes / (kb_ms * 1e-3) / 1e9
    traffic = ncu_traffic("k_bucket_clip_ws<float,bf16>/bert_large_52")
    # at N=1 the timed step IS one K1 launch: the roofline comes from the same timed loop
    # (sustained: after 0.6 s of load the board sits at its power cap); the kernel timed
    # alone right after (burst) is reported beside it
    step_us = ms * 1e3 if world == 1 else kb_ms * 1e3
    step_gbs = alg_bytes / (step_us * 1e-6) / 1e9
    res = {
        "ms_per_step": ms,
        "value": world * dim * 4 / (ms * 1e-3) / 1e9,
        "mode": mode,
        "roofline": {
            "bound": "hbm", "kernel": "k_bucket_clip_ws<f32,bf16>: one launch, 52 x 25 MiB buckets",
            "achieved": step_gbs, "peak": pk["hbm_gbs"], "peak_src": pk["src"], "unit": "GB/s",
            "frac": step_gbs / pk["hbm_gbs"], "traffic": traffic, "bytes_per_launch": alg_bytes,
            "launch_us": step_us,
            "timing": ("CUDA events over the timed step loop (the step is this launch)" if world == 1 else
                       "CUDA events over K launches of K1 alone (the step is K4)"),
            "burst": {"launch_us": kb_ms * 1e3, "achieved": kb_gbs, "frac": kb_gbs / pk["hbm_gbs"],
                      "note": "the same launch timed alone right after the step loop"},
            "copy_peak_same_state_gbs": sustained_copy,
            "frac_vs_copy_same_state": (step_gbs / sustained_copy) if sustained_copy else None,
            "per_bucket_launches": pb,
        },
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk.summary(),
    }
    if world > 1:
        algbw = dim * 2 / (ms * 1e-3) / 1e9
        # NCCL alone on the same 52 bf16 buckets (no clip) = the comm floor of the step
        for _ in range(3):
            for b in order:
                bsync.nccl.all_reduce_avg(bsync.comm[layout[b][0]:layout[b][1]], compute)
        torch.cuda.synchronize()
        barrier(world)
        k0.record(compute)
        for _ in range(args.steps):
            for b in order:
                bsync.nccl.all_reduce_avg(bsync.comm[layout[b][0]:layout[b][1]], compute)
        k1.record(compute)
        torch.cuda.synchronize()
        nccl_ms = max_over_ranks(k0.elapsed_time(k1) / args.steps, world)
        nccl_algbw = dim * 2 / (nccl_ms * 1e-3) / 1e9
        for _ in range(3):
            nccl_replay()
        torch.cuda.synchronize()
        barrier(world)
        k0.record(compute)
        for _ in range(args.steps):
            nccl_replay()
        k1.record(compute)
        torch.cuda.synchronize()
        nccl_step_ms = max_over_ranks(k0.elapsed_time(k1) / args.steps, world)
        # parity mode: K4 with an fp32 stage (the 1e-5 contract across ranks), same workload
        f32_ms = None
        if launches_per_step == 1:
            try:
                f32sync = FusedBucketSync(layout, cfg, transport="p2p", comm_dtype=torch.float32)
                f32_replay, _ = capture(lambda s_: f32sync.sync(g, stream=s_))
                for _ in range(3):
                    f32_replay()
                torch.cuda.synchronize()
                barrier(world)
                k0.record(compute)
                for _ in range(args.steps):
                    f32_replay()
                k1.record(compute)
                torch.cuda.synchronize()
                f32_ms = max_over_ranks(k0.elapsed_time(k1) / args.steps, world)
                f32sync.close()
            except Exception as e:  # report, do not fail the bench
                f32_ms = f"unavailable: {str(e)[:100]}"
        bus = lambda a: a * 2 * (world - 1) / world
        res["nvlink"] = {"algbw_gbs": algbw, "busbw_gbs": bus(algbw), "peak_gbs": 900.0,
                         "busbw_frac": bus(algbw) / 900.0, "peak_measured_gbs": 770.0,
                         "nccl_only_ms": nccl_ms, "nccl_only_busbw_gbs": bus(nccl_algbw),
                         "nccl_step_ms": nccl_step_ms, "speedup_vs_nccl_step": nccl_step_ms / ms,
                         "comm_dtype": "bf16",
                         "fp32_parity_mode_ms": f32_ms,
                         "collective": (f"fused in K4 ({fsync.transport})" if launches_per_step == 1
                                        else "ncclAllReduce avg per 25 MiB bucket, side stream")}
        # roofline of the fused step (B200_PROFILING.md): bytes that must cross NVLink per
        # direction per GPU / the measured 770 GB/s peer copy; two-shot P2P moves 2(N-1)/N of
        # the bf16 gradient each way, NVLS one full copy
        per_dir = dim * 2 * (2 * (world - 1) / world if getattr(fsync, "mc", 0) == 0 else 1.0) \
            if launches_per_step == 1 else dim * 2 * 2 * (world - 1) / world
        res["nvlink"]["roofline"] = {
            "bound": "nvlink", "bytes_per_dir_per_gpu": per_dir, "achieved": per_dir / (ms * 1e-3) / 1e9,
            "peak": 770.0, "peak_src": "measured peer copy per direction (B200_PROFILING.md)", "unit": "GB/s",
            "frac": per_dir / (ms * 1e-3) / 1e9 / 770.0, "floor_ms": per_dir / 770e9 * 1e3}

    # e2e: pinned host fp32 gradients -> device -> sync -> host result, through the public API
    host = torch.empty((1, dim), dtype=torch.float32, pin_memory=True)
    host.copy_(g.view(1, -1).cpu())
    e2e_steps = max(2, min(args.steps, 5))
    if world == 1:
        out_bf16 = torch.empty(dim, dtype=torch.bfloat16, pin_memory=True)
        out_f32 = torch.empty(dim, dtype=torch.float32, pin_memory=True)

        def e2e_step():  # the host-resident form of GradientState + sync_bucketwise, streamed per bucket
            return B.sync_bucketwise_host(host, layout, cfg, out=out_bf16)
        d2h = dim * 2
        api = ("sync_bucketwise_host (= GradientState + sync_bucketwise; pinned host fp32 in, host bf16 out — "
               "the step's comm dtype, as at N>1; H2D / K1 / D2H streamed per bucket)")
    else:
        out_host = torch.empty(dim, dtype=torch.bfloat16, pin_memory=True)
        if launches_per_step == 1:
            def e2e_step():
                return fsync.sync_host(host.view(-1), out=out_host)
            api = ("FusedBucketSync.sync_host (pinned host fp32 in, host bf16 out; H2D / K4 / D2H "
                   "streamed per 4-bucket chunk)")
        else:
            def e2e_step():
                dg = host.view(-1).to("cuda", non_blocking=True)
                bsync.sync(dg)
                out_host.copy_(bsync.wait(), non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return out_host
            api = "BucketwiseSync.sync (pinned host fp32 in, host bf16 out)"
        d2h = dim * 2
    e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    ts = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - ts, world) / e2e_steps
    res["e2e"] = {"value": world * dim * 4 / e2e_s / 1e9, "unit": "GB/s", "ms_per_step": e2e_s * 1e3,
                  "h2d_bytes_per_step": dim * 4, "d2h_bytes_per_step": d2h, "steps": e2e_steps, "api": api}
    if world == 1:  # the same call returning the fp32 result (2 x 1.34 GB over PCIe)
        B.sync_bucketwise_host(host, layout, cfg, out=out_f32)
        ts = time.perf_counter()
        for _ in range(e2e_steps):
            B.sync_bucketwise_host(host, layout, cfg, out=out_f32)
        t32 = (time.perf_counter() - ts) / e2e_steps
        res["e2e"]["f32_out"] = {"value": dim * 4 / t32 / 1e9, "ms_per_step": t32 * 1e3, "d2h_bytes_per_step": dim * 4}
    del host
    if world == 1:
        # the drop-in call exactly as a reference user makes it: a host fp64 (1, D) numpy array
        # through GradientState + sync_bucketwise, host fp64 result (pageable copies both ways)
        w64 = g.double().cpu().numpy()[None, :]
        st_ = B.GradientState(w64, layout)
        B.sync_bucketwise(st_, cfg)
        del st_
        torch.cuda.synchronize()
        times = []
        for _ in range(2):
            t = time.perf_counter()
            out64 = B.sync_bucketwise(B.GradientState(w64, layout), cfg)
            times.append(time.perf_counter() - t)
        dt = min(times)
        res["e2e_drop_in"] = {
            "value": dim * 4 / dt / 1e9, "unit": "GB/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": dim * 8, "d2h_bytes_per_step": dim * 8, "steps": len(times),
            "api": "sync_bucketwise(GradientState(numpy float64 (1, D), layout), ClipConfig(1.0, 'bucket_wise')) "
                   "-> numpy float64: the reference's own call (fp64 H2D from the caller's pageable array, "
                   "fp64 result D2H into pinned memory)",
            "result_type": type(out64).__name__}
        del w64, out64
    return res


# --------------------------------------------------------------------- H2 (ours)
def presort_inputs():
    """10M-sample corpus, 8 rank shards; per rank, an epoch of REAL reference draws.

    Strata per shard come from K2 (stratify_shards); every rank's draws are
    draw_batch with seed derive_seed(2402, rank, step) (seeding.py:18-21),
    produced by the bit-exact native port (NativeDraws) on host threads.
    Returns (lengths, {lb: (pool_ids, pool_lens, steps)}, draw_stats).
    """
    from concurrent.futures import ThreadPoolExecutor

    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths

    lens = generate_lengths(LengthDistribution(), CORPUS_N, CORPUS_SEED)
    shard = CORPUS_N // SHARDS
    strata = B.stratify_shards(lens, [r * shard for r in range(SHARDS + 1)], BOUNDS)
    shard_pools = []
    for r, ds in enumerate(strata):
        ids = ds.ids.cpu().numpy().astype(np.int64) + r * shard
        o = np.concatenate([[0], np.cumsum(ds.counts)])
        shard_pools.append(([ids[o[k]:o[k + 1]] for k in range(len(BOUNDS))], ds.probs))
    out, stats = {}, {}
    for lb in (16, 48):
        def rank_epoch(r):
            pools, probs = shard_pools[r]
            counts = B.allocate_counts(probs, lb).counts
            nd = B.NativeDraws(pools, BOUNDS)
            ids, done = nd.epoch(counts, CORPUS_SEED, key=(r,), nsteps=shard // lb + 1)
            nd.close()
            return ids.astype(np.int32), done

        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=SHARDS) as ex:
            res = list(ex.map(rank_epoch, range(SHARDS)))
        dt = time.perf_counter() - t0
        steps = min(d for _, d in res)
        ids = np.stack([x[:steps] for x, _ in res], axis=1).reshape(-1)  # pool of step t: GPU 0..7 draws
        out[lb] = (ids, lens[ids].astype(np.int32), steps)
        stats[lb] = {"keys": int(sum(d for _, d in res) * lb), "seconds": dt,
                     "keys_per_s": sum(d for _, d in res) * lb / dt, "threads": SHARDS,
                     "impl": "NativeDraws (bit-exact numpy PCG64 draw_batch port, host C++)"}
    return lens, out, stats


def reference_presort_inputs():
    """Reference arm (CPU only): same corpus, pools of the first 20k node-steps from oracle draws."""
    from oracle import ddp_oracle as O

    lens = O.generate_lengths(CORPUS_N, CORPUS_SEED)
    shard = CORPUS_N // SHARDS
    out = {}
    for lb in (48,):
        ids_r = []
        for r in range(SHARDS):
            part = lens[r * shard:(r + 1) * shard]
            pools, probs = O.stratify(part)
            pl = [(p + r * shard).tolist() for p in pools]
            counts = O.allocate_counts(probs, lb)
            steps = 200  # bounded sample: the oracle's Python draw loop is slow
            ids_r.append(np.array([O.draw_batch(pl, BOUNDS, counts, O_derive(r, t)) for t in range(steps)]))
        ids = np.stack(ids_r, axis=1).reshape(-1).astype(np.int32)
        out[lb] = (ids, lens[ids].astype(np.int32), 200)
    return lens, out


def O_derive(r, t):
    s = np.random.SeedSequence(entropy=CORPUS_SEED, spawn_key=(r, t))
    return int(s.generate_state(1, np.uint64)[0])


def bench_presort(args):
    import torch

    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200 import _lib

    lens, pools, draw_stats = presort_inputs()
    lib = _lib.load()
    shard = CORPUS_N // SHARDS
    d_lens = torch.from_numpy(lens).cuda()
    ws_bytes = lib.b2_strata_workspace_bytes(CORPUS_N)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    ids_out = torch.empty(CORPUS_N, dtype=torch.int32, device="cuda")
    counts = torch.empty((SHARDS, 4), dtype=torch.int64, device="cuda")
    bad = torch.empty(SHARDS, dtype=torch.int64, device="cuda")
    bnds = _lib.i32_array(BOUNDS)
    offs = _lib.i64_array(r * shard for r in range(SHARDS + 1))
    sp = _lib.stream_ptr()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def k2():  # every rank shard stratified in one pass (2 launches)
        _lib.check(lib.b2_strata_partition_shards(
            d_lens.data_ptr(), None, offs, SHARDS, bnds, 4, ids_out.data_ptr(), counts.data_ptr(),
            bad.data_ptr(), ws.data_ptr(), ws_bytes, sp))

    res = {"draws": {f"lb{k}": v for k, v in draw_stats.items()}}
    for lb in (16, 48):
        ids, ln, steps = pools[lb]
        d_ids, d_ln = torch.from_numpy(ids).cuda(), torch.from_numpy(ln).cuda()
        seg = GPN * lb
        out = torch.empty(ids.size, dtype=torch.int32, device="cuda")
        tok = torch.empty((steps, GPN), dtype=torch.int64, device="cuda")
        pbad = torch.empty(1, dtype=torch.int64, device="cuda")

        def k3():
            _lib.check(lib.b2_presort_deal(d_ids.data_ptr(), d_ln.data_ptr(), steps, seg, GPN, 1, 512,
                                           CORPUS_N - 1, out.data_ptr(), None, tok.data_ptr(),
                                           pbad.data_ptr(), sp))

        for _ in range(args.warmup):
            k2(); k3()
        t2 = t3 = 0.0
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (inputs are 40-120 MB)
            torch.cuda.synchronize()
            ev[0].record(); k2(); ev[1].record(); k3(); ev[2].record()
            torch.cuda.synchronize()
            t2 += ev[0].elapsed_time(ev[1])
            t3 += ev[1].elapsed_time(ev[2])
        t2 /= args.steps
        t3 /= args.steps
        keys = ids.size
        hbm = peaks()["hbm_gbs"]
        k2_gbs = CORPUS_N * 8 / (t2 * 1e-3) / 1e9
        k3_gbs = keys * 12 / (t3 * 1e-3) / 1e9
        res[f"lb{lb}"] = {
            "keys_per_s": keys / ((t2 + t3) * 1e-3), "ms_per_step": t2 + t3, "node_steps": steps,
            "keys_presorted": keys, "keys_partitioned": CORPUS_N,
            "k2_partition": {"ms": t2, "achieved_gbs": k2_gbs, "frac": k2_gbs / hbm, "bytes_per_key": 8,
                             "launches": 2, "shards": SHARDS},
            "k3_presort_deal": {"ms": t3, "achieved_gbs": k3_gbs, "frac": k3_gbs / hbm, "bytes_per_key": 12,
                                "launches": 1},
        }
    # a 10x batched run (100 M keys) shows the asymptote once
    # launch latency no longer matters: the corpus tiled 10x through K2 (8
    # shards of 12.5 M) and the lb-16 epoch's pools tiled 10x through K3
    reps = 10
    big_lens = d_lens.repeat(reps)
    nbig = big_lens.numel()
    ws_big = lib.b2_strata_workspace_bytes(nbig)
    wsb = torch.empty(ws_big, dtype=torch.uint8, device="cuda")
    ids_big = torch.empty(nbig, dtype=torch.int32, device="cuda")
    offs_big = _lib.i64_array(r * (nbig // SHARDS) for r in range(SHARDS + 1))
    ids16, ln16, steps16 = pools[16]
    b_ids = torch.from_numpy(ids16).cuda().repeat(reps)
    b_ln = torch.from_numpy(ln16).cuda().repeat(reps)
    b_out = torch.empty_like(b_ids)
    b_tok = torch.empty((steps16 * reps, GPN), dtype=torch.int64, device="cuda")
    pbad = torch.empty(1, dtype=torch.int64, device="cuda")

    def k2b():
        _lib.check(lib.b2_strata_partition_shards(
            big_lens.data_ptr(), None, offs_big, SHARDS, bnds, 4, ids_big.data_ptr(), counts.data_ptr(),
            bad.data_ptr(), wsb.data_ptr(), ws_big, sp))

    def k3b():
        _lib.check(lib.b2_presort_deal(b_ids.data_ptr(), b_ln.data_ptr(), steps16 * reps, GPN * 16, GPN, 1, 512,
                                       CORPUS_N - 1, b_out.data_ptr(), None, b_tok.data_ptr(), pbad.data_ptr(), sp))

    for _ in range(2):
        k2b(); k3b()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t2 = t3 = 0.0
    nrep = max(3, min(args.steps, 10))
    for _ in range(nrep):
        torch.cuda.synchronize()
        ev[0].record(); k2b(); ev[1].record(); k3b(); ev[2].record()
        torch.cuda.synchronize()
        t2 += ev[0].elapsed_time(ev[1]) / nrep
        t3 += ev[1].elapsed_time(ev[2]) / nrep
    hbm = peaks()["hbm_gbs"]
    res["batched_10x_lb16"] = {
        "keys": int(nbig), "keys_per_s": nbig / ((t2 + t3) * 1e-3), "ms": t2 + t3,
        "k2_partition": {"ms": t2, "achieved_gbs": nbig * 8 / (t2 * 1e-3) / 1e9,
                         "frac": nbig * 8 / (t2 * 1e-3) / 1e9 / hbm},
        "k3_presort_deal": {"ms": t3, "achieved_gbs": b_ids.numel() * 12 / (t3 * 1e-3) / 1e9,
                            "frac": b_ids.numel() * 12 / (t3 * 1e-3) / 1e9 / hbm},
        "note": "corpus and epoch pools tiled 10x (inputs 0.4-1.2 GB >> L2)"}
    del big_lens, wsb, ids_big, b_ids, b_ln, b_out, b_tok
    res["k5_shard_sort"] = bench_k5(args, lens, flush)
    res["e2e"] = bench_presort_e2e(args, lens, pools[48])
    return res


def bench_k5(args, lens, flush):
    """K5 (device-wide stable radix sort + deal): every 1.25M-sample rank shard of the 10M corpus
    sorted by (-length, id) in one call (north_star's per-rank radix sort on length keys),
    (a) ids in shard order (the stratified shard: the id digits are skipped on the device) and
    (b) ids shuffled inside each shard (every digit pass).  12 B/key algorithmic."""
    import torch

    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200.balance import presort_workspace_bytes

    shard = CORPUS_N // SHARDS
    d_len = torch.from_numpy(lens.astype(np.int32)).cuda()
    rng = np.random.default_rng(5)
    cases = {"ids_in_order": np.arange(CORPUS_N, dtype=np.int32),
             "ids_shuffled": np.concatenate([rng.permutation(np.arange(r * shard, (r + 1) * shard, dtype=np.int32))
                                             for r in range(SHARDS)])}
    ws = torch.empty(presort_workspace_bytes(SHARDS, shard, 512, CORPUS_N - 1), dtype=torch.uint8, device="cuda")
    hbm = peaks()["hbm_gbs"]
    out = {}
    for name, ids in cases.items():
        d_ids = torch.from_numpy(ids).cuda()

        def run():
            return B.presort_deal(d_ids, d_len, shard, 1, "raster", max_len=512, max_id=CORPUS_N - 1,
                                  workspace=ws)
        r = run()
        assert int(r[3]) == -1
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            ev[0].record()
            run()
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = statistics.median(ts)
        gbs = CORPUS_N * 12 / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "keys_per_s": CORPUS_N / (ms * 1e-3), "achieved_gbs": gbs, "frac": gbs / hbm,
                     "bytes_per_key": 12}
    out["config"] = "8 rank shards x 1.25M samples, one presort_deal(seg_len=1.25M, lanes=1) call, L2 flushed"
    return out


def bench_presort_e2e(args, lens, pool48):
    """The batch former end to end through the public API with HOST buffers: host lengths and
    host draws (an lb48 epoch of Topology(1,8) node steps) in, host stratum ids, dealt ids and
    token counts out; every H2D / D2H inside the timed region (stratify_shards + presort_deal,
    strata.py:61-83, balance.py:158-184)."""
    import torch

    import paper_2402_02447_b200 as B

    ids, ln, steps = pool48
    shard = CORPUS_N // SHARDS
    offs = [r * shard for r in range(SHARDS + 1)]
    h_lens = torch.from_numpy(lens.astype(np.int32)).pin_memory()
    h_ids = torch.from_numpy(ids).pin_memory()
    h_ln = torch.from_numpy(ln).pin_memory()
    h_strata = torch.empty(CORPUS_N, dtype=torch.int32).pin_memory()
    h_out = torch.empty(ids.size, dtype=torch.int32).pin_memory()
    h_tok = torch.empty((steps, GPN), dtype=torch.int64).pin_memory()

    # the two calls are independent here (the epoch's draws are given), so they run on
    # separate streams: the lengths' H2D first, then the presort as NCH chunks of whole node
    # pools on two alternating streams (each chunk's H2D / K3 / D2H overlaps its
    # neighbours'), then the stratification (whose wrapper reads the shard counts back) on
    # a third; PCIe then carries H2D and D2H at once
    s_pre = [torch.cuda.Stream(), torch.cuda.Stream()]
    s_str = torch.cuda.Stream()
    NCH = 4
    pool = GPN * 48
    bounds = [(steps * k // NCH) * pool for k in range(NCH + 1)]

    def step():
        with torch.cuda.stream(s_str):  # the lengths' H2D goes first, so K2 (and its host read) is early
            d_lens = h_lens.to("cuda", non_blocking=True)
        bads = []
        for k in range(NCH):
            a, b = bounds[k], bounds[k + 1]
            sp = s_pre[k % 2]
            with torch.cuda.stream(sp):
                d_ids = h_ids[a:b].to("cuda", non_blocking=True)
                d_ln = h_ln[a:b].to("cuda", non_blocking=True)
                out, tok, _, bad = B.presort_deal(d_ids, d_ln, pool, GPN, "snake", max_len=512,
                                                  max_id=CORPUS_N - 1, stream=sp)
                h_out[a:b].copy_(out.view(-1), non_blocking=True)
                h_tok[a // pool:b // pool].copy_(tok, non_blocking=True)
                bads.append(bad)
        with torch.cuda.stream(s_str):
            st = B.stratify_shards(d_lens, offs, BOUNDS, stream=s_str)  # K2, shard counts to host
            for r, ds in enumerate(st):
                h_strata[offs[r]:offs[r + 1]].copy_(ds.ids, non_blocking=True)
        torch.cuda.synchronize()
        return max(int(x) for x in bads)

    assert step() == -1
    n = max(3, min(args.steps, 10))
    t = time.perf_counter()
    for _ in range(n):
        step()
    sec = (time.perf_counter() - t) / n
    return {"value": CORPUS_N / sec, "unit": "keys/s", "ms_per_step": sec * 1e3, "steps": n,
            "h2d_bytes_per_step": CORPUS_N * 4 + ids.size * 8, "d2h_bytes_per_step": CORPUS_N * 4 + ids.size * 4
            + steps * GPN * 8,
            "api": "stratify_shards(pinned host lengths) -> host stratum ids; presort_deal(host lb48 draws of a "
                   "whole epoch, 4 chunks of node pools) -> host dealt ids + token counts; the independent calls on "
                   "separate streams",
            "keys": "10M samples stratified + 10M presorted and dealt per step"}




def bench_mcsim(args, lens):
    """the Monte-Carlo balance engine at paper scale
    (Topology(128, 8) = 1,024 GPUs, lb 16, LOCAL_PRESORT + snake, the 10 M corpus).
    Unit: keys = trials x lb x GPUs drawn, dealt and summed."""
    import torch

    from paper_2402_02447_b200 import Topology
    from paper_2402_02447_b200.mcsim import (BalanceExperiment, _prepare, draw_trials, draw_trials_device, run_trials,
                                             trial_token_counts)

    T = args.mc_trials
    exp = BalanceExperiment("local_presort", Topology(128, 8), lens, seed=CORPUS_SEED, local_batch=16, trials=T,
                            scan="snake")
    prep = _prepare(exp)
    keys_per_trial = 16 * 1024
    threads = len(os.sched_getaffinity(0))
    # draws alone (host threads)
    n_d = min(T, 4096)
    t0 = time.perf_counter()
    mat = draw_trials(exp, 0, n_d, prep=prep, threads=threads)
    t_draw = time.perf_counter() - t0
    # device draws alone (one warp per trial, CUDA events)
    pools = prep.pools_dev
    dmat = torch.empty((n_d, keys_per_trial), dtype=torch.int32, device="cuda")
    draw_trials_device(exp, 0, n_d, out=dmat, prep=prep, pools=pools)
    torch.cuda.synchronize()
    evd = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    evd[0].record()
    draw_trials_device(exp, 0, n_d, out=dmat, prep=prep, pools=pools)
    evd[1].record()
    torch.cuda.synchronize()
    t_ddraw = evd[0].elapsed_time(evd[1]) * 1e-3
    same = bool(np.array_equal(dmat.cpu().numpy(), mat))
    # kernel alone (device-resident matrices, CUDA events)
    for _ in range(3):
        trial_token_counts(exp, dmat, prep.max_len)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        trial_token_counts(exp, dmat, prep.max_len)
    ev[1].record()
    torch.cuda.synchronize()
    t_k = ev[0].elapsed_time(ev[1]) / 10 * 1e-3
    # end to end (draws overlapped with H2D + kernel, then the reference's aggregation)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mins, maxs = run_trials(exp, chunk=4096, threads=threads)
    t_e2e = time.perf_counter() - t0
    kbytes = n_d * keys_per_trial * 4  # int32 length read per key
    return {"metric": "mc keys/s", "unit": "keys/s",
            "config": f"BalanceExperiment(LOCAL_PRESORT, snake, Topology(128, 8), lb 16, {T} trials, 10M corpus)",
            "keys": T * keys_per_trial, "keys_per_s": T * keys_per_trial / t_e2e, "seconds": t_e2e,
            "avg_min": float(mins.mean()), "avg_max": float(maxs.mean()),
            "draws": {"keys_per_s": n_d * keys_per_trial / t_draw, "threads": threads,
                      "impl": "b2_mc_draw (bit-exact numpy SeedSequence/PCG64/choice port, host C++)"},
            "draws_device": {"keys_per_s": n_d * keys_per_trial / t_ddraw, "ms_per_4096_trials": t_ddraw * 1e3,
                             "bit_identical_to_host": same,
                             "impl": "b2_mc_draw_device (same port on the GPU, one warp per trial)"},
            "e2e_draws": "device (every stratum in numpy's Floyd branch)",
            "kernel": {"keys_per_s": n_d * keys_per_trial / t_k, "ms_per_4096_trials": t_k * 1e3,
                       "achieved_gbs": kbytes / t_k / 1e9, "frac": kbytes / t_k / 1e9 / peaks()["hbm_gbs"],
                       "bytes_per_key": 4}}


def cpu_mcsim_baseline(lens: np.ndarray, trials: int = 40) -> dict:
    """The reference algorithm on the host (oracle numpy, strata prepared once
    like mcsim._prepare): per-trial draws + local presort + min/max."""
    from oracle import ddp_oracle as O

    pools, probs = O.stratify(lens, BOUNDS, ids=np.arange(lens.size))
    counts = O.allocate_counts(probs, 16)
    pl = [lens[np.asarray(p, dtype=np.int64)] for p in pools]
    G = 1024
    t0 = time.perf_counter()
    for t in range(trials):
        rng = np.random.default_rng(np.random.SeedSequence(entropy=CORPUS_SEED, spawn_key=(t,)))
        blocks = [p[rng.choice(p.size, size=c * G, replace=False)].reshape(c, G) for c, p in zip(counts, pl) if c]
        tok = O.mcsim_local_presort_tokens(np.concatenate(blocks), 128, 8, True)
        tok.min(), tok.max()
    dt = time.perf_counter() - t0
    return {"value": trials * 16 * G / dt, "unit": "keys/s", "cores": 1, "kind": "port",
            "sample": f"{trials} trials of the 1,024-GPU LOCAL_PRESORT experiment (oracle numpy loop, strata prepared once)"}


# --------------------------------------------------------------------- CPU baselines
def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max([int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        return 1


BERT_LARGE_DIM, BUCKET_ELEMS, BUCKET_SCALES = 335_141_888, 25 * 1024 * 1024 // 4, (1e-5, 1e-4, 1e-3)


def host_bert_grads(seed: int = 2402, rank: int = 0):
    """The H1 workload on the host (numpy only): BERT-large D fp32, 52 x 25 MiB buckets,
    per-bucket scales drawn exactly like synthetic.bert_grads (same seed -> same scale per
    bucket, so the same buckets clip); values are numpy normals, not the CUDA generator's."""
    from oracle import ddp_oracle as O

    layout = O.capped_bucket_layout(BERT_LARGE_DIM, BUCKET_ELEMS)
    scales = np.random.default_rng(seed + 7919 * rank).choice(np.asarray(BUCKET_SCALES), size=len(layout))
    rng = np.random.default_rng(seed + rank)
    g = np.empty(BERT_LARGE_DIM, np.float32)
    for (a, b), sc in zip(layout, scales):
        g[a:b] = rng.standard_normal(b - a, dtype=np.float32) * np.float32(sc)
    return g, layout


def reference_clip_step(workers_f32: np.ndarray, layout, threshold: float = 1.0):
    """One reference-path step: GradientState(workers) (fp64 conversion + finiteness check,
    gradsync.py:50,182-191) then sync_bucketwise (gradsync.py:148-162), as oracle restatements."""
    from oracle import ddp_oracle as O

    w = O.as_worker_matrix(workers_f32)
    return O.sync_bucketwise(w, layout, threshold)


def cpu_clip_baseline(reps: int = 2) -> dict:
    """The reference CPU path on this host over the SAME workload as the GPU arm (full config)."""
    g, layout = host_bert_grads()
    reference_clip_step(g[None, :], layout)  # warm (page-in)
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        reference_clip_step(g[None, :], layout)
        times.append(time.perf_counter() - t)
    med = statistics.median(times)
    return {"value": g.size * 4 / med / 1e9, "unit": "GB/s", "cores": blas_threads(), "kind": "port",
            "sample": f"full config: GradientState(fp32 (1, {g.size}) -> fp64) + sync_bucketwise over the 52 x 25 MiB "
                      f"BERT-large buckets (oracle numpy restatement), median of {reps} steps",
            "same_config": True, "seconds_per_step": med,
            "threads_note": "numpy elementwise ops single-threaded; the fp64 norm (BLAS ddot) uses `cores` threads",
            "host_cpus": len(os.sched_getaffinity(0))}


def bench_bert_base(args) -> dict:
    """BASELINE config 0 (the reference's own CPU-runnable case): bucket-wise clip of BERT-base
    synthetic gradients (109.5 M fp32, 17 x 25 MiB buckets), K=1: K1 in one launch (CUDA
    events, inputs 438 MB > L2) next to the reference path on the host (same layout, same
    per-bucket scale draw, GradientState fp64 conversion included)."""
    import torch

    import paper_2402_02447_b200 as B
    from paper_2402_02447_b200 import synthetic
    from oracle import ddp_oracle as O

    dim = synthetic.BERT_BASE_DIM
    g, layout, _ = synthetic.bert_grads(dim)
    comm = torch.empty(dim, dtype=torch.bfloat16, device="cuda")
    out32 = torch.empty(dim, dtype=torch.float32, device="cuda")
    segs = [(a, a, b - a) for a, b in reversed(layout)]
    clip = B.BucketClipper()
    lim = 1.0 / math.sqrt(len(layout))
    res = {"workload": f"BERT-base synthetic gradients (D={dim:,} fp32, {len(layout)} x 25 MiB buckets), K=1"}
    for name, out, bpe in (("bf16_out", comm, 6), ("f32_out", out32, 8)):
        f = clip.prepare(g, out, segs, lim)
        for _ in range(3):
            f()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(args.steps):
            f()
        ev[1].record()
        torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) / args.steps * 1e3
        res[name] = {"us": us, "value_gbs": dim * 4 / (us * 1e-6) / 1e9, "hbm_frac": dim * bpe / (us * 1e-6) / 1e9
                     / peaks()["hbm_gbs"]}
    # the reference path on the host, same workload shape
    scales = np.random.default_rng(2402).choice(np.asarray(BUCKET_SCALES), size=len(layout))
    rng = np.random.default_rng(2402)
    h = np.empty(dim, np.float32)
    for (a, b), sc in zip(layout, scales):
        h[a:b] = rng.standard_normal(b - a, dtype=np.float32) * np.float32(sc)
    t = time.perf_counter()
    reference_clip_step(h[None, :], layout)
    sec = time.perf_counter() - t
    res["cpu_baseline"] = {"value": dim * 4 / sec / 1e9, "unit": "GB/s", "cores": blas_threads(), "kind": "port",
                           "sample": "one full step: GradientState(fp32 -> fp64) + sync_bucketwise (oracle numpy)"}
    return res


def cpu_presort_baseline(lens: np.ndarray, pools: dict) -> dict:
    from oracle import ddp_oracle as O

    shard = CORPUS_N // SHARDS
    t = time.perf_counter()
    for r in range(2):
        O.stratify(lens[r * shard:(r + 1) * shard], BOUNDS)
    t_strat = (time.perf_counter() - t) / (2 * shard)
    ids, ln, steps = pools[48]
    m = 20_000 * GPN * 48 if steps > 20_000 else ids.size
    t = time.perf_counter()
    O.presort_deal_segments(ids[:m], ln[:m], GPN * 48, GPN, True)
    t_sort = (time.perf_counter() - t) / m
    return {"value": 1.0 / (t_strat + t_sort), "unit": "keys/s", "cores": 1, "kind": "port",
            "sample": f"oracle stratify 2 x 1.25M shard + presort_deal of {m} keys (lb48, Topology(1,8))"}


# --------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """Reference arm: the reference CPU path (oracle restatement of gradsync/strata/balance;
    /root/reference is not on the GPU box) on this host.  N=1: the full BERT-large config
    every step.  N>1: K = N simulated workers (the reference's single-process form) over the
    last ceil(52/N) buckets, so a step touches about D elements; declared as a sample."""
    if rank != 0:
        return None
    from oracle import ddp_oracle as O

    g, layout = host_bert_grads()
    nb = len(layout)
    if world == 1:
        w = g[None, :]
        lay, thr, same = layout, 1.0, True
        sample = "full config per step (K=1, 52 x 25 MiB buckets, GradientState fp64 conversion included)"
    else:
        nb_s = -(-nb // world)
        sel = layout[nb - nb_s:]
        a0 = sel[0][0]
        lay = tuple((a - a0, b - a0) for a, b in sel)
        # K workers: rank r's gradients are a rotated copy of the same buckets (distinct per worker)
        w = np.stack([np.roll(g[a0:], 7919 * r) for r in range(world)])
        thr = math.sqrt(nb_s) / math.sqrt(nb)  # the full config's per-bucket limit c/sqrt(52)
        same = False
        sample = (f"K={world} workers x the last {nb_s} of 52 buckets ({w.size} elements per step, "
                  "GradientState fp64 conversion included)")
    for _ in range(min(args.warmup, 1)):
        reference_clip_step(w, lay, thr)
    t = time.perf_counter()
    for _ in range(args.steps):
        reference_clip_step(w, lay, thr)
    sec = (time.perf_counter() - t) / args.steps
    v = w.size * 4 / sec / 1e9
    lens, pools = reference_presort_inputs()
    pre = cpu_presort_baseline(lens, pools)
    return {
        "metric": "clip+allreduce GB/s", "value": v, "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "BERT-large synthetic gradients (D=335,141,888 fp32, 52 x 25 MiB buckets), "
                               "bucket-wise clip c/sqrt(52) + average over workers",
                   "sample": sample, "same_config": same},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": blas_threads(), "kind": "port", "sample": sample,
                         "threads_note": "numpy elementwise single-threaded; BLAS ddot uses `cores` threads"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "presort": {"keys_per_s": pre["value"], "unit": "keys/s", "cpu_baseline": pre},
    }


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-presort", action="store_true")
    ap.add_argument("--no-bert", action="store_true")
    ap.add_argument("--no-mcsim", action="store_true")
    ap.add_argument("--mc-trials", type=int, default=20000)
    ap.add_argument("--comm", choices=("fused", "nccl"), default="fused",
                    help="N>1: fused clip+NVLink allreduce kernel (default) or per-bucket NCCL")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    rank, world, local = dist_init(args.gpus)
    r = bench_clip(args, rank, world, local)
    bert = None
    if not args.no_bert:  # BERT-large MLPerf phase-2 step under the three clip disciplines (all ranks)
        try:
            from paper_2402_02447_b200.train_step import bert_large_step_bench

            bert = {}
            for mode in ("stock", "after", "bucketwise", "reducer", "presort"):
                r_ = bert_large_step_bench(mode, steps=max(3, min(args.steps, 10)), warmup=2)
                bert[mode] = {"samples_per_s": r_["samples_per_s"], "ms_per_step": r_["ms_per_step"]}
                for k in ("buckets", "buckets_iter0", "buckets_after_rebuild", "comm_dtype", "batch_former",
                          "batch_former_ms_per_step", "same_mask_without_former_ms_per_step"):
                    if k in r_:
                        bert[mode][k] = r_[k]
            bert["config"] = ("BertForPreTraining 336M (random init), seq 512, batch 48/GPU, bf16 autocast, AdamW, "
                              "25 MiB buckets; stock/after/bucketwise = DDP (fp32 allreduce), reducer = "
                              "BucketwiseReducer (Algorithm 1, bf16 comm), presort = reducer + per-step batch former "
                              "(K2 strata, native draws, LocalPresort/K3) inside the timed loop")
        except Exception as e:  # transformers missing etc.: report, do not fail the bench
            bert = {"error": str(e)[:200]}
    presort = None
    if rank == 0 and not args.no_presort:
        presort = bench_presort(args)
    bert_base = bench_bert_base(args) if (world == 1 and not args.no_cpu_baseline) else None
    mc = None
    if rank == 0 and not args.no_mcsim:
        from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths

        mc = bench_mcsim(args, generate_lengths(LengthDistribution(), CORPUS_N, CORPUS_SEED))
    if rank == 0:
        line = {
            "metric": "clip+allreduce GB/s", "value": r["value"], "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32->bf16",
            "data": "synthetic",
            "config": {"workload": "BERT-large synthetic gradients (D=335,141,888 fp32, 52 x 25 MiB buckets), "
                                   "bucket-wise clip c/sqrt(52) + bf16 NCCL avg allreduce per bucket",
                       "step": r["mode"],
                       "global_batch": None, "parallelism": f"dp{world}",
                       "l2": "inputs 1.34 GB/rank > 126 MB L2 (no flush needed)"},
            "roofline": r["roofline"], "e2e": r["e2e"], "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
        }
        if "e2e_drop_in" in r:
            line["e2e_drop_in"] = r["e2e_drop_in"]
        if "nvlink" in r:
            line["nvlink"] = r["nvlink"]
        if bert is not None:
            line["bert_large_train"] = bert
        if presort is not None:
            line["presort"] = {"metric": "presort keys/s", "unit": "keys/s",
                               "config": "10M lengths (seed 2402) over 8 shards, Topology(1,8), snake, whole epoch",
                               "l2": "flushed (512 MB write) before every timed iteration", **presort}
        if mc is not None:
            line["mcsim"] = mc
        if bert_base is not None:
            line["config0_bert_base"] = bert_base
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_clip_baseline()
            if presort is not None:
                lens, pools, _ = presort_inputs()
                line["presort"]["cpu_baseline"] = cpu_presort_baseline(lens, pools)
            if mc is not None:
                from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths

                line["mcsim"]["cpu_baseline"] = cpu_mcsim_baseline(
                    generate_lengths(LengthDistribution(), CORPUS_N, CORPUS_SEED))
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
