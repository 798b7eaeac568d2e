"""H1/H2 across ranks (one process per GPU, NCCL) == reference semantics.

Runs at world = min(#GPUs, 4): on a 1-GPU box every test still runs at
world size 1, so the multi-rank code paths (NCCL communicator, K4's role
split, flags, epochs and graph replay, the DDP hook, LocalPresort) are
exercised by the single-GPU suite too; `gpurun --gpus 2|4` runs them across
ranks.
"""

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests import dist_helpers as H

pytestmark = pytest.mark.gpu

DIM = 20_000_003
LAYOUT = ((0, 6_553_600), (6_553_600, 13_107_200), (13_107_200, 19_660_800), (19_660_800, DIM))
DIM8 = 20_000_008  # the fused path needs 8-element aligned buckets
LAYOUT8 = ((0, 6_553_600), (6_553_600, 13_107_200), (13_107_200, 19_660_800), (19_660_800, DIM8))


def _world():
    return max(1, min(torch.cuda.device_count(), 4))


def _sync_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import BucketwiseSync

    H.init(rank, world, port, "nccl")
    try:
        g = H.worker_grad(rank, DIM).cuda()
        res = {}
        for dt in (torch.float32, torch.bfloat16):
            sync = BucketwiseSync(LAYOUT, ClipConfig(1.0, "bucket_wise"), comm_dtype=dt)
            sync.sync(g)
            res[str(dt)] = sync.wait().float().cpu().numpy()
            res["norms"] = sync.norms.cpu().numpy()
        torch.cuda.synchronize()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _fused_worker(rank, world, port, q, transport="p2p"):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import FusedBucketSync

    H.init(rank, world, port, "nccl")
    try:
        g = H.worker_grad(rank, DIM8).cuda()
        sync = FusedBucketSync(LAYOUT8, ClipConfig(1.0, "bucket_wise"), transport=transport)
        outs = []
        for it in range(3):  # repeated launches exercise the epoch protocol
            outs.append(sync.sync(g).float().cpu().numpy())
        # CUDA-graph replay of the fused step (epoch advanced on the device)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            sync.sync(g, stream=s)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        outs.append(sync.stage.float().cpu().numpy())
        # host-resident streamed step (H2D / K4 per chunk / D2H), several chunk sizes
        gh = g.cpu().pin_memory()
        for cb in (1, 3, 128):
            outs.append(sync.sync_host(gh, chunk_buckets=cb).float().numpy())
        res = {"outs": outs, "norms": sync.norms.cpu().numpy()}
        sync.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _hook_worker(rank, world, port, q):
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import bucketwise_clip_hook, make_hook_state

    H.init(rank, world, port, "nccl")
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.Tanh(), torch.nn.Linear(512, 64)).cuda()
        ref_model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.Tanh(), torch.nn.Linear(512, 64)).cuda()
        ref_model.load_state_dict(model.state_dict())
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=100)  # one bucket: B = 1
        ddp.register_comm_hook(make_hook_state(ClipConfig(0.5, "bucket_wise"), 1), bucketwise_clip_hook)
        torch.manual_seed(10 + rank)
        x = torch.randn(32, 256, device="cuda") * (1.0 + 10.0 * rank)
        ddp(x).pow(2).sum().backward()
        ref_model(x).pow(2).sum().backward()
        raw = torch.cat([p.grad.reshape(-1) for p in ref_model.parameters()]).cpu().numpy()
        synced = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).cpu().numpy()
        q.put((rank, {"raw": raw, "synced": synced}))
    finally:
        dist.destroy_process_group()


def _run(target, world, attempts: int = 3):
    """Spawn `world` ranks of `target`; a rendezvous that dies early (e.g. the picked port was
    taken: EADDRINUSE) is retried on a fresh port instead of waiting out the queue timeout."""
    import queue as _queue
    import time

    ctx = mp.get_context("spawn")
    for attempt in range(attempts):
        q = ctx.Queue()
        port = H.free_port()
        procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        res, failed, t0 = {}, False, time.monotonic()
        while len(res) < world and time.monotonic() - t0 < 300:
            try:
                r, v = q.get(timeout=2)
                res[r] = v
            except _queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    failed = True
                    break
        if failed and attempt + 1 < attempts:
            for p in procs:
                if p.is_alive():
                    p.terminate()
                p.join(timeout=30)
            continue
        assert len(res) == world, f"{world - len(res)} rank(s) produced no result"
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        return res
    raise AssertionError("multi-rank run failed")


def test_bucketwise_sync_nccl_matches_reference():
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_sync_worker, world)
    W = np.stack([H.worker_grad(r, DIM).double().numpy() for r in range(world)])
    ref = O.sync_bucketwise(W, LAYOUT, 1.0)
    scale = np.abs(ref).max()
    for r in range(world):
        out32 = res[r][str(torch.float32)]
        assert np.abs(out32 - ref).max() <= 1e-5 * scale  # fp32 comm buffer: the 1e-5 contract
        out16 = res[r][str(torch.bfloat16)]
        assert np.abs(out16 - ref).max() <= 2.0 ** -7 * scale  # bf16 comm + bf16 NCCL sum
        rn = np.array([np.linalg.norm(W[r, a:b]) for a, b in LAYOUT])
        np.testing.assert_allclose(res[r]["norms"], rn, rtol=1e-6)


def test_ddp_comm_hook_nccl():
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_hook_worker, world)
    raws = np.stack([res[r]["raw"].astype(np.float64) for r in range(world)])
    ref = O.sync_before(raws, 0.5)
    for r in range(world):
        assert np.abs(res[r]["synced"] - ref).max() <= 1e-5 * np.abs(ref).max()


def test_fused_clip_allreduce_p2p_matches_reference():
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_fused_worker, world)
    W = np.stack([H.worker_grad(r, DIM8).double().numpy() for r in range(world)])
    ref = O.sync_bucketwise(W, LAYOUT8, 1.0)
    scale = np.abs(ref).max()
    first = res[0]["outs"][0]
    for r in range(world):
        for out in res[r]["outs"]:
            # bf16 stage per rank + bf16 result: within two bf16 roundings of the fp64 reference
            assert np.abs(out - ref).max() <= 2.0 ** -7 * scale
            # fixed rank-order fp32 sum: every rank, every launch, bit-identical
            np.testing.assert_array_equal(out, first)
        rn = np.array([np.linalg.norm(W[r, a:b]) for a, b in LAYOUT8])
        np.testing.assert_allclose(res[r]["norms"], rn, rtol=1e-6)


def _presort_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import Topology
    from paper_2402_02447_b200.presort_dist import LocalPresort

    H.init(rank, world, port, "nccl")
    try:
        rng = np.random.default_rng(70 + rank)
        ids = (rng.permutation(1_000_000)[: 200 * 48].reshape(200, 48) + 1_000_000 * rank).astype(np.int32)
        lens = rng.integers(1, 513, size=(200, 48)).astype(np.int32)
        lp = LocalPresort(Topology(1, world), 48, 512, 10_000_000, "snake")
        step_ids, step_tok = lp.step(torch.from_numpy(ids[0]).cuda(), torch.from_numpy(lens[0]).cuda())
        ep_ids, ep_tok = lp.epoch(torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda())
        q.put((rank, {"ids": ids, "lens": lens, "step": step_ids.cpu().numpy(), "step_tok": step_tok.cpu().numpy(),
                      "ep": ep_ids.cpu().numpy(), "ep_tok": ep_tok.cpu().numpy()}))
    finally:
        dist.destroy_process_group()


def test_local_presort_nccl_matches_reference():
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_presort_worker, world)
    for t in range(200):
        per_gpu, tok = O.assign_local_presort([res[r]["ids"][t] for r in range(world)],
                                              [res[r]["lens"][t] for r in range(world)], 1, world, True)
        for r in range(world):
            assert res[r]["ep"][t].tolist() == per_gpu[r]
            assert res[r]["ep_tok"][t].tolist() == list(tok)
            if t == 0:
                assert res[r]["step"].tolist() == per_gpu[r]
                assert res[r]["step_tok"].tolist() == list(tok)


def _fused_nvls_worker(rank, world, port, q):
    try:
        _fused_worker(rank, world, port, q, transport="nvls")
    except RuntimeError as e:
        if "multicast" not in str(e):
            raise
        q.put((rank, {"skip": str(e)}))


def test_fused_clip_allreduce_nvls_matches_reference():
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_fused_nvls_worker, world)
    if any("skip" in res[r] for r in range(world)):
        pytest.skip(res[0].get("skip", "no multicast"))
    W = np.stack([H.worker_grad(r, DIM8).double().numpy() for r in range(world)])
    ref = O.sync_bucketwise(W, LAYOUT8, 1.0)
    scale = np.abs(ref).max()
    first = res[0]["outs"][0]
    for r in range(world):
        for out in res[r]["outs"]:
            assert np.abs(out - ref).max() <= 2.0 ** -7 * scale
            np.testing.assert_array_equal(out, first)  # one in-switch sum, broadcast: identical everywhere


def _hook_multi_worker(rank, world, port, q):
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import bucketwise_clip_hook, make_hook_state

    H.init(rank, world, port, "nccl")
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(*[torch.nn.Linear(512, 512) for _ in range(6)]).cuda()  # ~1.6M params
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=1, gradient_as_bucket_view=True)
        state = make_hook_state(ClipConfig(0.7, "bucket_wise"), 1)
        ddp.register_comm_hook(state, bucketwise_clip_hook)
        torch.manual_seed(10 + rank)
        x = torch.randn(16, 512, device="cuda") * (1.0 + 5.0 * rank)
        ddp(x).pow(2).sum().backward()  # iteration 0: one bucket, then DDP rebuilds them
        model.zero_grad(set_to_none=False)
        state.norms.clear()
        ddp(x).pow(2).sum().backward()  # iteration 1: the rebuilt buckets
        state.set_num_buckets(max(state.norms) + 1)
        model.zero_grad(set_to_none=False)
        state.record = {}
        ddp(x).pow(2).sum().backward()
        raw = {k: v.cpu().numpy() for k, v in state.record.items()}
        q.put((rank, {"raw": raw, "nb": state.num_buckets,
                      "grads": torch.cat([p.grad.reshape(-1) for p in model.parameters()]).cpu().numpy()}))
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_multi_bucket_nccl():
    """DDP with several buckets: every parameter gradient equals mean_r clip(bucket_r, c/sqrt(B))."""
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_hook_multi_worker, world)
    nb = res[0]["nb"]
    assert nb >= 3 and all(res[r]["nb"] == nb for r in range(world))
    limit = 0.7 / np.sqrt(nb)
    expected = {}
    for b in range(nb):
        rows = np.stack([res[r]["raw"][b].astype(np.float64) for r in range(world)])
        expected[b] = O.allreduce_mean(np.stack([O.clip_by_norm(row, limit) for row in rows]))
    # every gradient element appears in exactly one bucket: compare multisets of values per rank
    allexp = np.sort(np.concatenate([expected[b] for b in range(nb)]))
    for r in range(world):
        got = np.sort(res[r]["grads"].astype(np.float64))
        assert got.size == allexp.size
        assert np.abs(got - allexp).max() <= 1e-5 * np.abs(allexp).max()


def _fused_large_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig, synthetic
    from paper_2402_02447_b200.ddp import FusedBucketSync

    H.init(rank, world, port, "nccl")
    try:
        dim = synthetic.BERT_LARGE_DIM
        g, layout, _ = synthetic.bert_grads(dim, rank=rank)
        sync = FusedBucketSync(layout, ClipConfig(1.0, "bucket_wise"))
        dev = sync.sync(g).clone()
        host = sync.sync_host(g.cpu().pin_memory())
        torch.cuda.synchronize()
        same = bool(torch.equal(dev.cpu(), host))
        # a few sampled bucket slices, for the oracle comparison in the parent
        picks = [layout[0], layout[len(layout) // 2], layout[-1]]
        q.put((rank, {"same": same, "picks": picks, "norms": sync.norms.cpu().numpy(),
                      "slices": [dev[a:b].float().cpu().numpy() for a, b in picks]}))
        sync.close()
    finally:
        dist.destroy_process_group()


def test_fused_bert_large_streamed_equals_device_and_oracle():
    """BERT-large (52 x 25 MiB): sync_host (H2D / K4 / D2H per chunk) == sync (device),
    bit for bit, identical on every rank, and within bf16 of the oracle on sampled buckets."""
    from oracle import ddp_oracle as O
    from paper_2402_02447_b200 import synthetic

    world = _world()
    res = _run(_fused_large_worker, world)
    dim = synthetic.BERT_LARGE_DIM
    gs = [synthetic.bert_grads(dim, rank=r)[0].cpu().numpy() for r in range(world)]
    for r in range(world):
        assert res[r]["same"]
        for a, b in zip(res[r]["slices"], res[0]["slices"]):
            np.testing.assert_array_equal(a, b)
    B = 52
    limit = 1.0 / np.sqrt(B)
    for (a, b), got in zip(res[0]["picks"], res[0]["slices"]):
        rows = np.stack([gs[r][a:b].astype(np.float64) for r in range(world)])
        ref = O.allreduce_mean(np.stack([O.clip_by_norm(row, limit) for row in rows]))
        assert np.abs(got - ref).max() <= 2.0 ** -7 * np.abs(ref).max()


def _reducer_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.reducer import BucketwiseReducer

    H.init(rank, world, port, "nccl")
    try:
        torch.manual_seed(0)  # identical init on every rank
        m = torch.nn.Sequential(torch.nn.Linear(64, 300), torch.nn.GELU(), torch.nn.Linear(300, 512),
                                torch.nn.GELU(), torch.nn.Linear(512, 10)).cuda()
        g = torch.Generator(device="cuda").manual_seed(100 + rank)  # a different batch per rank
        x = torch.randn(64, 64, device="cuda", generator=g)
        y = torch.randint(0, 10, (64,), device="cuda", generator=g)
        out = {}
        for dt in (torch.float32, torch.bfloat16):
            r = BucketwiseReducer(m.parameters(), ClipConfig(0.5, "bucket_wise"), bucket_cap_mb=0.1, comm_dtype=dt)
            for p_ in m.parameters():  # this rank's own gradient (no reducer hooks)
                p_.grad = None
            r.remove()
            loss = torch.nn.functional.cross_entropy(m(x), y)
            raw = torch.cat([torch.autograd.grad(loss, p_, retain_graph=True)[0].reshape(-1) for p_ in m.parameters()])
            r = BucketwiseReducer(m.parameters(), ClipConfig(0.5, "bucket_wise"), bucket_cap_mb=0.1, comm_dtype=dt)
            torch.nn.functional.cross_entropy(m(x), y).backward()
            r.finish()
            out[str(dt)] = (raw.double().cpu().numpy(), r.flat.double().cpu().numpy(), r.layout)
            r.remove()
        torch.cuda.synchronize()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bucketwise_reducer_nccl_matches_reference():
    """BucketwiseReducer across ranks (rank r = worker row r): every rank ends with
    sync_bucketwise of all ranks' gradients over the reducer's layout (gradsync.py:148-162)."""
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_reducer_worker, world)
    for dt, tol in ((str(torch.float32), 1e-5), (str(torch.bfloat16), 2.0 ** -7)):
        W = np.stack([res[r][dt][0] for r in range(world)])
        layout = res[0][dt][2]
        ref = O.sync_bucketwise(W, layout, 0.5)
        for r in range(world):
            assert np.abs(res[r][dt][1] - ref).max() <= tol * np.abs(ref).max(), (dt, r)


def _fused_f32_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import FusedBucketSync

    H.init(rank, world, port, "nccl")
    try:
        g = H.worker_grad(rank, DIM8).cuda()
        sync = FusedBucketSync(LAYOUT8, ClipConfig(1.0, "bucket_wise"), transport="p2p", comm_dtype=torch.float32)
        assert sync.stage.dtype == torch.float32
        outs = [sync.sync(g).cpu().numpy() for _ in range(2)]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            sync.sync(g, stream=s)
        graph.replay()
        torch.cuda.synchronize()
        outs.append(sync.stage.cpu().numpy())
        outs.append(sync.sync_host(g.cpu().pin_memory(), chunk_buckets=2).numpy())
        res = {"outs": outs, "norms": sync.norms.cpu().numpy()}
        sync.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_fused_clip_allreduce_fp32_parity_mode():
    """K4 with an fp32 stage (b2_bucket_clip_allreduce_p2p_dtype, B2_F32): the fused multi-rank
    path meets the 1e-5 fp32 contract of sync_bucketwise (gradsync.py:148-162), bit-identical
    on every rank and every launch (device, graph replay, host-streamed)."""
    from oracle import ddp_oracle as O

    world = _world()
    res = _run(_fused_f32_worker, world)
    W = np.stack([H.worker_grad(r, DIM8).double().numpy() for r in range(world)])
    ref = O.sync_bucketwise(W, LAYOUT8, 1.0)
    scale = np.abs(ref).max()
    first = res[0]["outs"][0]
    for r in range(world):
        for out in res[r]["outs"]:
            assert np.abs(out - ref).max() <= 1e-5 * scale
            np.testing.assert_array_equal(out, first)
