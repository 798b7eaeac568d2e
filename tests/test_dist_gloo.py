"""World-size-2 gloo tests of the multi-rank H1 orchestration (CPU, no GPU).

Rank r plays worker row r of the reference's (K, D) matrix
(gradsync.py:43-48): each rank clips its own buckets (no norm collective) and
one allreduce per bucket averages them, in reverse bucket order
(gradsync.py:157).  The clip itself is the oracle here (CUDA is covered by the
-m gpu suites); what is tested is the BucketwiseSync / DDP-hook plumbing.
"""

import numpy as np
import torch
import torch.multiprocessing as mp

from tests import dist_helpers as H

WORLD = 2
DIM = 10_007
LAYOUT = ((0, 3000), (3000, 6000), (6000, 9000), (9000, DIM))


def _sync_worker(rank, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import BucketwiseSync

    H.init(rank, WORLD, port, "gloo")
    try:
        sync = BucketwiseSync(LAYOUT, ClipConfig(1.0, "bucket_wise"), comm_dtype=torch.float32,
                              device="cpu", clip=H.oracle_clip)
        sync.sync(H.worker_grad(rank, DIM))
        out = sync.wait().clone()
        q.put((rank, out.numpy(), sync.norms.numpy()))
    finally:
        dist.destroy_process_group()


def _hook_worker(rank, port, q):
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2402_02447_b200 import ClipConfig
    from paper_2402_02447_b200.ddp import bucketwise_clip_hook, make_hook_state

    H.init(rank, WORLD, port, "gloo")
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 4))
        ddp = DDP(model, bucket_cap_mb=25)  # one bucket: B = 1
        ddp.register_comm_hook(make_hook_state(ClipConfig(0.5, "bucket_wise"), 1, clip=H.oracle_clip),
                               bucketwise_clip_hook)
        torch.manual_seed(10 + rank)
        x = torch.randn(8, 16) * (1.0 + 20.0 * rank)
        ddp(x).pow(2).sum().backward()
        # this rank's raw (unsynchronised) gradient, for the oracle
        model2 = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 4))
        model2.load_state_dict(model.state_dict())
        model2(x).pow(2).sum().backward()
        raw = torch.cat([p.grad.reshape(-1) for p in model2.parameters()])
        synced = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
        q.put((rank, raw.numpy(), synced.numpy()))
    finally:
        dist.destroy_process_group()


def _run(target, attempts: int = 3):
    """WORLD gloo ranks of `target`; a rendezvous that dies early (the picked port was taken)
    is retried on a fresh port."""
    import queue as _queue
    import time

    ctx = mp.get_context("spawn")
    for attempt in range(attempts):
        q = ctx.Queue()
        port = H.free_port()
        procs = [ctx.Process(target=target, args=(r, port, q)) for r in range(WORLD)]
        for p in procs:
            p.start()
        res, failed, t0 = {}, False, time.monotonic()
        while len(res) < WORLD and time.monotonic() - t0 < 120:
            try:
                r, a, b = q.get(timeout=2)
                res[r] = (a, b)
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
        assert len(res) == WORLD, f"{WORLD - len(res)} rank(s) produced no result"
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        return res
    raise AssertionError("multi-rank run failed")


def test_bucketwise_sync_two_ranks_matches_reference_semantics():
    from oracle import ddp_oracle as O

    res = _run(_sync_worker)
    W = np.stack([H.worker_grad(r, DIM).double().numpy() for r in range(WORLD)])
    ref = O.sync_bucketwise(W, LAYOUT, 1.0)
    for r in range(WORLD):
        out, norms = res[r]
        np.testing.assert_allclose(out, ref, rtol=0, atol=1e-6 * np.abs(ref).max())
        rn = [np.linalg.norm(W[r, a:b]) for a, b in reversed(LAYOUT)][::-1]
        np.testing.assert_allclose(norms, rn, rtol=1e-12)
    # both ranks hold the identical averaged gradient
    np.testing.assert_array_equal(res[0][0], res[1][0])


def test_ddp_comm_hook_two_ranks_single_bucket():
    from oracle import ddp_oracle as O

    res = _run(_hook_worker)
    raws = np.stack([res[r][0].astype(np.float64) for r in range(WORLD)])
    ref = O.sync_before(raws, 0.5)  # B = 1: bucket-wise == before-allreduce (criterion 2)
    for r in range(WORLD):
        np.testing.assert_allclose(res[r][1], ref, rtol=0, atol=1e-6 * np.abs(ref).max())
    assert np.linalg.norm(ref) <= 0.5 + 1e-9


LB = 16
STEPS = 5


def _draws(rank):
    rng = np.random.default_rng(50 + rank)
    ids = rng.permutation(100_000)[: STEPS * LB].reshape(STEPS, LB).astype(np.int32) + 100_000 * rank
    lens = rng.integers(1, 513, size=(STEPS, LB)).astype(np.int32)
    return ids, lens


def _oracle_deal(ids, lens, seg_len, lanes, scan):
    from oracle import ddp_oracle as O

    out, tok = O.presort_deal_segments(ids.numpy(), lens.numpy(), seg_len, lanes, scan.value == "snake")
    return torch.from_numpy(out), torch.from_numpy(tok)


def _presort_worker(rank, port, q):
    import torch.distributed as dist

    from paper_2402_02447_b200 import Topology
    from paper_2402_02447_b200.presort_dist import LocalPresort

    H.init(rank, WORLD, port, "gloo")
    try:
        ids, lens = _draws(rank)
        lp = LocalPresort(Topology(1, WORLD), LB, 512, 10**6, "snake", deal=_oracle_deal)
        steps = [lp.step(torch.from_numpy(ids[t]), torch.from_numpy(lens[t])) for t in range(STEPS)]
        ep_ids, ep_tok = lp.epoch(torch.from_numpy(ids), torch.from_numpy(lens))
        q.put((rank, ([o.numpy() for o, _ in steps], [t.numpy() for _, t in steps]), (ep_ids.numpy(), ep_tok.numpy())))
    finally:
        dist.destroy_process_group()


def test_local_presort_two_ranks_matches_reference_semantics():
    from oracle import ddp_oracle as O

    res = _run(_presort_worker)
    draws = [_draws(r) for r in range(WORLD)]
    for t in range(STEPS):
        per_gpu, tok = O.assign_local_presort([d[0][t] for d in draws], [d[1][t] for d in draws], 1, WORLD, True)
        for r in range(WORLD):
            (step_ids, step_tok), (ep_ids, ep_tok) = res[r]
            assert step_ids[t].tolist() == per_gpu[r]
            assert step_tok[t].tolist() == list(tok)
            assert ep_ids[t].tolist() == per_gpu[r]
            assert ep_tok[t].tolist() == list(tok)
