"""Every product kernel once at small sizes, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py [--only k1,k2,...]

Covers K1 (multi-bucket warp-specialised, lone bucket, fp64, non-finite flags),
K1b, K2 (all shards, ragged + misaligned shards, 16 strata), K3 (counting sort,
bitonic network, block radix with slots), K5 (device-wide onesweep with and
without slots, snake deal), the Monte-Carlo draw/count kernels and K4 at
nranks = 1 (its flag/epoch protocol on one GPU).  Each result is checked
against the oracle so a sanitizer pass also means a correct run.
"""

from __future__ import annotations

import argparse
import ctypes
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2402_02447_b200 as B  # noqa: E402
from oracle import ddp_oracle as O  # noqa: E402
from paper_2402_02447_b200 import _lib  # noqa: E402


def k1():
    rng = np.random.default_rng(1)
    D = 3_000_011
    g = (rng.normal(size=D) * 1e-3).astype(np.float32)
    layout = B.equal_bucket_layout(D, 6)
    lim = 1.0 / math.sqrt(len(layout))
    ref = O.sync_bucketwise(g.astype(np.float64)[None, :], layout, 1.0)
    dg = torch.from_numpy(g).cuda()
    clip = B.BucketClipper()
    out = torch.empty_like(dg)
    segs = [(a, a, b - a) for a, b in reversed(layout)]
    clip.clip_cast(dg, out, segs, lim)  # every bucket in one launch
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-5 * np.abs(ref).max()
    for s in segs[:2]:  # the lone-bucket (hook) shape
        clip.clip_cast(dg, out, [s], lim)
    comm = torch.empty(D, dtype=torch.bfloat16, device="cuda")
    clip.clip_cast(dg, comm, segs, lim)
    d64 = dg.double()
    o64 = torch.empty_like(d64)
    flags = torch.zeros(len(segs), dtype=torch.int32, device="cuda")
    clip.clip_cast(d64, o64, segs, lim, nonfinite=flags)
    assert np.abs(o64.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    bad = dg.clone()
    bad[5] = float("inf")
    clip.clip_cast(bad, out, segs, lim, nonfinite=flags)
    assert int(flags.sum()) == 1
    w = rng.normal(size=(5, 20_000))
    got = B.sync_bucketwise(B.GradientState(w, B.equal_bucket_layout(20_000, 3)), B.ClipConfig(1.0, "bucket_wise"))
    ref = O.sync_bucketwise(w, B.equal_bucket_layout(20_000, 3), 1.0)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def k2():
    rng = np.random.default_rng(2)
    sizes = [1, 4095, 4097, 10_001, 3, 50_000]
    offs = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    lens = rng.integers(1, 513, size=offs[-1]).astype(np.int32)
    for bounds in ((128, 256, 384, 512), (100, 300, 512), tuple(range(32, 513, 32))):
        out = B.stratify_shards(lens, offs, bounds)
        for gi in range(len(sizes)):
            pools, probs = O.stratify(lens[offs[gi]:offs[gi + 1]], bounds)
            assert np.array_equal(out[gi].ids.cpu().numpy(), np.concatenate(pools)) and out[gi].probs == probs


def k3():
    rng = np.random.default_rng(3)
    for seg, lanes, max_len, pos in ((384, 8, 512, False), (128, 8, 512, False), (96, 3, 4096, False),
                                     (512, 4, 1000, False), (384, 8, 512, True), (2048, 8, 512, True)):
        nseg = 37
        ids = rng.integers(0, 10 * seg, size=nseg * seg).astype(np.int32)
        ln = rng.integers(1, min(max_len, 512) + 1, size=nseg * seg).astype(np.int32)
        out, tok, _, bad = B.presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(ln).cuda(), seg, lanes,
                                          "snake", max_len=max_len, max_id=10 * seg, with_pos=pos)
        ro, rt = O.presort_deal_segments(ids, ln, seg, lanes, True)
        assert int(bad) == -1 and np.array_equal(out.cpu().numpy(), ro) and np.array_equal(tok.cpu().numpy(), rt)


def k5():
    rng = np.random.default_rng(5)
    for seg, lanes, pos in ((20_000, 1, False), (20_000, 8, True), (9_000, 3, False)):
        nseg = 3
        ids = rng.permutation(nseg * seg).astype(np.int32)
        ln = rng.integers(1, 513, size=nseg * seg).astype(np.int32)
        out, tok, _, bad = B.presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(ln).cuda(), seg, lanes,
                                          "snake", max_len=512, max_id=nseg * seg, with_pos=pos)
        ro, rt = O.presort_deal_segments(ids, ln, seg, lanes, True)
        assert int(bad) == -1 and np.array_equal(out.cpu().numpy(), ro) and np.array_equal(tok.cpu().numpy(), rt)
    ids = np.arange(30_000, dtype=np.int32)  # ids in order: the id digits are skipped
    ln = rng.integers(1, 513, size=30_000).astype(np.int32)
    out, tok, _, _ = B.presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(ln).cuda(), 30_000, 1, "raster",
                                    max_len=512, max_id=30_000)
    ro, rt = O.presort_deal_segments(ids, ln, 30_000, 1, False)
    assert np.array_equal(out.cpu().numpy(), ro)


def mc():
    from paper_2402_02447_b200.mcsim import run_trials

    lens = B.seqdata.generate_lengths(B.LengthDistribution(), 20_000, 2402)
    exp = B.BalanceExperiment("local_presort", B.Topology(2, 8), lens, seed=7, local_batch=16, trials=4, scan="snake")
    mins, maxs = run_trials(exp, draws="device")
    ref = [O.mcsim_trial_counts("local_presort", lens, O.DEFAULT_BOUNDS, 16, 2, 8, True, 7, t) for t in range(4)]
    assert mins.tolist() == [int(r.min()) for r in ref]


def k4():
    lib = _lib.load()
    D = 2_000_008
    layout = ((0, 500_000), (500_000, 1_500_000), (1_500_000, D))
    stage = torch.zeros(D, dtype=torch.bfloat16, device="cuda")
    flags = torch.zeros(lib.b2_p2p_flag_bytes(), dtype=torch.uint8, device="cuda")
    ws = torch.empty(lib.b2_clip_workspace_bytes(), dtype=torch.uint8, device="cuda")
    _lib.check(lib.b2_clip_workspace_init(ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
    order = list(reversed(range(len(layout))))
    offs = _lib.i64_array(layout[b][0] for b in order)
    lens = _lib.i64_array(layout[b][1] - layout[b][0] for b in order)
    norms = torch.zeros(len(layout), dtype=torch.float64, device="cuda")
    nonfin = torch.zeros(len(layout), dtype=torch.int32, device="cuda")
    g = torch.from_numpy((np.random.default_rng(4).normal(size=D) * 1e-3).astype(np.float32)).cuda()
    for _ in range(2):
        _lib.check(lib.b2_bucket_clip_allreduce_p2p(
            g.data_ptr(), (ctypes.c_void_p * 1)(stage.data_ptr()), (ctypes.c_void_p * 1)(flags.data_ptr()), 1, 0,
            offs, lens, len(layout), 1.0 / math.sqrt(len(layout)), norms.data_ptr(), nonfin.data_ptr(),
            ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
    ref = O.sync_bucketwise(g.double().cpu().numpy()[None, :], layout, 1.0)
    assert np.abs(stage.float().cpu().numpy() - ref).max() <= 2.0 ** -7 * np.abs(ref).max()


ALL = {"k1": k1, "k2": k2, "k3": k3, "k5": k5, "mc": mc, "k4": k4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(ALL))
    a = ap.parse_args()
    for name in a.only.split(","):
        ALL[name]()
        torch.cuda.synchronize()
        print(f"{name} ok", flush=True)


if __name__ == "__main__":
    main()
