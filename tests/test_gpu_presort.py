"""H2 parity on the GPU: K2 (strata partition) and K3 (presort + deal) are bit-exact.

Pinned against the reference's golden vectors (tests/golden/h2_golden.json),
the reference KATs, and the oracle at the BASELINE size (10M lengths over 8
rank shards; a whole epoch of node-step pools).
"""

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import (  # noqa: E402
    LengthDistribution,
    Sample,
    StratumAllocation,
    Topology,
    allocate_counts,
    assign_global_presort,
    assign_local_presort,
    draw_batch,
    generate_corpus,
    presort_deal,
    stratify,
    stratify_lengths,
    stratify_shards,
)
from paper_2402_02447_b200 import synthetic  # noqa: E402

BOUNDS = (128, 256, 384, 512)


def make(lengths):
    return [Sample(i, int(x)) for i, x in enumerate(lengths)]


# ------------------------------------------------------------- K2 stratify
def test_stratify_golden(h2_golden):
    for c in h2_golden["corpora"]:
        samples = generate_corpus(LengthDistribution(), c["n"], c["seed"])
        st = stratify(samples, BOUNDS)
        assert [[s.id for s in p] for p in st.buckets] == c["pools"]
        assert list(st.probs) == c["probs"]
        assert list(allocate_counts(st.probs, 16).counts) == c["alloc16"]
        ds = stratify_lengths(np.array(c["lengths"], dtype=np.int32), BOUNDS)
        assert [ds.pool(k).cpu().tolist() for k in range(4)] == c["pools"]
        assert list(ds.probs) == c["probs"]
    e = h2_golden["edge_stratify"]
    st = stratify(make(e["lengths"]), BOUNDS)
    assert [[s.id for s in p] for p in st.buckets] == e["pools"]


def test_stratify_kats():
    st = stratify(make([100, 200, 300, 500]), BOUNDS)
    assert [len(b) for b in st.buckets] == [1, 1, 1, 1] and st.probs == (0.25,) * 4
    st = stratify(make([64] * 10), BOUNDS)
    assert [len(b) for b in st.buckets] == [10, 0, 0, 0] and st.probs == (1.0, 0.0, 0.0, 0.0)
    assert [len(b) for b in stratify(make([128, 129, 256, 257]), BOUNDS).buckets] == [1, 2, 1, 0]
    st = stratify(make([10, 300, 20, 5, 290]), BOUNDS)
    assert [s.id for s in st.buckets[0]] == [0, 2, 3] and [s.id for s in st.buckets[2]] == [1, 4]
    with pytest.raises(ValueError, match="id 7"):
        stratify([Sample(0, 100), Sample(7, 600)], BOUNDS)
    with pytest.raises(ValueError):
        stratify([], BOUNDS)
    with pytest.raises(ValueError):
        stratify(make([10]), (128, 64))
    # first offending sample (input order) is the one named
    with pytest.raises(ValueError, match="id 3 has length 700"):
        stratify([Sample(9, 5), Sample(3, 700), Sample(4, 900)], BOUNDS)
    with pytest.raises(ValueError, match="id 12345"):
        lens = np.full(20000, 7, dtype=np.int32)
        lens[12345] = 513
        lens[19999] = 600
        stratify_lengths(lens, BOUNDS)


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 100_003])
@pytest.mark.parametrize("bounds", [BOUNDS, (512,), (100, 300, 512), (50, 100, 150, 200, 300, 400, 512),
                                    (10, 20, 30, 40, 50, 60, 70, 80, 90, 100, 200, 300, 400, 450, 500, 512)])
def test_stratify_sizes_vs_oracle(n, bounds):
    rng = np.random.default_rng(n + len(bounds))
    lens = rng.integers(1, 513, size=n).astype(np.int32)
    ids = rng.permutation(10 * n)[:n].astype(np.int32)
    ds = stratify_lengths(lens, bounds, ids=ids)
    pools, probs = O.stratify(lens, bounds, ids=ids)
    assert ds.probs == probs
    got = ds.ids.cpu().numpy()
    np.testing.assert_array_equal(got, np.concatenate(pools))


def test_stratify_full_config():
    """10M Wikipedia-like lengths, 8 rank shards of 1.25M: bit-exact per shard."""
    lens = synthetic_lengths()
    shard = lens.size // 8
    offs = [r * shard for r in range(9)]
    sharded = stratify_shards(lens, offs, BOUNDS)  # one device pass over all shards
    for r in range(8):
        part = lens[r * shard:(r + 1) * shard]
        ids = np.arange(r * shard, (r + 1) * shard, dtype=np.int32)
        ds = stratify_lengths(part, BOUNDS, ids=ids)
        pools, probs = O.stratify(part, BOUNDS, ids=ids)
        assert ds.probs == probs and sharded[r].probs == probs
        np.testing.assert_array_equal(ds.ids.cpu().numpy(), np.concatenate(pools))
        np.testing.assert_array_equal(sharded[r].ids.cpu().numpy() + r * shard, np.concatenate(pools))


def test_stratify_shards_ragged_and_errors():
    rng = np.random.default_rng(9)
    sizes = [1, 4095, 4096, 4097, 10_000, 3]
    offs = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    lens = rng.integers(1, 513, size=offs[-1]).astype(np.int32)
    out = stratify_shards(lens, offs, BOUNDS)
    for g in range(len(sizes)):
        part = lens[offs[g]:offs[g + 1]]
        pools, probs = O.stratify(part, BOUNDS)
        assert out[g].probs == probs
        np.testing.assert_array_equal(out[g].ids.cpu().numpy(), np.concatenate(pools))
    lens[offs[4] + 77] = 999
    with pytest.raises(ValueError, match="id 77 has length 999"):
        stratify_shards(lens, offs, BOUNDS)


_LENS = None


def synthetic_lengths():
    global _LENS
    if _LENS is None:
        from paper_2402_02447_b200.seqdata import generate_lengths

        _LENS = generate_lengths(LengthDistribution(), 10_000_000, 2402)
    return _LENS


# ------------------------------------------------------------- K3 presort + deal
def test_local_presort_golden(h2_golden):
    for c in h2_golden["local_presort"]:
        draws = [[Sample(i, x) for i, x in zip(di, dl)] for di, dl in zip(c["draw_ids"], c["draw_lens"])]
        a = assign_local_presort(draws, Topology(c["nodes"], c["gpn"]), c["scan"])
        assert a.to_dict() == {"per_gpu_ids": c["per_gpu_ids"], "token_counts": c["token_counts"]}


def test_global_presort_golden(h2_golden):
    for c in h2_golden["global_presort"]:
        samples = [Sample(i, x) for i, x in zip(c["ids"], c["lens"])]
        a = assign_global_presort(samples, Topology(2, 4), c["scan"])
        assert a.to_dict() == {"per_gpu_ids": c["per_gpu_ids"], "token_counts": c["token_counts"]}


def test_presort_kats():
    def draws(lengths, gpus, per_gpu):
        s = make(lengths)
        return [s[g * per_gpu:(g + 1) * per_gpu] for g in range(gpus)]

    assert assign_local_presort(draws(range(16, 0, -1), 4, 4), Topology(1, 4), "snake").token_counts == (34,) * 4
    assert assign_local_presort(draws(range(16, 0, -1), 4, 4), Topology(1, 4), "raster").token_counts == (40, 36, 32, 28)
    a = assign_local_presort(draws([1, 2, 3, 4, 501, 502, 503, 504], 4, 2), Topology(2, 2), "snake")
    assert {s.id for g in a.per_gpu[:2] for s in g} == {0, 1, 2, 3}
    assert {s.id for g in a.per_gpu[2:] for s in g} == {4, 5, 6, 7}
    a = assign_local_presort(draws([8, 6, 4, 2, 100, 75, 50, 25], 4, 2), Topology(2, 2), "snake")
    assert sum(a.token_counts[:2]) == 20 and sum(a.token_counts[2:]) == 250
    with pytest.raises(ValueError, match="differ"):
        assign_local_presort([make([1, 2]), make([3])], Topology(1, 2), "snake")
    with pytest.raises(ValueError):
        assign_local_presort([make([1]), make([2])], Topology(1, 4), "snake")
    g = assign_global_presort(make(range(16, 0, -1)), Topology(1, 4), "raster")
    assert [s.length for s in g.per_gpu[0]] == [16, 12, 8, 4]
    g = assign_global_presort(make([3, 16, 9, 1, 14, 2, 4, 15]), Topology(1, 2), "raster")
    assert [s.length for s in g.per_gpu[0]] == [16, 14, 4, 2]
    assert [[s.id for s in gpu] for gpu in assign_global_presort(make([9, 9, 9, 9]), Topology(1, 2), "raster").per_gpu] == [[0, 2], [1, 3]]
    with pytest.raises(ValueError, match="divide"):
        assign_global_presort(make([1, 2, 3]), Topology(1, 2))


def test_duplicate_samples_stable():
    """Identical (length, id) samples keep their input order (Timsort stability)."""
    s = [Sample(5, 10), Sample(5, 10), Sample(1, 10), Sample(5, 10)]
    a = assign_global_presort(s, Topology(1, 2), "raster")
    ref = sorted(s, key=lambda x: (-x.length, x.id))
    assert [x is y for x, y in zip([a.per_gpu[0][0], a.per_gpu[1][0], a.per_gpu[0][1], a.per_gpu[1][1]], ref)] == [True] * 4


@pytest.mark.parametrize("seg_len,lanes", [(8, 8), (128, 8), (384, 8), (96, 4), (500, 5), (2048, 8), (4096, 64), (3000, 3)])
@pytest.mark.parametrize("snake", [True, False])
def test_presort_deal_vs_oracle(seg_len, lanes, snake):
    rng = np.random.default_rng(seg_len * 7 + lanes)
    nseg = max(1, 20000 // seg_len)
    lens = rng.integers(1, 513, size=nseg * seg_len).astype(np.int32)
    ids = rng.integers(0, 50_000, size=nseg * seg_len).astype(np.int32)  # repeats allowed
    out, tok, _, bad = presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda(),
                                    seg_len, lanes, "snake" if snake else "raster", max_len=512, max_id=49_999)
    assert int(bad) == -1
    ro, rt = O.presort_deal_segments(ids, lens, seg_len, lanes, snake)
    np.testing.assert_array_equal(out.cpu().numpy(), ro)
    np.testing.assert_array_equal(tok.cpu().numpy(), rt)


def test_presort_full_epoch_vs_oracle():
    """BASELINE config: Topology(1, 8), lb 16 / 48, one epoch of node-step pools."""
    lens = synthetic_lengths()
    shard = lens.size // 8
    for lb in (16, 48):
        ids_r, lens_r = [], []
        for r in range(8):
            part = lens[r * shard:(r + 1) * shard]
            _, probs = O.stratify(part)
            counts = O.allocate_counts(probs, lb)
            i, l = synthetic.epoch_draws(part, (128, 256, 384, 512), counts, None, seed=100 + r)
            ids_r.append(i + r * shard)
            lens_r.append(l)
        steps = min(x.shape[0] for x in ids_r)
        # pool of step t = GPU0's draw, GPU1's draw, ... (balance.py:179-182)
        ids = np.stack([x[:steps] for x in ids_r], axis=1).reshape(-1)
        ln = np.stack([x[:steps] for x in lens_r], axis=1).reshape(-1)
        out, tok, _, bad = presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(ln).cuda(),
                                        8 * lb, 8, "snake", max_len=512, max_id=lens.size - 1)
        assert int(bad) == -1
        ro, rt = O.presort_deal_segments(ids, ln, 8 * lb, 8, True)
        np.testing.assert_array_equal(out.cpu().numpy(), ro)
        np.testing.assert_array_equal(tok.cpu().numpy(), rt)
        # size-independent: every id appears exactly once across the epoch
        assert np.unique(out.cpu().numpy()).size == ids.size


def test_mcsim_second_oracle(h2_golden):
    """Token counts of mcsim's LOCAL_PRESORT trial (mcsim.py:201-212) from K3."""
    for c in h2_golden["mcsim"]:
        mat = np.array(c["mat"], dtype=np.int32)  # (b, G) lengths
        b, G = mat.shape
        gpn, nodes = c["gpn"], c["nodes"]
        pools = mat.reshape(b, nodes, gpn).transpose(1, 0, 2).reshape(-1)
        ids = np.arange(pools.size, dtype=np.int32)
        _, tok, _, _ = presort_deal(torch.from_numpy(ids).cuda(), torch.from_numpy(pools).cuda(),
                                    b * gpn, gpn, c["scan"], max_len=512, max_id=pools.size)
        assert tok.cpu().reshape(-1).tolist() == c["tokens"]


def test_draws_then_presort_end_to_end(h2_golden):
    """Host draws (bit-exact PCG64) -> device presort == reference assignment."""
    for d in h2_golden["draws"]:
        samples = generate_corpus(LengthDistribution(), d["n"], d["seed"])
        st = stratify(samples, d["bounds"])
        al = allocate_counts(st.probs, d["lb"])
        assert list(al.counts) == d["counts"]
        for step, expect in enumerate(d["batches"]):
            if isinstance(expect, dict):
                with pytest.raises(ValueError) as ei:
                    draw_batch(st, al, seed=1000 + step)
                assert str(ei.value) == expect["error"]
                break
            assert [s.id for s in draw_batch(st, al, seed=1000 + step)] == expect
    with pytest.raises(ValueError):
        StratumAllocation((1, 1), 3)


def test_h2_pipeline_end_to_end_full_config():
    """BASELINE config 1 end to end: K2 strata of 8 shards of the 10M corpus ->
    native draws with the real per-(rank, step) seeds derive_seed(2402, r, t)
    -> K3 deal of every node pool; equal, step by step, to the reference
    algorithm (oracle stratify + numpy draw_batch + assign_local_presort)."""
    from paper_2402_02447_b200 import NativeDraws

    lens = synthetic_lengths()
    shard = lens.size // 8
    strata = stratify_shards(lens, [r * shard for r in range(9)], BOUNDS)
    lb, steps = 48, 40
    nat_ids, ref_pools, counts_r = [], [], []
    for r in range(8):
        ds = strata[r]
        ids = ds.ids.cpu().numpy().astype(np.int64) + r * shard
        o = np.concatenate([[0], np.cumsum(ds.counts)])
        pools = [ids[o[k]:o[k + 1]] for k in range(4)]
        counts = allocate_counts(ds.probs, lb).counts
        got, done = NativeDraws(pools, BOUNDS).epoch(counts, 2402, key=(r,), nsteps=steps)
        assert done == steps
        nat_ids.append(got)
        # reference: oracle strata of the shard (input order) + numpy draws
        rp, probs = O.stratify(lens[r * shard:(r + 1) * shard], BOUNDS, ids=np.arange(r * shard, (r + 1) * shard))
        assert probs == ds.probs
        ref_pools.append([p.tolist() for p in rp])
        counts_r.append(O.allocate_counts(probs, lb))
    pool_ids = np.stack(nat_ids, axis=1).reshape(-1).astype(np.int32)  # [steps][gpu][lb]
    pool_lens = lens[pool_ids].astype(np.int32)
    out, tok, _, bad = presort_deal(torch.from_numpy(pool_ids).cuda(), torch.from_numpy(pool_lens).cuda(),
                                    8 * lb, 8, "snake", max_len=512, max_id=lens.size - 1)
    assert int(bad) == -1
    out, tok = out.cpu().numpy(), tok.cpu().numpy()
    for t in range(steps):
        per_gpu_ids, per_gpu_lens = [], []
        for r in range(8):
            s = np.random.SeedSequence(entropy=2402, spawn_key=(r, t)).generate_state(1, np.uint64)[0]
            d = O.draw_batch(ref_pools[r], BOUNDS, counts_r[r], int(s))
            per_gpu_ids.append(d)
            per_gpu_lens.append(lens[np.asarray(d)].tolist())
        for r in range(8):
            assert nat_ids[r][t].tolist() == per_gpu_ids[r], (r, t)
        ref_gpu, ref_tok = O.assign_local_presort(per_gpu_ids, per_gpu_lens, 1, 8, True)
        assert out[t].tolist() == ref_gpu, t
        assert tok[t].tolist() == list(ref_tok), t


@pytest.mark.parametrize("lenrange", [(1, 4), (1, 40), (1, 192), (180, 192)])
@pytest.mark.parametrize("seg_len,lanes", [(128, 8), (384, 8), (512, 4), (96, 3)])
def test_presort_paths_agree_with_heavy_ties(lenrange, seg_len, lanes):
    """Counting-sort path (max_len <= min(1024, 2 pool)), bitonic path (max_len > 1024) and
    the stable radix path (with_pos) give the oracle's deal, with many equal
    lengths (ties broken by id) and ragged pools."""
    rng = np.random.default_rng(seg_len * 7 + lenrange[1])
    nseg = 300
    ids = np.stack([rng.permutation(10 * seg_len)[:seg_len] for _ in range(nseg)]).astype(np.int32)
    lens = rng.integers(lenrange[0], lenrange[1] + 1, size=(nseg, seg_len)).astype(np.int32)
    di, dl = torch.from_numpy(ids.reshape(-1)).cuda(), torch.from_numpy(lens.reshape(-1)).cuda()
    outs = []
    for max_len, pos in ((2 * seg_len, False), (4096, False), (512, True)):
        r = presort_deal(di, dl, seg_len, lanes, "snake", max_len=max_len, max_id=10 * seg_len, with_pos=pos)
        outs.append((r[0].cpu().numpy(), r[1].cpu().numpy()))
    for o, t in outs[1:]:
        assert np.array_equal(o, outs[0][0]) and np.array_equal(t, outs[0][1])
    ro, rt = O.presort_deal_segments(ids.reshape(-1), lens.reshape(-1), seg_len, lanes, True)
    np.testing.assert_array_equal(outs[0][0], ro)
    np.testing.assert_array_equal(outs[0][1], rt)


def test_strategy_properties_conservation_and_snake():
    """TestStrategyProperties (test_balance.py:173-216) on the K3 path:
    conservation + exact token counts over random corpora (hypothesis), and
    snake never worse than raster over 1,000 random global deals."""
    from collections import Counter

    from hypothesis import given, settings
    from hypothesis import strategies as hst

    @given(lengths=hst.lists(hst.integers(1, 512), min_size=1, max_size=96), gpus=hst.sampled_from([1, 2, 4]))
    @settings(max_examples=100, deadline=None)
    def conservation(lengths, gpus):
        usable = len(lengths) - len(lengths) % gpus
        if usable == 0:
            return
        samples = make(lengths[:usable])
        expected = Counter(s.id for s in samples)
        for scan in ("raster", "snake"):
            a = assign_global_presort(samples, Topology(1, gpus), scan)
            assert Counter(s.id for gpu in a.per_gpu for s in gpu) == expected
            assert a.token_counts == tuple(sum(s.length for s in gpu) for gpu in a.per_gpu)
            assert sum(a.token_counts) == sum(s.length for s in samples)

    conservation()
    rng = np.random.default_rng(424242)
    for _ in range(1000):
        gpus = int(rng.choice([2, 4, 8]))
        rows = int(rng.integers(1, 9))
        samples = make(rng.integers(1, 513, size=gpus * rows))
        raster = assign_global_presort(samples, Topology(1, gpus), "raster")
        snake = assign_global_presort(samples, Topology(1, gpus), "snake")
        assert max(snake.token_counts) - min(snake.token_counts) <= max(raster.token_counts) - min(raster.token_counts)


@pytest.mark.parametrize("max_len", [64, 512, 1000])
@pytest.mark.parametrize("seg_len,lanes", [(32, 8), (128, 8), (200, 8), (256, 256), (384, 8), (384, 1), (480, 3),
                                           (512, 16)])
def test_counting_path_every_instantiation(seg_len, lanes, max_len):
    """The warp counting-sort path (b2_presort_deal when 4 * pool >= max_len, max_len <= 1024) in
    every (keys per lane, histogram words) instantiation, one row per lane up to one lane per
    key, raster and snake, with repeated samples (same id, same length) and runs of equal
    lengths: equal to the oracle (balance.py:59-75)."""
    rng = np.random.default_rng(seg_len * 31 + lanes + max_len)
    nseg = 257
    ids = rng.integers(0, 5 * seg_len, size=(nseg, seg_len)).astype(np.int32)  # repeats inside a pool
    lens = rng.integers(1, max_len + 1, size=(nseg, seg_len)).astype(np.int32)
    lens[::3, : seg_len // 2] = rng.integers(max(1, max_len - 3), max_len + 1, size=(len(lens[::3]), seg_len // 2))
    lens[ids % 7 == 0] = 1 + ids[ids % 7 == 0] % max_len  # repeated ids -> identical samples
    di, dl = torch.from_numpy(ids.reshape(-1)).cuda(), torch.from_numpy(lens.reshape(-1)).cuda()
    for scan in ("raster", "snake"):
        out, tok, _, bad = presort_deal(di, dl, seg_len, lanes, scan, max_len=max_len, max_id=5 * seg_len)
        assert int(bad) == -1
        ro, rt = O.presort_deal_segments(ids.reshape(-1), lens.reshape(-1), seg_len, lanes, scan == "snake")
        np.testing.assert_array_equal(out.cpu().numpy(), ro)
        np.testing.assert_array_equal(tok.cpu().numpy(), rt)


def test_counting_path_all_equal_lengths_and_bad_keys():
    """Worst case for the in-bin id ordering (every key in one bin), and the first bad key
    (length 0 / above max_len / negative id) reported as the flat index, as before."""
    seg_len, lanes, nseg = 384, 8, 40
    rng = np.random.default_rng(5)
    ids = np.stack([rng.permutation(100_000)[:seg_len] for _ in range(nseg)]).astype(np.int32)
    lens = np.full((nseg, seg_len), 77, dtype=np.int32)
    di, dl = torch.from_numpy(ids.reshape(-1)).cuda(), torch.from_numpy(lens.reshape(-1)).cuda()
    out, tok, _, bad = presort_deal(di, dl, seg_len, lanes, "snake", max_len=512, max_id=100_000)
    ro, rt = O.presort_deal_segments(ids.reshape(-1), lens.reshape(-1), seg_len, lanes, True)
    np.testing.assert_array_equal(out.cpu().numpy(), ro)
    np.testing.assert_array_equal(tok.cpu().numpy(), rt)
    for flat, field, val in ((5000, "len", 0), (1234, "len", 513), (9000, "id", -3)):
        l2, i2 = lens.reshape(-1).copy(), ids.reshape(-1).copy()
        (l2 if field == "len" else i2)[flat] = val
        r = presort_deal(torch.from_numpy(i2).cuda(), torch.from_numpy(l2).cuda(), seg_len, lanes, "snake",
                         max_len=512, max_id=100_000)
        assert int(r[3]) == flat
