"""H2 parity on the GPU for pools larger than one CTA: K5, the device-wide stable radix sort + deal.

The reference sorts any batch with a stable (-length, id) Timsort
(balance.py:73-75) and deals it (balance.py:59-70); assign_global_presort
(balance.py:83-88) does so over a whole batch.  Every case here is `==`
against the oracle (numpy's stable lexsort) or against Python's own
``sorted`` on the reference's Sample objects: whole 1.25M-sample rank shards
(ids in order -> the device skips the id digits; ids shuffled -> every digit
pass runs), a 100k-sample global presort with duplicate samples, many pools
per launch, ragged tile tails, full-width keys and invalid samples.
"""

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import (  # noqa: E402
    Sample,
    Topology,
    assign_global_presort,
    generate_lengths,
    LengthDistribution,
    presort_deal,
    stratify_lengths,
)
from paper_2402_02447_b200.balance import MAX_POOL, sort_shard  # noqa: E402


def oracle_pos(ids, lens, seg_len, lanes, snake):
    """Input slot of every dealt sample (stable order), shaped like out_ids."""
    ids = np.asarray(ids, np.int64)
    lens = np.asarray(lens, np.int64)
    nseg = ids.size // seg_len
    rows = seg_len // lanes
    out = np.empty((nseg, lanes, rows), np.int64)
    lane_of = O.deal_lanes(seg_len, lanes, snake)
    row_of = np.arange(seg_len) // lanes
    for s in range(nseg):
        sl = slice(s * seg_len, (s + 1) * seg_len)
        order = O.sorted_desc_order(lens[sl], ids[sl]) + s * seg_len
        out[s, lane_of, row_of] = order
    return out


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def check(ids, lens, seg_len, lanes, snake, max_len, max_id, with_pos=True):
    out, tok, pos, bad = presort_deal(dev(ids), dev(lens), seg_len, lanes, "snake" if snake else "raster",
                                      max_len=max_len, max_id=max_id, with_pos=with_pos)
    ro, rt = O.presort_deal_segments(ids, lens, seg_len, lanes, snake)
    assert int(bad) == -1
    np.testing.assert_array_equal(out.cpu().numpy(), ro)
    np.testing.assert_array_equal(tok.cpu().numpy(), rt)
    if with_pos:
        np.testing.assert_array_equal(pos.cpu().numpy(), oracle_pos(ids, lens, seg_len, lanes, snake))


def test_whole_shard_ids_in_order():
    """One 1.25M-sample rank shard (BASELINE config), ids ascending: length passes only."""
    n = 1_250_000
    lens = generate_lengths(LengthDistribution(), n, 2402).astype(np.int64)
    ids = np.arange(n)
    s_ids, tok, _, bad = sort_shard(dev(ids), dev(lens), max_len=512, max_id=n - 1)
    order = O.sorted_desc_order(lens, ids)
    assert int(bad) == -1
    np.testing.assert_array_equal(s_ids.cpu().numpy(), ids[order])
    assert int(tok[0]) == int(lens.sum())
    check(ids, lens, n, 8, True, 512, n - 1)


def test_whole_shard_ids_shuffled_and_stratified():
    """Ids out of order (every digit pass runs): a random permutation and K2's stratified order."""
    n = 1_250_000
    rng = np.random.default_rng(5)
    lens = generate_lengths(LengthDistribution(), 10_000_000, 2402)[:n].astype(np.int64)
    ids = rng.permutation(10_000_000)[:n]
    check(ids, lens, n, 1, False, 512, 10_000_000 - 1)
    check(ids, lens, n, 8, True, 512, 10_000_000 - 1, with_pos=False)
    ds = stratify_lengths(lens.astype(np.int32))  # ids grouped by stratum, input order inside
    sids = ds.ids.cpu().numpy().astype(np.int64)
    check(sids, lens[sids], n, 8, True, 512, n - 1)


def test_global_presort_100k_with_duplicates():
    """assign_global_presort over a 100k-sample batch (balance.py:83-88), Sample objects, ties."""
    rng = np.random.default_rng(11)
    n = 100_000
    ids = rng.integers(0, 30_000, n)  # many duplicate (len, id) samples
    lens = rng.integers(1, 65, n)
    batch = [Sample(int(i), int(x)) for i, x in zip(ids, lens)]
    topo = Topology(2, 8)
    for scan in ("raster", "snake"):
        got = assign_global_presort(batch, topo, scan)
        ordered = sorted(batch, key=lambda s: (-s.length, s.id))  # the reference's Timsort
        g = topo.total_gpus
        want = [[] for _ in range(g)]
        for r in range(n // g):
            row = ordered[r * g:(r + 1) * g]
            if scan == "snake" and r % 2 == 1:
                row = row[::-1]
            for lane, s in enumerate(row):
                want[lane].append(s)
        assert all(len(a) == len(b) and all(x is y for x, y in zip(a, b)) for a, b in zip(got.per_gpu, want))
        assert got.token_counts == tuple(sum(s.length for s in gpu) for gpu in want)


@pytest.mark.parametrize("seg_len,nseg,lanes", [(MAX_POOL + 8, 3, 8), (8192, 5, 16), (12_289, 2, 1),
                                                (40_000, 7, 40), (102_400, 2, 1024), (65_536, 3, 2048)])
def test_many_pools_ragged_tiles(seg_len, nseg, lanes):
    if seg_len % lanes:
        pytest.skip("indivisible")
    rng = np.random.default_rng(seg_len + nseg)
    ids = rng.integers(0, 1 << 20, seg_len * nseg)
    lens = rng.integers(1, 513, seg_len * nseg)
    check(ids, lens, seg_len, lanes, True, 512, (1 << 20) - 1)
    check(ids, lens, seg_len, lanes, False, 512, (1 << 20) - 1, with_pos=False)


@pytest.mark.parametrize("max_len,lanes,nseg", [(4096, 300, 3), (512, 1, 5), (100_000, 7, 2)])
def test_ordered_ids_multi_length_pass(max_len, lanes, nseg):
    """Ids ascending in every pool: the first length pass takes tabled tile bases; with wide lengths
    the later length passes resolve theirs by look-back.  Lanes > 256 (token sums straight to
    global memory), one lane (register sums), ragged last tile, many pools."""
    rng = np.random.default_rng(max_len + lanes)
    seg_len = lanes * (21_000 // lanes + 1)
    ids = np.concatenate([np.sort(rng.integers(0, 1 << 24, seg_len)) for _ in range(nseg)])
    lens = rng.integers(1, max_len + 1, seg_len * nseg)
    lens[::5] = max_len // 3 + 1  # ties on length
    check(ids, lens, seg_len, lanes, True, max_len, (1 << 24) - 1)
    check(ids, lens, seg_len, lanes, False, max_len, (1 << 24) - 1, with_pos=False)


def test_full_width_keys_and_sorted_segments():
    """Default bounds (31-bit ids and lengths -> 7 digit passes); ids sorted in some pools only."""
    rng = np.random.default_rng(3)
    seg_len, nseg = 9000, 3
    ids = np.concatenate([np.arange(seg_len), rng.integers(0, 2**31 - 1, seg_len), np.arange(seg_len)[::-1]])
    lens = rng.integers(1, 2**31 - 1, seg_len * nseg)
    lens[::7] = 5  # ties on length
    check(ids, lens, seg_len, 9, True, 2**31 - 1, 2**31 - 1)


def test_all_equal_keys_keep_input_order():
    n = 20_000
    ids = np.full(n, 7)
    lens = np.full(n, 100)
    check(ids, lens, n, 4, True, 512, 7)


def test_bad_samples_and_indivisible():
    n = 10_000
    ids = np.arange(n)
    lens = np.full(n, 10)
    lens[4321] = 0
    lens[9000] = 600
    _, _, _, bad = presort_deal(dev(ids), dev(lens), n, 8, "snake", max_len=512, max_id=n - 1)
    assert int(bad) == 4321
    with pytest.raises(ValueError, match="do not divide"):
        presort_deal(dev(ids), dev(lens), n, 3, "snake", max_len=512, max_id=n - 1)


def test_repeatable_and_graph_capturable():
    """Two launches give identical bits; the launch sequence replays inside a CUDA graph."""
    n = 300_000
    rng = np.random.default_rng(9)
    ids, lens = dev(rng.integers(0, 1 << 22, n)), dev(rng.integers(1, 513, n))
    from paper_2402_02447_b200.balance import presort_workspace_bytes

    ws = torch.empty(presort_workspace_bytes(1, n, 512, (1 << 22) - 1, True), dtype=torch.uint8, device="cuda")
    a = presort_deal(ids, lens, n, 8, "snake", 512, (1 << 22) - 1, True, workspace=ws)
    b = presort_deal(ids, lens, n, 8, "snake", 512, (1 << 22) - 1, True, workspace=ws)
    assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2]) and torch.equal(a[1], b[1])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        presort_deal(ids, lens, n, 8, "snake", 512, (1 << 22) - 1, True, workspace=ws)  # warm
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        c = presort_deal(ids, lens, n, 8, "snake", 512, (1 << 22) - 1, True, workspace=ws)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(a[0], c[0]) and torch.equal(a[2], c[2]) and torch.equal(a[1], c[1])
