"""Property tests (hypothesis) of the H2 kernels on the GPU: random shapes, every path.

K2 (stratify_shards: random shard sizes and strata), K3 and K5 (presort_deal:
pools from 1 key to above one CTA's 4096, 1-16 lanes, lengths with many ties,
repeated ids, raster/snake, with and without input slots) against the oracle
(strata.py:61-83, balance.py:54-75) — `==` on ids, slots and token counts.
"""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import presort_deal, stratify_shards  # noqa: E402

SETTINGS = settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@SETTINGS
@given(data=st.data())
def test_presort_deal_random_shapes(data):
    lanes = data.draw(st.integers(1, 16), label="lanes")
    rows = data.draw(st.sampled_from([1, 2, 3, 5, 16, 48, 64, 257, 300, 600]), label="rows")
    nseg = data.draw(st.integers(1, 6), label="nseg")
    max_len = data.draw(st.sampled_from([1, 7, 64, 512, 1024, 5000]), label="max_len")
    tie_len = data.draw(st.integers(1, max_len), label="tie_len")
    snake = data.draw(st.booleans(), label="snake")
    with_pos = data.draw(st.booleans(), label="with_pos")
    seed = data.draw(st.integers(0, 2**31 - 1), label="seed")
    seg = lanes * rows
    n = nseg * seg
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_len + 1, size=n)
    lens[rng.random(n) < 0.3] = tie_len  # runs of equal lengths
    ids = rng.integers(0, max(1, 2 * n), size=n)  # repeats inside a pool
    max_id = int(max(1, 2 * n))
    out, tok, pos, bad = presort_deal(torch.from_numpy(ids.astype(np.int32)).cuda(),
                                      torch.from_numpy(lens.astype(np.int32)).cuda(), seg, lanes,
                                      "snake" if snake else "raster", max_len=max_len, max_id=max_id,
                                      with_pos=with_pos)
    assert int(bad) == -1
    ro, rt = O.presort_deal_segments(ids, lens, seg, lanes, snake)
    np.testing.assert_array_equal(out.cpu().numpy(), ro)
    np.testing.assert_array_equal(tok.cpu().numpy(), rt)
    if with_pos:  # the slot of every dealt sample: Timsort-stable (equal keys keep input order)
        p = pos.cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(ids[p], ro)
        order = np.lexsort((np.arange(n) % seg, ids, -lens, np.arange(n) // seg))
        ref_pos = order.reshape(nseg, rows, lanes)
        if snake:
            ref_pos[:, 1::2, :] = ref_pos[:, 1::2, ::-1]
        np.testing.assert_array_equal(p, ref_pos.transpose(0, 2, 1))


@SETTINGS
@given(data=st.data())
def test_stratify_shards_random(data):
    nshard = data.draw(st.integers(1, 9), label="nshard")
    sizes = data.draw(st.lists(st.integers(1, 30_000), min_size=nshard, max_size=nshard), label="sizes")
    nb = data.draw(st.integers(1, 16), label="nb")
    top = data.draw(st.sampled_from([16, 512, 4096]), label="top")
    bounds = tuple(sorted(np.random.default_rng(nb * top).choice(np.arange(1, top), size=nb - 1,
                                                               replace=False).tolist()) + [top]) if nb > 1 else (top,)
    seed = data.draw(st.integers(0, 2**31 - 1), label="seed")
    rng = np.random.default_rng(seed)
    offs = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    lens = rng.integers(1, top + 1, size=offs[-1]).astype(np.int32)
    out = stratify_shards(lens, offs, bounds)
    for g in range(nshard):
        pools, probs = O.stratify(lens[offs[g]:offs[g + 1]], bounds)
        assert out[g].probs == probs
        np.testing.assert_array_equal(out[g].ids.cpu().numpy(), np.concatenate(pools))
