"""Native draw port vs numpy (CPU, no GPU): bit-exact draw_batch / derive_seed.

The native port (csrc/draws.cpp) restates numpy's SeedSequence, PCG64,
Lemire bounded ints and Generator.choice(replace=False) (tail shuffle and
Floyd branches); the oracle here is numpy itself running the reference
algorithm (oracle/ddp_oracle.draw_batch, pinned by tests/golden).
"""

import numpy as np
import pytest

from oracle import ddp_oracle as O
from paper_2402_02447_b200 import NativeDraws, derive_seed


def ref_derive(seed, *key):
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))
    return int(ss.generate_state(1, np.uint64)[0])


def test_derive_seed_matches_numpy():
    rng = np.random.default_rng(0)
    cases = [(0,), (1,), (2402,), (2**32 - 1,), (2**32,), (2**63 + 5,), (2**64 - 1,)]
    for s in cases:
        assert derive_seed(*s) == ref_derive(*s)
    for _ in range(300):
        seed = int(rng.integers(0, 2**63))
        key = tuple(int(x) for x in rng.integers(0, 2**40, size=int(rng.integers(0, 4))))
        assert derive_seed(seed, *key) == ref_derive(seed, *key), (seed, key)


def _pools(sizes, seed=0):
    rng = np.random.default_rng(seed)
    out, base = [], 0
    for n in sizes:
        out.append(list(rng.permutation(n) + base))
        base += 10 * n + 7
    return out


@pytest.mark.parametrize("sizes,counts", [
    ([5, 2, 3, 6], [5, 2, 3, 6]),                 # exhaustive (test_strata.py:104-112)
    ([300, 200, 100, 400], [6, 3, 2, 5]),          # Floyd branch (pop <= 10000)
    ([150_000, 80_000, 47_000, 125_000], [6, 3, 2, 5]),    # Floyd branch (pop > 10000, size <= pop/50)
    ([466_000, 246_000, 146_000, 392_000], [18, 9, 6, 15]),  # BASELINE shard, lb 48
    ([20_000, 20_000, 20_000, 20_000], [900, 10, 500, 1]),   # size > pop/50 -> tail shuffle
    ([10_001, 10_001, 30, 30], [201, 200, 30, 1]),           # both sides of the cutoff
    ([1, 5, 5], [3, 0, 0]),                        # borrowing (test_strata.py:140-152)
])
def test_draw_batch_matches_numpy(sizes, counts):
    bounds = [100, 200, 300, 512][: len(sizes)]
    pools_ref = _pools(sizes)
    pools_nat = NativeDraws(pools_ref, bounds)
    for step in range(8):
        seed = ref_derive(2402, 3, step)
        try:
            ref = O.draw_batch(pools_ref, bounds, counts, seed)
        except ValueError as e:
            with pytest.raises(ValueError) as ei:
                pools_nat.draw(counts, seed)
            assert str(ei.value) == str(e)
            break
        got = pools_nat.draw(counts, seed)
        assert got.tolist() == ref, step
        assert pools_nat.remaining() == tuple(len(p) for p in pools_ref)


def test_epoch_and_exhaustion_match_reference(h2_golden):
    """The golden epoch walks (reference run) replayed by the native port."""
    for d in h2_golden["draws"]:
        lens = O.generate_lengths(d["n"], d["seed"])
        pools, probs = O.stratify(lens, d["bounds"])
        nat = NativeDraws([p.tolist() for p in pools], d["bounds"])
        for step, expect in enumerate(d["batches"]):
            if isinstance(expect, dict):
                with pytest.raises(ValueError) as ei:
                    nat.draw(d["counts"], 1000 + step)
                assert str(ei.value) == expect["error"]
                break
            assert nat.draw(d["counts"], 1000 + step).tolist() == expect


def test_epoch_call_equals_step_loop():
    sizes, counts = [150_000, 80_000, 47_000, 125_000], [6, 3, 2, 5]
    bounds = [128, 256, 384, 512]
    a = NativeDraws(_pools(sizes), bounds)
    ids, done = a.epoch(counts, 2402, key=(5,), first_step=0, nsteps=200)
    assert done == 200 and ids.shape == (200, 16)
    ref_pools = _pools(sizes)
    ref = []
    for t in range(200):
        ref.append(O.draw_batch(ref_pools, bounds, counts, ref_derive(2402, 5, t)))
    np.testing.assert_array_equal(ids, np.array(ref))
