"""The reference's acceptance criteria on the B200 paths (pkg/tests/test_acceptance.py).

Criteria 1-4 (H1 norm cap, single-bucket equivalence, clip formula,
apportionment) are covered in test_gpu_gradsync.py / test_oracle.py; this file
holds the balance-engine criteria, run at the reference's own sizes through
the GPU Monte-Carlo engine.
"""

import numpy as np
import pytest

from oracle import ddp_oracle as O
from paper_2402_02447_b200 import BalanceExperiment, Topology, run_ablation, run_balance_experiment

pytestmark = pytest.mark.gpu


def test_criterion_05_balance_ablation_ordering():
    """test_acceptance.py:99-115: avg_range strictly decreases along none ->
    +stratification -> +local_presorting -> +snake_scanning (gap > 1.645 SE),
    and snake <= 1.05 x global presort; 10,000 trials on Topology(8, 8)."""
    corpus = O.generate_lengths(100_000, 505)
    base = BalanceExperiment("local_presort", Topology(8, 8), corpus, seed=55, local_batch=16, trials=10_000)
    rows = dict(run_ablation(base))
    chain = ["none", "+stratification", "+local_presorting", "+snake_scanning"]
    for earlier, later in zip(chain, chain[1:]):
        a, b = rows[earlier], rows[later]
        gap = a.avg_range - b.avg_range
        assert gap > 1.645 * np.hypot(a.stderr_range, b.stderr_range), (earlier, later)
    assert rows["+snake_scanning"].avg_range <= 1.05 * rows["global_presort"].avg_range


@pytest.mark.parametrize("strategy", ["none", "global_presort", "local_presort", "stratified"])
@pytest.mark.parametrize("scan", ["raster", "snake"])
def test_criterion_06_uniform_corpus_degeneracy(strategy, scan):
    """test_acceptance.py:118-128: an all-512 corpus gives avg_min = avg_max =
    16 x 512 = 8192 for every strategy (PACKING is out of scope here)."""
    corpus = np.full(4096, 512, dtype=np.int64)
    exp = BalanceExperiment(strategy, Topology(8, 8), corpus, seed=66, local_batch=16, trials=25, scan=scan)
    s = run_balance_experiment(exp)
    assert s.avg_min == 8192.0 and s.avg_max == 8192.0
