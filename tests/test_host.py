"""CPU-only checks: the C-ABI library, host-side logic and validation (no GPU).

The compute paths themselves are covered by the -m gpu suites; here we pin
what runs on the host (allocate_counts, draw_batch, corpus generation, the
reference's validation errors) and that the library exports every symbol
include/b2ddp.h declares.
"""

import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2402_02447_b200 as B
from paper_2402_02447_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "b2ddp.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(b2_\w+)\(", text, re.M)))


def test_library_exports_header_symbols():
    lib = _lib.load(require_device=False)
    syms = header_symbols()
    assert len(syms) == 35, syms
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, s
    assert lib.b2_version().decode().startswith("b2ddp")
    assert lib.b2_clip_workspace_bytes() > 0


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_argument_errors_without_device():
    """Validation in the C-ABI runs before any device work (returns B2_ERR_*)."""
    lib = _lib.load(require_device=False)
    rc = lib.b2_presort_deal(None, None, 1, 10, 3, 1, 512, 10, None, None, None, None, None)
    assert rc == _lib.B2_ERR_INDIVISIBLE
    assert "do not divide over 3 GPUs" in lib.b2_last_error().decode()
    rc = lib.b2_strata_partition(None, None, 1, None, 4, None, None, None, None, 0, None)
    assert rc == _lib.B2_ERR_INVALID
    rc = lib.b2_weighted_mean(None, 0, 1, 1, 1, None, None, 1, None, 0, None)
    assert rc == _lib.B2_ERR_INVALID
    rc = lib.b2_presort_sort_deal(None, None, 1, 10000, 3, 1, 512, 10, None, None, None, None, None, 0, None)
    assert rc == _lib.B2_ERR_INDIVISIBLE
    # the device-wide sort's scratch: keys x2, histograms, look-back words (1.25M-sample shard)
    ws = lib.b2_presort_workspace_bytes(1, 1_250_000, 512, 1_249_999, 0)
    assert 2 * 8 * 1_250_000 < ws < 40 * 1_250_000
    assert lib.b2_presort_workspace_bytes(1, 4096, 512, 100, 0) == 0  # K3-sized pools need none


def test_spin_timeout_setting():
    """Cross-GPU waits of the fused kernels: configurable bound, 0 = wait forever."""
    lib = _lib.load(require_device=False)
    old = lib.b2_get_spin_timeout()
    assert old >= 0
    assert lib.b2_set_spin_timeout(0.0) == _lib.B2_OK and lib.b2_get_spin_timeout() == 0.0
    assert lib.b2_set_spin_timeout(-1.0) == _lib.B2_ERR_INVALID
    assert lib.b2_set_spin_timeout(old) == _lib.B2_OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(_lib.B2Error, match="no CPU fallback"):
        B.sync_bucketwise(B.GradientState(np.ones((1, 4)), ((0, 4),)), B.ClipConfig(1.0, "bucket_wise"))
    with pytest.raises(_lib.B2Error):
        B.stratify([B.Sample(0, 5)])


def test_config_validation():
    with pytest.raises(ValueError):
        B.ClipConfig(0.0, "after_allreduce")
    with pytest.raises(ValueError):
        B.ClipConfig(float("inf"), "after_allreduce")
    with pytest.raises(ValueError):
        B.ClipConfig(1.0, "sideways")
    assert B.ClipConfig(2.0, "bucket_wise").mode is B.ClipMode.BUCKET_WISE


def test_bucket_layouts():
    assert B.equal_bucket_layout(7, 3) == ((0, 2), (2, 4), (4, 7))
    assert B.equal_bucket_layout(10, 3) == ((0, 3), (3, 6), (6, 10))
    assert B.equal_bucket_layout(4, 4) == ((0, 1), (1, 2), (2, 3), (3, 4))
    with pytest.raises(ValueError):
        B.equal_bucket_layout(3, 4)
    with pytest.raises(ValueError):
        B.equal_bucket_layout(3, 0)
    from paper_2402_02447_b200 import synthetic

    base = synthetic.bert_layout(synthetic.BERT_BASE_DIM)
    large = synthetic.bert_layout(synthetic.BERT_LARGE_DIM)
    assert len(base) == 17 and base[-1][1] - base[-1][0] == 4_624_640
    assert len(large) == 52 and large[-1][1] - large[-1][0] == 908_288


def test_types_validation():
    with pytest.raises(ValueError):
        B.Sample(-1, 5)
    with pytest.raises(ValueError):
        B.Sample(0, 0)
    with pytest.raises(ValueError):
        B.Topology(0, 8)
    assert B.Topology(2, 4).total_gpus == 8
    with pytest.raises(ValueError):
        B.LengthDistribution(bin_probs=(0.5, 0.5, 0.5, 0.5))
    with pytest.raises(ValueError):
        B.StratumAllocation((1, 1), 3)


def test_host_generation_matches_reference(h2_golden):
    for c in h2_golden["corpora"]:
        s = B.generate_corpus(B.LengthDistribution(), c["n"], c["seed"])
        assert [x.length for x in s] == c["lengths"]


def test_allocate_counts_golden(h2_golden):
    for a in h2_golden["allocate"]:
        assert list(B.allocate_counts(a["probs"], a["lb"]).counts) == a["counts"]
    assert B.allocate_counts((5 / 16, 2 / 16, 3 / 16, 6 / 16), 16).counts == (5, 2, 3, 6)
    assert B.allocate_counts((0.373, 0.197, 0.117, 0.314), 16).counts == (6, 3, 2, 5)
    assert B.allocate_counts((0.5, 0.5), 3).counts == (2, 1)
    assert B.allocate_counts((0.3, 0.7), 0).counts == (0, 0)
    with pytest.raises(ValueError, match="negative"):
        B.allocate_counts((0.5, -0.1, 0.6), 8)
    with pytest.raises(ValueError):
        B.allocate_counts((0.0, 0.0), 8)


def test_draw_batch_golden(h2_golden):
    """Host draws reproduce the reference's PCG64 draw sequence and errors exactly."""
    from oracle import ddp_oracle as O

    for d in h2_golden["draws"]:
        lens = B.seqdata.generate_lengths(B.LengthDistribution(), d["n"], d["seed"])
        pools, probs = O.stratify(lens, d["bounds"])  # strata built by the oracle (no GPU here)
        samples = [B.Sample(i, int(x)) for i, x in enumerate(lens)]
        st = B.strata.Strata(tuple(d["bounds"]), [[samples[i] for i in p] for p in pools], probs)
        al = B.allocate_counts(st.probs, d["lb"])
        for step, expect in enumerate(d["batches"]):
            if isinstance(expect, dict):
                with pytest.raises(ValueError) as ei:
                    B.draw_batch(st, al, seed=1000 + step)
                assert str(ei.value) == expect["error"]
                break
            assert [s.id for s in B.draw_batch(st, al, seed=1000 + step)] == expect


def test_timeline_model_restatement_matches_reference_golden():
    """tools/timeline_calibrate.schedule_total == ddpsim timeline.schedule (golden, timeline.py:97-152)."""
    import importlib.util
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    spec = importlib.util.spec_from_file_location("tc", root / "tools" / "timeline_calibrate.py")
    tc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(tc)
    for c in json.loads((root / "tests" / "golden" / "timeline_golden.json").read_text()):
        for mode, total in c["total"].items():
            got = tc.schedule_total(c["t_comp"], c["t_comm"], c["t_clip"], c["t_gclip"], c["t_nred"], mode)
            assert got == total, (mode, got, total)


def test_acceptance_criteria_07_08_timeline():
    """test_acceptance.py:149-165 on the restated model: bucket-wise <= before,
    bucket-wise - after <= the clip costs, over random plans; and the
    hand-scheduled B=2 pipeline."""
    import importlib.util
    from pathlib import Path

    import numpy as np

    spec = importlib.util.spec_from_file_location(
        "tc", Path(__file__).resolve().parent.parent / "tools" / "timeline_calibrate.py")
    tc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(tc)
    rng = np.random.default_rng(7)
    for _ in range(500):
        B = int(rng.integers(1, 13))
        comp = rng.uniform(0.0, 5.0, B) * (rng.random(B) < 0.9)
        comm = rng.uniform(0.0, 5.0, B) * (rng.random(B) < 0.9)
        if comm.sum() == 0.0:
            comm[int(rng.integers(B))] = rng.uniform(0.1, 5.0)
        clip = rng.uniform(0.0, 0.6, B) * (rng.random(B) < 0.8)
        args = (list(comp), list(comm), list(clip), float(clip.sum()), float(rng.uniform(0.0, 1.0)))
        bw = tc.schedule_total(*args, "bucket_wise")
        assert bw <= tc.schedule_total(*args, "before_allreduce") + 1e-9
        assert bw - tc.schedule_total(*args, "after_allreduce") <= clip.sum() + args[3] + 1e-9
    # criterion 8 (test_acceptance.py:161-165): B=2, comp [2, 2], comm [3, 3]
    assert tc.schedule_total([2, 2], [3, 3], [0, 0], 0.0, 0.0, "after_allreduce") == 8.0
    assert tc.schedule_total([2, 2], [3, 3], [0, 0], 0.0, 0.0, "before_allreduce") == 10.0


def test_fused_sync_host_chunks_cover_layout_in_backward_order():
    """FusedBucketSync.sync_host's chunk plan (host logic): consecutive buckets in
    reverse order, each chunk one contiguous range, together covering [0, D)."""
    from paper_2402_02447_b200 import capped_bucket_layout
    from paper_2402_02447_b200.ddp import FusedBucketSync

    for dim, cap, cb in ((335_141_888, 6_553_600, 4), (1000, 96, 3), (1000, 96, 1), (64, 8, 128)):
        fs = object.__new__(FusedBucketSync)  # no device state needed for the plan
        fs.layout = capped_bucket_layout(dim, cap)
        chunks = fs._host_chunks(cb)
        edge = dim
        seen = []
        for c0, n, offs, lens, a, b in chunks:
            assert b == edge and a < b  # walks down from the end without gaps
            seen += list(range(len(fs.layout) - 1 - c0, len(fs.layout) - 1 - c0 - n, -1))
            assert [int(x) for x in offs] == [fs.layout[q][0] for q in seen[-n:]]
            assert sum(int(x) for x in lens) == b - a
            edge = a
        assert edge == 0 and seen == list(range(len(fs.layout) - 1, -1, -1))


def test_allocate_counts_apportionment_stability():
    """test_strata.py:86-97: counts sum to the batch and each is within 1 of its quota."""
    import numpy as np
    from hypothesis import given, settings
    from hypothesis import strategies as hst

    @given(probs=hst.lists(hst.floats(0.0, 1.0), min_size=1, max_size=8).filter(lambda p: sum(p) > 1e-6),
           batch=hst.integers(0, 200))
    @settings(max_examples=200, deadline=None)
    def prop(probs, batch):
        alloc = B.allocate_counts(probs, batch)
        assert sum(alloc.counts) == batch
        quotas = batch * np.asarray(probs) / sum(probs)
        assert all(abs(c - q) < 1.0 for c, q in zip(alloc.counts, quotas))

    prop()
    with pytest.raises(ValueError):
        B.StratumAllocation((1, 1), 3)


def test_c_abi_from_plain_c(tmp_path):
    """The boundary from a non-Python caller: a C program includes
    include/b2ddp.h, links libb2ddp.so and calls host entry points
    (b2_version, b2_derive_seed == numpy's SeedSequence, seeding.py:18-21)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = Path(__file__).resolve().parent.parent
    lib = root / "paper_2402_02447_b200" / "_native"
    src = tmp_path / "abi.c"
    src.write_text(r'''
#include <stdio.h>
#include <inttypes.h>
#include "b2ddp.h"
int main(void) {
  const uint64_t key[2] = {3, 17};
  printf("%s\n%" PRIu64 "\n", b2_version(), b2_derive_seed(2402, key, 2));
  return 0;
}
''')
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c99", "-I", str(root / "include"), str(src), "-L", str(lib), "-lb2ddp",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()
    assert out[0]  # the version string
    ref = int(np.random.SeedSequence(entropy=2402, spawn_key=(3, 17)).generate_state(1, np.uint64)[0])
    assert int(out[1]) == ref
