"""The device entry points from a plain-C caller.

tests/c/abi_device.c includes include/b2ddp.h, links libb2ddp.so and the CUDA
runtime, cudaMallocs its buffers and calls b2_bucket_clip_cast (K1),
b2_strata_partition (K2) and b2_presort_deal (K3) — no Python, no torch on
the call path.  Its outputs are checked against the oracle here.
"""

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_device_entry_points_from_plain_c(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    cuda = Path("/usr/local/cuda")
    lib = ROOT / "paper_2402_02447_b200" / "_native"
    exe = tmp_path / "abi_device"
    subprocess.run(["gcc", "-std=c99", "-O2", "-I", str(ROOT / "include"), "-I", str(cuda / "include"),
                    str(ROOT / "tests" / "c" / "abi_device.c"), "-L", str(lib), "-lb2ddp", "-L", str(cuda / "lib64"),
                    "-lcudart", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{cuda / 'lib64'}", "-o", str(exe)], check=True)
    rng = np.random.default_rng(42)
    n, m, nseg, seg, lanes = 1_000_003, 100_003, 50, 384, 8
    g = (rng.normal(size=n) * rng.choice([1e-4, 1e-2], size=n)).astype(np.float32)
    lens = rng.integers(1, 513, size=m).astype(np.int32)
    pids = rng.integers(0, 1 << 24, size=nseg * seg).astype(np.int32)
    plens = rng.integers(1, 513, size=nseg * seg).astype(np.int32)
    for name, arr in (("grad.bin", g), ("lens.bin", lens), ("pool_ids.bin", pids), ("pool_lens.bin", plens)):
        arr.tofile(tmp_path / name)
    out = subprocess.run([str(exe), str(tmp_path), str(n), str(m), str(nseg), str(seg), str(lanes)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("ok")
    # K1 vs sync_bucketwise (one worker, three buckets)
    layout = ((0, n // 3), (n // 3, 2 * (n // 3)), (2 * (n // 3), n))
    ref = O.sync_bucketwise(g.astype(np.float64)[None, :], layout, 1.0)
    clip = np.fromfile(tmp_path / "clip_out.bin", dtype=np.float32)
    assert np.abs(clip - ref).max() <= 1e-5 * np.abs(ref).max()
    norms = np.fromfile(tmp_path / "clip_norms.bin", dtype=np.float64)[::-1]  # call order was reversed
    np.testing.assert_allclose(norms, O.bucket_norms(g, layout), rtol=1e-6)
    # K2 vs stratify
    pools, probs = O.stratify(lens)
    assert np.array_equal(np.fromfile(tmp_path / "strata_ids.bin", dtype=np.int32), np.concatenate(pools))
    cnt = np.fromfile(tmp_path / "strata_counts.bin", dtype=np.int64)
    assert cnt[:4].tolist() == [len(p) for p in pools] and cnt[4] == -1
    # K3 vs the local presort's sort + deal
    ro, rt = O.presort_deal_segments(pids, plens, seg, lanes, True)
    assert np.array_equal(np.fromfile(tmp_path / "deal_ids.bin", dtype=np.int32), ro.reshape(-1))
    assert np.array_equal(np.fromfile(tmp_path / "deal_tokens.bin", dtype=np.int64), rt.reshape(-1))
