"""Programmatic dependent launches chained across kernel families on ONE stream.

K1's lone-bucket launch, K2's scan/scatter, K5's passes and the tile scan are programmatic
dependent launches: each may start under its predecessor's tail and waits for it
(griddepcontrol.wait) before reading.  This interleaves them back to back on a single
stream -- K5 sort, K1 lone bucket, K3 pools, K1, K5 again, K1 -- with no host sync in
between, and checks every result against the oracle (the same bits as run one by one).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import BucketClipper, presort_deal  # noqa: E402
from paper_2402_02447_b200.balance import presort_workspace_bytes  # noqa: E402
from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths  # noqa: E402


def test_pdl_chain_k5_k1_k3_one_stream():
    rng = np.random.default_rng(21)
    st = torch.cuda.Stream()
    # K5 input: two 300k-sample pools, ids shuffled (every digit pass runs) and in order
    n5 = 300_000
    lens5 = generate_lengths(LengthDistribution(), 2 * n5, 77).astype(np.int64)
    ids5 = np.concatenate([rng.permutation(n5), np.arange(n5, 2 * n5)])
    # K3 input: 400 pools of 384
    n3 = 400 * 384
    lens3 = rng.integers(1, 513, n3)
    ids3 = rng.integers(0, 1 << 20, n3)
    # K1 input: three lone buckets of mixed scale
    sizes = [3_000_001, 2_500_000, 4_100_003]
    g = np.concatenate([rng.normal(size=s) * sc for s, sc in zip(sizes, (1e-3, 1e-1, 1e-4))]).astype(np.float32)
    layout, a = [], 0
    for s in sizes:
        layout.append((a, a + s))
        a += s
    lim = 0.3
    with torch.cuda.stream(st):
        d = lambda x: torch.from_numpy(np.ascontiguousarray(x).astype(np.int32)).cuda()
        d_ids5, d_lens5, d_ids3, d_lens3 = d(ids5), d(lens5), d(ids3), d(lens3)
        gd = torch.from_numpy(g).cuda()
        out = torch.empty_like(gd)
        ws = torch.empty(presort_workspace_bytes(2, n5, 512, 2 * n5 - 1), dtype=torch.uint8, device="cuda")
        clip = BucketClipper(stream=st)
    st.synchronize()
    with torch.cuda.stream(st):
        r5a = presort_deal(d_ids5, d_lens5, n5, 8, "snake", max_len=512, max_id=2 * n5 - 1, stream=st, workspace=ws)
        clip.clip_cast(gd, out, [(layout[0][0], layout[0][0], sizes[0])], lim)
        r3 = presort_deal(d_ids3, d_lens3, 384, 8, "raster", max_len=512, max_id=(1 << 20) - 1, stream=st)
        clip.clip_cast(gd, out, [(layout[1][0], layout[1][0], sizes[1])], lim)
        r5b = presort_deal(d_ids5, d_lens5, n5, 1, "raster", max_len=512, max_id=2 * n5 - 1, stream=st,
                           workspace=torch.empty_like(ws))
        clip.clip_cast(gd, out, [(layout[2][0], layout[2][0], sizes[2])], lim)
    st.synchronize()
    for (o, tok, _, bad), seg, lanes, snake, ids, lens in (
            (r5a, n5, 8, True, ids5, lens5), (r3, 384, 8, False, ids3, lens3), (r5b, n5, 1, False, ids5, lens5)):
        ro, rt = O.presort_deal_segments(ids, lens, seg, lanes, snake)
        assert int(bad) == -1
        np.testing.assert_array_equal(o.cpu().numpy().reshape(ro.shape), ro)
        np.testing.assert_array_equal(tok.cpu().numpy().reshape(rt.shape), rt)
    _, rc = O.bucket_coefficients(g.astype(np.float64), layout, lim)
    ref = np.concatenate([g[s:e].astype(np.float64) * rc[b] for b, (s, e) in enumerate(layout)])
    got = out.cpu().numpy().astype(np.float64)
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-5
