"""K4 (fused clip + NVLink allreduce) through the C-ABI on ONE GPU: nranks = 1.

The fused kernel's whole protocol — SM role split, registration barrier,
ready/done flags with per-launch epochs, the workspace restore and CUDA-graph
replay — runs at nranks = 1 with this rank's own stage and flag area, so the
1-GPU suite covers it.  Every rank-count instantiation (RMAX 2/4/8, forced
with B2_K4_RMAX) runs, and the result equals the oracle's sync_bucketwise for
one worker (gradsync.py:148-162) within one bf16 rounding.  A non-finite
bucket comes back all-NaN (the rank-local detector the multi-rank path uses).
"""

import ctypes
import os

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import _lib  # noqa: E402

DIM = 6_000_008
LAYOUT = ((0, 1_000_000), (1_000_000, 3_500_000), (3_500_000, 3_500_008), (3_500_008, DIM))


class Single:
    def __init__(self, dim, layout):
        self.lib = _lib.load()
        self.dim, self.layout = dim, layout
        self.stage = torch.zeros(dim, dtype=torch.bfloat16, device="cuda")
        self.flags = torch.zeros(self.lib.b2_p2p_flag_bytes(), dtype=torch.uint8, device="cuda")
        self.ws = torch.empty(self.lib.b2_clip_workspace_bytes(), dtype=torch.uint8, device="cuda")
        _lib.check(self.lib.b2_clip_workspace_init(self.ws.data_ptr(), self.ws.numel(), _lib.stream_ptr()))
        order = list(reversed(range(len(layout))))
        self.offs = _lib.i64_array(layout[b][0] for b in order)
        self.lens = _lib.i64_array(layout[b][1] - layout[b][0] for b in order)
        self.norms = torch.zeros(len(layout), dtype=torch.float64, device="cuda")
        self.nonfinite = torch.zeros(len(layout), dtype=torch.int32, device="cuda")
        self.stages = (ctypes.c_void_p * 1)(self.stage.data_ptr())
        self.flagp = (ctypes.c_void_p * 1)(self.flags.data_ptr())
        self.limit = 1.0 / np.sqrt(len(layout))

    def run(self, g, stream=None):
        _lib.check(self.lib.b2_bucket_clip_allreduce_p2p(
            g.data_ptr(), self.stages, self.flagp, 1, 0, self.offs, self.lens, len(self.layout), self.limit,
            self.norms.data_ptr(), self.nonfinite.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_ptr(stream)))


def grads():
    rng = np.random.default_rng(4)
    g = rng.normal(size=DIM).astype(np.float32)
    g[: 1_000_000] *= 1e-5  # bucket 0 below the limit
    g[1_000_000:3_500_000] *= 1e-2
    return g


@pytest.mark.parametrize("rmax", ["", "2", "4", "8"])
def test_k4_single_rank_matches_oracle(rmax, monkeypatch):
    if rmax:
        monkeypatch.setenv("B2_K4_RMAX", rmax)
    else:
        monkeypatch.delenv("B2_K4_RMAX", raising=False)
    gh = grads()
    g = torch.from_numpy(gh).cuda()
    k = Single(DIM, LAYOUT)
    ref = O.sync_bucketwise(gh.astype(np.float64)[None, :], LAYOUT, 1.0)
    scale = np.abs(ref).max()
    outs = []
    for _ in range(3):  # repeated launches: epoch protocol without resets
        k.stage.zero_()
        k.run(g)
        outs.append(k.stage.float().cpu().numpy())
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        k.run(g, stream=s)
    for _ in range(3):
        k.stage.zero_()
        graph.replay()
        torch.cuda.synchronize()
        outs.append(k.stage.float().cpu().numpy())
    for out in outs:
        assert np.abs(out - ref).max() <= 2.0 ** -8 * scale  # one bf16 rounding of the stage
        np.testing.assert_array_equal(out, outs[0])
    norms = k.norms.flip(0).cpu().numpy()  # call order is reversed bucket order
    rn = np.array([np.linalg.norm(gh[a:b].astype(np.float64)) for a, b in LAYOUT])
    np.testing.assert_allclose(norms, rn, rtol=1e-6)
    assert k.nonfinite.cpu().tolist() == [0] * len(LAYOUT)


def test_k4_nonfinite_bucket_is_all_nan():
    gh = grads()
    gh[2_000_000] = np.inf
    gh[5_000_000] = np.nan
    k = Single(DIM, LAYOUT)
    k.run(torch.from_numpy(gh).cuda())
    out = k.stage.float().cpu().numpy()
    nf = k.nonfinite.flip(0).cpu().tolist()
    assert nf == [0, 1, 0, 1]
    for (a, b), bad in zip(LAYOUT, nf):
        assert np.isnan(out[a:b]).all() if bad else np.isfinite(out[a:b]).all()


def test_k4_rejects_bad_arguments():
    k = Single(DIM, LAYOUT)
    lib = k.lib
    g = torch.zeros(DIM, device="cuda")
    rc = lib.b2_bucket_clip_allreduce_p2p(g.data_ptr(), k.stages, k.flagp, 9, 0, k.offs, k.lens, 4, 0.5,
                                          None, None, k.ws.data_ptr(), k.ws.numel(), None)
    assert rc == _lib.B2_ERR_UNSUPPORTED
    bad_lens = _lib.i64_array([5])
    rc = lib.b2_bucket_clip_allreduce_p2p(g.data_ptr(), k.stages, k.flagp, 1, 0, k.offs, bad_lens, 1, 0.5,
                                          None, None, k.ws.data_ptr(), k.ws.numel(), None)
    assert rc == _lib.B2_ERR_UNSUPPORTED
    os.environ["B2_K4_RMAX"] = "3"
    try:
        rc = lib.b2_bucket_clip_allreduce_p2p(g.data_ptr(), k.stages, k.flagp, 1, 0, k.offs, k.lens, 4, 0.5,
                                              None, None, k.ws.data_ptr(), k.ws.numel(), None)
        assert rc == _lib.B2_ERR_INVALID
    finally:
        del os.environ["B2_K4_RMAX"]


@pytest.mark.parametrize("rmax", ["", "8"])
def test_k4_fp32_stage_single_rank(rmax, monkeypatch):
    """The parity-mode K4 (fp32 stage) at nranks = 1: within the 1e-5 fp32 contract of the oracle."""
    if rmax:
        monkeypatch.setenv("B2_K4_RMAX", rmax)
    else:
        monkeypatch.delenv("B2_K4_RMAX", raising=False)
    gh = grads()
    g = torch.from_numpy(gh).cuda()
    k = Single(DIM, LAYOUT)
    k.stage = torch.zeros(DIM, dtype=torch.float32, device="cuda")
    k.stages = (ctypes.c_void_p * 1)(k.stage.data_ptr())
    ref = O.sync_bucketwise(gh.astype(np.float64)[None, :], LAYOUT, 1.0)
    for _ in range(2):
        _lib.check(k.lib.b2_bucket_clip_allreduce_p2p_dtype(
            g.data_ptr(), k.stages, _lib.B2_F32, k.flagp, 1, 0, k.offs, k.lens, len(LAYOUT), k.limit,
            k.norms.data_ptr(), k.nonfinite.data_ptr(), k.ws.data_ptr(), k.ws.numel(), _lib.stream_ptr()))
        out = k.stage.cpu().numpy()
        assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()
    rc = k.lib.b2_bucket_clip_allreduce_p2p_dtype(g.data_ptr(), k.stages, _lib.B2_F64, k.flagp, 1, 0, k.offs,
                                                  k.lens, len(LAYOUT), k.limit, None, None, k.ws.data_ptr(),
                                                  k.ws.numel(), None)
    assert rc == _lib.B2_ERR_UNSUPPORTED
