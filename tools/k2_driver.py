"""K2 alone on the 10M corpus tiled 10x (100M keys, 8 shards): for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2402_02447_b200 import _lib  # noqa: E402
from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths  # noqa: E402

lens = torch.from_numpy(generate_lengths(LengthDistribution(), 10_000_000, 2402)).cuda().repeat(10)
n = lens.numel()
lib = _lib.load()
ws_b = lib.b2_strata_workspace_bytes(n)
ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
ids = torch.empty(n, dtype=torch.int32, device="cuda")
counts = torch.empty((8, 4), dtype=torch.int64, device="cuda")
bad = torch.empty(8, dtype=torch.int64, device="cuda")
offs = _lib.i64_array(r * (n // 8) for r in range(9))
for _ in range(4):
    _lib.check(lib.b2_strata_partition_shards(lens.data_ptr(), None, offs, 8, _lib.i32_array((128, 256, 384, 512)), 4,
                                              ids.data_ptr(), counts.data_ptr(), bad.data_ptr(), ws.data_ptr(), ws_b,
                                              _lib.stream_ptr()))
torch.cuda.synchronize()
print("ok", counts.sum().item())
