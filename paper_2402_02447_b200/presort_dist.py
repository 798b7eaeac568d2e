"""H2 across ranks: stratified local presort with one intra-node all-gather per step.

Reference semantics: assign_local_presort (balance.py:158-184) pools each
node's GPU draws in GPU order (:179-182 — the simulated intra-node
all-gather), sorts by (-length, id) and deals; no sample crosses a node
boundary.  Here every rank of a node contributes its `lb` draws through one
all-gather of (id, length) int32 pairs on the node's process group, then runs
K3 on the identical pool and keeps its own lane — deterministic, no scatter,
no cross-node traffic.

``LocalPresort.step`` handles one data-loader step; ``LocalPresort.epoch``
gathers a whole epoch of draws in one collective and deals every node-step
pool in one K3 launch.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .balance import ScanPattern, presort_deal
from .seqdata import Topology


def node_groups(topo: Topology):
    """One process group per node (ranks node*gpn .. node*gpn+gpn-1); returns this rank's."""
    rank = dist.get_rank()
    mine = None
    for node in range(topo.num_nodes):
        ranks = list(range(node * topo.gpus_per_node, (node + 1) * topo.gpus_per_node))
        g = dist.new_group(ranks) if topo.num_nodes > 1 else None
        if rank in ranks:
            mine = g
    return mine


class LocalPresort:
    """Per-step (or per-epoch) local presort of this node's draws; returns this rank's lane."""

    def __init__(self, topo: Topology, local_batch: int, max_len: int, max_id: int,
                 scan: ScanPattern | str = ScanPattern.SNAKE, group=None, deal=None, deferred_check: bool = False):
        self.topo = topo
        self.lb = int(local_batch)
        self.max_len, self.max_id = int(max_len), int(max_id)
        self.scan = ScanPattern(scan)
        self.group = group if group is not None else (node_groups(topo) if topo.num_nodes > 1 else None)
        self.gpn = topo.gpus_per_node
        if dist.get_world_size(self.group) != self.gpn:
            raise ValueError(f"node group has {dist.get_world_size(self.group)} ranks, topology says {self.gpn}")
        self.local = dist.get_rank(self.group)
        # deal(ids, lens, seg_len, lanes, scan) -> (out[nseg, lanes, rows], tokens[nseg, lanes]);
        # K3 by default, replaceable for CPU tests
        self.deal = deal if deal is not None else self._k3
        # deferred_check: keep K3's bad-sample index on the device (no host sync per step, so the
        # host keeps running ahead of the GPU); check() raises for every step since the last check
        self.deferred = bool(deferred_check)
        self._bad = None

    def _k3(self, ids, lens, seg_len, lanes, scan):
        out, tok, _, bad = presort_deal(ids, lens, seg_len, lanes, scan, max_len=self.max_len, max_id=self.max_id)
        if self.deferred:
            self._bad = bad.clone() if self._bad is None else torch.maximum(self._bad, bad)
        elif int(bad) >= 0:
            raise ValueError(f"sample at flat pool index {int(bad)} has length/id outside the declared range")
        return out, tok

    def check(self) -> None:
        """Raise if any deal since the last check met a sample outside the declared range (deferred mode)."""
        if self._bad is not None:
            bad, self._bad = int(self._bad.item()), None
            if bad >= 0:
                raise ValueError("a presorted sample has length/id outside the declared range")

    def _gather(self, mine: torch.Tensor) -> torch.Tensor:
        """[gpn, *mine.shape] of every node rank's tensor, in GPU order (balance.py:180-182)."""
        parts = [torch.empty_like(mine) for _ in range(self.gpn)]
        dist.all_gather(parts, mine.contiguous(), group=self.group)
        return torch.stack(parts)

    def step(self, ids: torch.Tensor, lens: torch.Tensor):
        """One step: this rank's lb draws -> (its dealt ids [lb], the node's token counts [gpn])."""
        if ids.numel() != self.lb or lens.numel() != self.lb:
            raise ValueError(f"per-GPU draw counts differ: expected {self.lb}")
        both = self._gather(torch.stack([ids.to(torch.int32), lens.to(torch.int32)]))  # [gpn, 2, lb]
        pool_ids = both[:, 0, :].reshape(-1)
        pool_lens = both[:, 1, :].reshape(-1)
        out, tok = self.deal(pool_ids, pool_lens, self.gpn * self.lb, self.gpn, self.scan)
        return out[0, self.local], tok[0]

    def epoch(self, ids: torch.Tensor, lens: torch.Tensor):
        """[steps, lb] draws of this rank -> ([steps, lb] dealt ids of this rank, [steps, gpn] tokens)."""
        both = self._gather(torch.stack([ids.to(torch.int32), lens.to(torch.int32)]))  # [gpn, 2, steps, lb]
        # pool of step t = GPU 0's draw, GPU 1's draw, ... -> [steps, gpn, lb]
        pool_ids = both[:, 0].permute(1, 0, 2).reshape(-1)
        pool_lens = both[:, 1].permute(1, 0, 2).reshape(-1)
        out, tok = self.deal(pool_ids, pool_lens, self.gpn * self.lb, self.gpn, self.scan)
        return out[:, self.local, :], tok
