"""Host-side multi-process plumbing for one party per GPU.

Rank layout: `world` processes form `world // parties` independent sessions
(replicas) of `parties` parties each; rank r is party `r % parties` of
session `r // parties`.  Party 0 of a session creates the NCCL unique id and
broadcasts it to its session through torch.distributed (any backend, gloo in
the CPU tests); the C library then builds its own ncclComm_t from it.
Timing is reduced as the max over ranks.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional


@dataclass(frozen=True)
class PartyLayout:
    rank: int
    world: int
    parties: int

    @property
    def session(self) -> int:
        return self.rank // self.parties

    @property
    def party(self) -> int:
        return self.rank % self.parties

    @property
    def sessions(self) -> int:
        return self.world // self.parties

    def session_ranks(self, session: Optional[int] = None) -> list[int]:
        s = self.session if session is None else session
        return list(range(s * self.parties, (s + 1) * self.parties))


def layout(rank: int, world: int, parties: int = 2) -> PartyLayout:
    if world % parties:
        raise ValueError(f"world size {world} is not a multiple of {parties} parties")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return PartyLayout(rank, world, parties)


def session_groups(lay: PartyLayout):
    """One torch.distributed group per session (every rank must create all of them)."""
    import torch.distributed as dist
    return [dist.new_group(lay.session_ranks(s)) for s in range(lay.sessions)]


def exchange_unique_id(lay: PartyLayout, groups, make_id: Callable[[], bytes]) -> bytes:
    """Party 0 of each session creates the id; every party of the session receives it."""
    import torch.distributed as dist
    obj = [make_id() if lay.party == 0 else None]
    dist.broadcast_object_list(obj, src=lay.session_ranks()[0], group=groups[lay.session])
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id received")
    return bytes(uid)


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
