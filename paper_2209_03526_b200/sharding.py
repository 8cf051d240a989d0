"""Row sharding across GPUs: one process per GPU.

secEval shards naturally: candidate rows are independent.  Vertex tables are
partitioned by vertex-id ranges whose sizes are multiples of 128 rows, so
every shard's packed output starts on a 16-byte CTR block of the zero-share
stream (128 rows = 4 words = 1 AES block).  Each rank evaluates its rows for
all three co-resident parties, blinds them with *its slice* of the
zero-share stream (random access by CTR block, ogm_zero_share_slice), and
the one exchange -- an all-gather of the packed blinded bits -- rebuilds the
full re-shared vector on every rank, bit-identical to the single-GPU run.
Party messages never cross NVLink: the three servers live on every GPU.

The plan / assembly logic is device-agnostic (covered by gloo tests on CPU);
:func:`sharded_sec_eval_trio` is the CUDA path (NCCL all-gather).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib, fss
from .bits import words_for

ALIGN_ROWS = 128  # one AES-CTR block of packed bits


@dataclass(frozen=True)
class ShardPlan:
    rows: int
    world: int
    align: int = ALIGN_ROWS

    @property
    def per_rank(self) -> int:
        per = -(-self.rows // self.world)
        return -(-per // self.align) * self.align

    def bounds(self, rank: int) -> tuple[int, int]:
        lo = min(rank * self.per_rank, self.rows)
        return lo, min(lo + self.per_rank, self.rows)

    def word_bounds(self, rank: int) -> tuple[int, int]:
        lo, hi = self.bounds(rank)
        return lo // 32, words_for(hi) if hi > lo else lo // 32

    @property
    def words_per_rank(self) -> int:
        return self.per_rank // 32

    @property
    def total_words(self) -> int:
        return words_for(self.rows)


def pad_slice(local: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """Local packed words -> fixed-size all-gather chunk (zero padded)."""
    out = torch.zeros((plan.words_per_rank,), dtype=local.dtype, device=local.device)
    out[: local.numel()] = local
    return out


def assemble(gathered: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """All-gathered chunks (world * words_per_rank) -> the full packed vector."""
    parts = []
    for r in range(plan.world):
        lo, hi = plan.word_bounds(r)
        parts.append(gathered[r * plan.words_per_rank: r * plan.words_per_rank + (hi - lo)])
    return torch.cat(parts)[: plan.total_words]


def all_gather_bits(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    import torch.distributed as dist
    chunk = pad_slice(local, plan)
    out = torch.empty((plan.world * plan.words_per_rank,), dtype=chunk.dtype, device=chunk.device)
    dist.all_gather_into_tensor(out, chunk, group=group)
    return assemble(out, plan)


def sharded_sec_eval_trio(comps, words: int, plan: ShardPlan, rank: int, inds, zero_keys, counters,
                          group=None) -> list:
    """One secEval for all three parties on this rank's row shard.

    comps: the three (rows_local, pitch) share components of this shard.
    inds:  [pass][party] -> (ind_a, ind_b) full-domain indicator words.
    zero_keys: [(k_own, k_prev)] per party (src/net.py:229-232).
    counters: zero-share counter per pass (identical across parties).
    Returns per pass the three parties' full blinded vectors (all ranks),
    i.e. the re-share messages; component j of the result is blinded_{j-1}.
    """
    lo, hi = plan.bounds(rank)
    nloc = hi - lo
    npass = len(inds)
    dev = comps[0].device
    outs = [torch.empty((max(words_for(nloc), 1),), dtype=torch.int32, device=dev) for _ in range(3 * npass)]
    A = _lib.ptr_array
    if nloc:
        flat = [t for ps in range(npass) for q in range(3) for t in inds[ps][q]]
        _lib.call("ogm_masked_parity", nloc, words, comps[0].stride(0), 3, A(comps), 3,
                  _lib.int_array([0, 1, 2]), _lib.int_array([1, 2, 0]), npass, A(flat), A(outs),
                  _lib.stream_ptr())
    w0, w1 = plan.word_bounds(rank)
    result = []
    for ps in range(npass):
        full = []
        for q in range(3):
            add = outs[ps * 3 + q][: w1 - w0]
            k_own, k_prev = zero_keys[q]
            if w1 > w0:
                _lib.call("ogm_zero_share_slice", k_own, k_prev, counters[ps], plan.rows, w0, w1 - w0,
                          _lib.ptr(add), _lib.ptr(add), _lib.stream_ptr())
            full.append(all_gather_bits(add, plan, group) if plan.world > 1 else add)
        result.append(full)
    return result


__all__ = ["ShardPlan", "pad_slice", "assemble", "all_gather_bits", "sharded_sec_eval_trio", "fss"]
