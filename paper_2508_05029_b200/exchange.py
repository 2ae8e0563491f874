"""Adaptive Exchange control logic and the row-group
assignment of workers — host-side, pure functions shared by
the single-process engine and the multi-GPU plans.  The data path of the
exchange is tq_comm_exchange / tq_comm_allgather (NCCL, exchange.cu)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

BROADCAST, HASH_PARTITION = "Broadcast", "HashPartition"
SAMPLE_FRACTION = 0.05
BROADCAST_THRESHOLD = 16 << 20      # 16 MiB per worker


def exchange_phase1(bytes_so_far: int, progress: float, sample_fraction: float = SAMPLE_FRACTION
                    ) -> Optional[int]:
    """once local scan progress >= sample_fraction emit
    estimate = bytes_so_far / progress (0 for an empty, finished scan)."""
    if progress >= 1.0 and bytes_so_far == 0:
        return 0
    if progress < sample_fraction or progress <= 0:
        return None
    return int(bytes_so_far / progress)


@dataclass(frozen=True)
class ExchangeDecision:
    strategy: str
    broadcast_side: Optional[int]   # 0 / 1 when Broadcast (the smaller side)
    totals: Tuple[int, int]


def exchange_decide(estimates_side0: Sequence[int], estimates_side1: Sequence[int], n_workers: int,
                    broadcast_threshold: int = BROADCAST_THRESHOLD) -> ExchangeDecision:
    """deterministic on every worker.  Broadcast the smaller
    side if min(total) <= threshold * n_workers, else HashPartition both."""
    t0, t1 = int(sum(estimates_side0)), int(sum(estimates_side1))
    if min(t0, t1) <= broadcast_threshold * n_workers:
        return ExchangeDecision(BROADCAST, 0 if t0 <= t1 else 1, (t0, t1))
    return ExchangeDecision(HASH_PARTITION, None, (t0, t1))


def shard_range(n: int, shard: int, nshards: int) -> Tuple[int, int]:
    """Contiguous row-group subset of worker `shard` (tq_datagen_shard)."""
    return n * shard // nshards, n * (shard + 1) // nshards


def assign_files(sizes: Sequence[int], n_workers: int) -> List[List[int]]:
    """greedy largest-first onto the least-loaded worker."""
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))
    load = [0] * n_workers
    out: List[List[int]] = [[] for _ in range(n_workers)]
    for i in order:
        w = min(range(n_workers), key=lambda k: (load[k], k))
        out[w].append(i)
        load[w] += sizes[i]
    return out
