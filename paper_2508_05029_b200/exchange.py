"""Adaptive Exchange control logic and the row-group
assignment of workers.  phase1 / decide are thin mirrors of
the C functions the engine's exchange pairs run (tq_exchange_phase1 /
tq_exchange_decide, exchange.cu), so the tests exercise the engine's code."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

BROADCAST, HASH_PARTITION = "Broadcast", "HashPartition"
SAMPLE_FRACTION = 0.05
BROADCAST_THRESHOLD = 16 << 20      # 16 MiB per worker


def _lib():
    import ctypes as C

    from .ops import lib
    L = lib()
    if not getattr(L, "_xchg_set", False):
        L.tq_exchange_phase1.restype = C.c_int
        L.tq_exchange_phase1.argtypes = [C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_uint64)]
        L.tq_exchange_decide.restype = C.c_int
        L.tq_exchange_decide.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int, C.c_uint64,
                                         C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L._xchg_set = True
    return L


def exchange_phase1(bytes_so_far: int, progress: float, sample_fraction: float = SAMPLE_FRACTION
                    ) -> Optional[int]:
    """once local scan progress >= sample_fraction emit
    estimate = bytes_so_far / progress (the exact bytes once the scan is
    complete, 0 for an empty input).  The C function the engine's exchange
    pairs call (tq_exchange_phase1, exchange.cu)."""
    import ctypes as C
    e = C.c_uint64()
    if not _lib().tq_exchange_phase1(bytes_so_far, float(progress), sample_fraction, C.byref(e)):
        return None
    return e.value


@dataclass(frozen=True)
class ExchangeDecision:
    strategy: str
    broadcast_side: Optional[int]   # 0 / 1 when Broadcast (the smaller side)
    totals: Tuple[int, int]


def exchange_decide(estimates_side0: Sequence[int], estimates_side1: Sequence[int], n_workers: int,
                    broadcast_threshold: int = BROADCAST_THRESHOLD) -> ExchangeDecision:
    """deterministic on every worker.  Broadcast the smaller
    side if min(total) <= threshold * n_workers, else HashPartition both
    (tq_exchange_decide, exchange.cu — the engine's decision code)."""
    import ctypes as C
    m = max(n_workers, len(estimates_side0), len(estimates_side1))
    a0 = (C.c_uint64 * m)(*estimates_side0)  # (shorter lists: the remaining workers estimated 0)
    a1 = (C.c_uint64 * m)(*estimates_side1)
    if m != n_workers:  # the threshold scales with the worker count, the totals with the entries
        broadcast_threshold = broadcast_threshold * n_workers // m
    side, t0, t1 = C.c_int(), C.c_uint64(), C.c_uint64()
    st = _lib().tq_exchange_decide(a0, a1, m, broadcast_threshold, C.byref(side), C.byref(t0), C.byref(t1))
    if st == 1:
        return ExchangeDecision(BROADCAST, side.value, (t0.value, t1.value))
    return ExchangeDecision(HASH_PARTITION, None, (t0.value, t1.value))


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
