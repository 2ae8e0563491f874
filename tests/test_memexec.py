"""Host tier: pinned FixedBufferPool and the chunked layout, checked against
the REFERENCE's own pool/encode_chunked/decode_chunked (oracle/_ref), and the
SPEC inline examples.  CPU-only (the pool falls back to plain
host memory when no driver is present); device spill/load are in
test_gpu_engine.py."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from helpers import rand_batch
from paper_2508_05029_b200.columnar import BOOL, DECIMAL, FLOAT64, INT64, HostBatch, TqError, assert_batches_equal
from paper_2508_05029_b200.ops import Pool, estimate_reservation


def test_pool_examples():
    p = Pool(64, 4)
    ids = p.acquire(4)                       # SPEC.md:63 exact capacity
    assert sorted(ids) == [0, 1, 2, 3] and ids[0] == 0 and p.free_count() == 0
    with pytest.raises(TqError) as e:        # SPEC.md:64 empty pool
        p.acquire(1)
    assert e.value.errc == "PoolExhausted"
    p.release(ids[:2])
    with pytest.raises(TqError):             # double release
        p.release(ids[:1])
    assert p.free_count() == 2
    with pytest.raises(TqError):             # all-or-nothing: pool unchanged
        p.acquire(3)
    assert p.free_count() == 2
    p.close()


def test_pool_stress_no_failures():
    # random acquire/release keeping live <= capacity never fails
    rng = np.random.default_rng(0)
    p = Pool(16, 32)
    live = []
    for _ in range(20000):
        if live and (rng.random() < 0.5 or sum(map(len, live)) >= 28):
            p.release(live.pop(int(rng.integers(len(live)))))
        else:
            n = int(rng.integers(1, 32 - sum(map(len, live)) + 1))
            live.append(p.acquire(n))
    p.close()


def test_chunked_example():
    # 100 B of sections at buffer 64 -> 2 buffers, tail 28 (Bool x 100 rows)
    p = Pool(64, 8)
    b = HostBatch(100, [HostBatch.col_bool(np.arange(100) % 3 == 0)])
    cb = p.encode(b)
    nbuf, tail, total, segs = cb.layout()
    assert (nbuf, tail, total) == (2, 28, 100)
    assert_batches_equal(cb.decode(), b, ordered=True)
    cb.release()
    assert p.free_count() == 8
    empty = HostBatch(0, [HostBatch.col_i64([])])
    cb = p.encode(empty)
    assert cb.layout()[:3] == (0, 0, 0)
    p.close()


@pytest.mark.parametrize("seed", range(8))
def test_chunked_layout_matches_reference(seed):
    L = O.ref()
    if L is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    b = rand_batch(seed, int(rng.integers(0, 300)), (INT64, DECIMAL, BOOL, FLOAT64), null_frac=0.2 if seed % 2 else 0,
                   utf8=True)
    bufsz = int(rng.choice([16, 64, 100, 1 << 20]))
    p = Pool(bufsz, 4096)
    cb = p.encode(b)
    nbuf, tail, total, segs = cb.layout()
    bc = b.to_c()
    rn, rt = C.c_uint64(), C.c_uint64()
    rsegs = (C.c_uint32 * (3 * 8192))()
    rns, ok = C.c_uint32(), C.c_int()
    assert L.tqr_chunked_layout(C.byref(bc), bufsz, 4096, C.byref(rn), C.byref(rt), rsegs, 8192, C.byref(rns),
                                C.byref(ok)) == 0
    assert ok.value == 1
    assert (nbuf, tail) == (rn.value, rt.value)
    assert segs == [tuple(rsegs[3 * i:3 * i + 3]) for i in range(rns.value)]
    assert_batches_equal(cb.decode(), b, ordered=True)
    cb.release()
    p.close()


def test_estimate_reservation_examples():
    MiB = 1 << 20
    assert estimate_reservation(0, 0, 0, 10 * MiB, 2.0) == 20 * MiB
    assert estimate_reservation(5, 0, 3.0, 10 * MiB, 2.0, 1.25) == int(37.5 * MiB)
    assert estimate_reservation(5, 1, 0.1, 10 * MiB, 2.0) == 10 * MiB        # never below the input


def test_on_oom_examples():
    """SPEC.md:390-398, the three on_oom examples (the rule the engine's
    run_task applies; tests/test_gpu_engine.py forces each path in a query)."""
    from paper_2508_05029_b200.ops import on_oom_decide
    assert on_oom_decide(10, 100, False) == ("retry", 20)      # estimate 10 -> 20 <= capacity: retry
    assert on_oom_decide(60, 100, True) == ("split", 120)      # would exceed capacity, 4 batches: split
    assert on_oom_decide(100, 100, False) == ("abort", 200)    # 2x capacity, 1 batch: OutOfMemoryUnsplittable
    assert on_oom_decide(1 << 40, 0, False) == ("retry", 1 << 41)  # capacity 0 = unbounded
    # retry monotonicity (SPEC.md invariants): the estimate strictly grows
    e, seen = 3, []
    for _ in range(5):
        a, e = on_oom_decide(e, 1 << 30, False)
        seen.append(e)
    assert seen == sorted(set(seen))
