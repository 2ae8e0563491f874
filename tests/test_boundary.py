"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/*.h declares, and refuses to run without one
(no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h)
           for h in ("tq_gpu.h", "tq_exchange.h", "tq_memexec.h", "tq_engine.h", "tq_storage.h")]


def declared_functions():
    names = []
    for h in HEADERS:
        if not os.path.exists(h):
            continue
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(tq_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2508_05029_b200 import ops
    L = ops.lib()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_struct_layouts_match_header():
    from paper_2508_05029_b200.columnar import TqBatchC, TqColumnC, TqExprNodeC
    assert C.sizeof(TqColumnC) == 40
    assert C.sizeof(TqBatchC) == 32
    assert C.sizeof(TqExprNodeC) == 32


def test_batch_set_rows_trims_the_descriptor():
    """tq_batch_set_rows (the asynchronous operators' trim) is host-only: it
    shortens rows and every fixed-width column's values_bytes, never grows."""
    import numpy as np
    from paper_2508_05029_b200 import ops
    from paper_2508_05029_b200.columnar import DECIMAL, INT64, HostBatch
    b = HostBatch(10)
    b.cols.append(HostBatch.col_i64(np.arange(10)))
    b.cols.append(HostBatch.col_dec(np.arange(10), 12, 2))
    c = b.to_c()
    ops.lib().tq_batch_set_rows(C.byref(c), 4)
    assert c.rows == 4
    assert [c.cols[i].values_bytes for i in range(2)] == [32, 64]
    ops.lib().tq_batch_set_rows(C.byref(c), 7)  # larger than the current rows: ignored
    assert c.rows == 4
    assert (c.cols[0].kind, c.cols[1].kind) == (INT64, DECIMAL)


def test_errc_names_mirror_reference():
    from paper_2508_05029_b200 import ops
    L = ops.lib()
    # reference proj/include/tierq/common.hpp:34-53 ordinal + 1
    assert L.tq_errc_name(11) == b"ReservationExceeded"
    assert L.tq_errc_name(16) == b"InvalidPlan"
    assert L.tq_errc_name(18) == b"Internal"


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_05029_b200 import ops
    from paper_2508_05029_b200.columnar import TqError
    with pytest.raises(TqError):
        ops.Context(0)


def test_product_does_not_reference_oracle():
    """The shipped package must not import, link or call oracle/."""
    pkg = os.path.join(ROOT, "paper_2508_05029_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "liboracle" not in src and "tqo_" not in src and "import oracle" not in src, f


BOUNDARY_TEST = os.path.join(ROOT, "oracle", "_ref", "boundary_test")


def test_cpp_boundary_binding_builds():
    """INTEGRATION.md §2-3's C++ binding compiles against the reference's own
    headers and links libtq_gpu.so (oracle/build_ref.sh)."""
    if not os.path.exists(BOUNDARY_TEST):
        pytest.skip("reference sources absent: oracle/_ref/boundary_test not built")
    out = subprocess.run(["ldd", BOUNDARY_TEST], capture_output=True, text=True).stdout
    assert "libtq_gpu.so" in out and "not found" not in out


@pytest.mark.gpu
def test_cpp_boundary_binding_runs():
    """reference ColumnBatch -> tq_batch -> tq_filter / tq_aggregate on the GPU
    -> ColumnBatch, equal to the reference's own take() / SPEC examples by the
    reference's operator==; statuses come back as tierq::Error{Errc}."""
    r = subprocess.run([BOUNDARY_TEST], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "boundary_test ok" in r.stdout
