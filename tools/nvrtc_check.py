"""Compile a (dumped) JIT source with NVRTC exactly as jit.cu does — runs on
the CPU build box, so codegen errors are caught without a GPU.

    python tools/nvrtc_check.py gpurun_out/jitdump/tq_jit_0.cu
    CUBIN_OUT=/tmp/k.cubin python tools/nvrtc_check.py x.cu && cuobjdump -sass /tmp/k.cubin
"""
import ctypes as C
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2508_05029_b200", "csrc")


def compile_src(src: str):
    L = C.CDLL("libnvrtc.so.12") if os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12") is False else \
        C.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
    prog = C.c_void_p()
    assert L.nvrtcCreateProgram(C.byref(prog), src.encode(), b"tq_jit.cu", 0, None, None) == 0
    opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"-DTQ_JIT=1", b"--device-int128",
            ("-I" + CSRC).encode(), ("-I" + os.path.join(ROOT, "include")).encode()]
    arr = (C.c_char_p * len(opts))(*opts)
    rc = L.nvrtcCompileProgram(prog, len(opts), arr)
    n = C.c_size_t()
    L.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    L.nvrtcGetProgramLog(prog, log)
    cubin = None
    if rc == 0:
        L.nvrtcGetCUBINSize(prog, C.byref(n))
        buf = C.create_string_buffer(n.value)
        L.nvrtcGetCUBIN(prog, buf)
        cubin = buf.raw
    return rc, log.value.decode(errors="replace"), cubin


if __name__ == "__main__":
    for path in sys.argv[1:]:
        src = open(path).read()
        src = re.sub(r"/\* NVRTC LOG:.*\*/\s*$", "", src, flags=re.S)
        rc, log, cubin = compile_src(src)
        if cubin and os.environ.get("CUBIN_OUT"):
            open(os.environ["CUBIN_OUT"], "wb").write(cubin)
        errs = [l for l in log.splitlines() if "error" in l]
        print(path, "rc", rc, "errors", len(errs))
        for l in errs[:10]:
            print("  ", l)
