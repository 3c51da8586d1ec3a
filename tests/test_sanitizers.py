"""SURVEY §5 aux: the host side of libpcr.so under AddressSanitizer + UndefinedBehaviorSanitizer.
The whole library is rebuilt with -fsanitize=address,undefined on the host compiler (device code is
unaffected; no GPU is needed) and a host-control-only context (device = -1, where the plan-table
arena is ordinary heap memory ASan watches) runs random traces through the C-ABI: submit / match
(with look-ahead windows) / store writes and reads / release, the SSD tier, and the context-split
tables at a geometry with zero rounding slack in the table region (region_words)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SAN = "-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer,-fno-sanitize-recover=undefined"

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2603_23049_b200.pcr as pcr
from pcrgen import make_rng
rng = make_rng(7)
C, S = 64, 16
for shard_mode, world, ssd in ((0, 1, 0), (1, 3, 0), (0, 1, 12), (1, 2, 12)):
    # max_tokens 816: 51 page + 13 chunk entries = 64 words -> 3 * 64 region words, no slack
    ctx = pcr.Context(2, 4, 2, 64, C, S, 10, 2, device=-1, pool_bytes=120 * 2 * 2 * 2 * S * 64 * 2,
                      rank=world - 1, world=world, shard_mode=shard_mode, max_inflight=1, max_tokens=816,
                      ssd_path="/tmp/pcr_asan_ssd.bin" if ssd else None, ssd_chunks=ssd)
    docs = [rng.integers(0, 50, C * int(rng.integers(1, 6)), dtype=np.uint32) for _ in range(6)]
    rec = np.zeros(ctx.slot_bytes // 2, np.uint16)
    for i in range(300):
        a, b = rng.choice(6, 2, replace=False)
        toks = np.concatenate([docs[a], docs[b], rng.integers(0, 50, int(rng.integers(1, 100)), dtype=np.uint32)])
        toks = toks[:816]
        ctx.submit(i, toks, n_cacheable=min(len(toks), len(docs[a]) + len(docs[b])))
        if i + 1 < 300:
            ctx.submit(10_000 + i, toks[::-1].copy())
        pend = [10_000 + j for j in range(max(0, i - 1), i + 1) if j + 1 < 300][:2]
        p = ctx.match_prefix(i, pend)
        for s_ in p["slots"][p["n_matched"]:]:
            rec[:] = i
            ctx.store_write(s_, rec)
            assert (ctx.store_read(s_) == i).all()
        ctx.release(i, bool(rng.integers(0, 2)))
    ctx.close()
print("ASAN-OK")
"""


@pytest.fixture(scope="module")
def asan_lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("asan")
    objs = []
    srcs = ["host/blake2b.cpp", "host/planner.cpp", "kernels/kv_copy.cu", "kernels/suffix_attn.cu",
            "runtime/nccl_dl.cpp", "runtime/ssd_io.cpp", "runtime/capi.cu"]
    csrc = os.path.join(ROOT, "paper_2603_23049_b200", "csrc")
    for src in srcs:
        o = str(out / (src.replace("/", "_") + ".o"))
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O1", "-g", "-std=c++17",
               "-Xcompiler", "-fPIC," + SAN, "-I" + os.path.join(ROOT, "include"),
               "-x", "cu" if src.endswith(".cu") else "c++", "-c", os.path.join(csrc, src), "-o", o]
        subprocess.run(cmd, check=True, capture_output=True, timeout=600)
        objs.append(o)
    lib = str(out / "libpcr_asan.so")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared",
                    "-Xcompiler", SAN, "-o", lib, *objs, "-lpthread", "-ldl"], check=True, capture_output=True,
                   timeout=600)
    return lib


def test_host_control_clean_under_asan_ubsan(asan_lib):
    rt = [subprocess.run(["gcc", f"-print-file-name={n}"], capture_output=True, text=True).stdout.strip()
          for n in ("libasan.so", "libubsan.so")]
    env = dict(os.environ, PCR_LIB_PATH=asan_lib, LD_PRELOAD=":".join(rt), CUDA_VISIBLE_DEVICES="",
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    res = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert res.returncode == 0 and "ASAN-OK" in res.stdout, (res.stdout[-2000:], res.stderr[-4000:])
