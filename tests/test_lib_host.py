"""libpcr.so on CPU (host-control-only contexts, no GPU): the library loads and exports every
symbol include/pcr.h declares; its BLAKE2b matches RFC 7693 vectors; its planner matches the
oracle bit-exactly (hits, slots, pages, eviction keys and order, leaf-list order, errors)."""
import os
import re

import numpy as np
import pytest

from oracle.tree import PlanError, PlanOracle
from pcrgen import appendix_c_trace, make_rng, random_tiny_trace

pcr = pytest.importorskip("paper_2603_23049_b200.pcr")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _host_ctx(C, S, store_chunks, n_pages, W, L=1, Hq=1, Hkv=1, d=8, max_inflight=8):
    page_bytes = L * Hkv * 2 * S * d * 2
    return pcr.Context(L, Hq, Hkv, d, C, S, store_chunks, W, device=-1, pool=None,
                       pool_bytes=n_pages * page_bytes, max_inflight=max_inflight)


def test_exports_every_declared_symbol():
    lib = pcr.load_library()
    hdr = open(os.path.join(ROOT, "include", "pcr.h")).read()
    declared = set(re.findall(r"\b(pcr_[a-z0-9_]+)\s*\(", hdr))
    assert {"pcr_match_prefix", "pcr_load_layer_kv", "pcr_prefill_attn_layer", "pcr_run_prefill"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert set(pcr.PROTOTYPES) == declared
    assert lib.pcr_abi_version() == 7


def test_blake2b_rfc7693_vectors():
    # RFC 7693 Appendix A: BLAKE2b-512("abc")
    assert pcr.blake2b(b"abc").hex() == (
        "ba80a53f981c4d0d6a2797b69f12f6e94c212f14685ac4b74b12bb6fdbffa2d1"
        "7d87c5392aab792dc252d5de4533cc9518d38aa8dbf1925ab92386edd4009923")
    # BLAKE2b-512("") and the keyed known-answer test (key 00..3f, empty message)
    assert pcr.blake2b(b"").hex() == (
        "786a02f742015903c6c6fd852552d272912f4740e15847618a86e217f71f5419"
        "d25e1031afee585313896444934eb04b903a685b1448b755d56f701afe9be2ce")
    assert pcr.blake2b(b"", key=bytes(range(64))).hex() == (
        "10ebb67700b1868efb4417987acf4690ae9d972fb7a590c2f02871799aaa4786"
        "b5e996e8f0f4eb981fc214b005f42d2ff4233499391653df7aefcbc13fc51568")
    # multi-block input crosses the 128-byte buffer boundary
    data = bytes(range(256)) * 3
    import hashlib
    for n in (0, 1, 127, 128, 129, 255, 256, 257, 768):
        assert pcr.blake2b(data[:n], 16) == hashlib.blake2b(data[:n], digest_size=16).digest()


def _both(C, S, cap, n_pages, W):
    return PlanOracle(C=C, S_pg=S, store_chunks=cap, n_pages=n_pages, window=W), _host_ctx(C, S, cap, n_pages, W)


def _cmp_plan(po, pl):
    for f in ("n_matched", "n_reserved", "n1", "n2", "slots", "pages"):
        assert po[f] == pl[f], (f, po[f], pl[f])
    assert po["evicted"] == pl["evicted"]


def _run_both(reqs, C, S, cap, n_pages, W, commit_pattern=None):
    o, lib = _both(C, S, cap, n_pages, W)
    for i, t in enumerate(reqs):
        o.submit(i, t)
        lib.submit(i, t)
    for i in range(len(reqs)):
        pend = list(range(i + 1, min(len(reqs), i + 1 + W + 1)))   # one extra: beyond-window ignored
        _cmp_plan(o.match_prefix(i, pend), lib.match_prefix(i, pend))
        assert o.leaf_list() == lib.leaf_list()
        commit = True if commit_pattern is None else bool(commit_pattern[i % len(commit_pattern)])
        o.release(i, commit)
        lib.release(i, commit)
        assert o.leaf_list() == lib.leaf_list()
    lib.close()


@pytest.mark.parametrize("W", [0, 2])
def test_appendix_c_parity(W):
    docs, order, reqs = appendix_c_trace(0)
    _run_both(reqs, 64, 16, 10, 1024, W)


def test_random_trace_parity():
    rng = make_rng(2024)
    for case in range(300):
        C = int(rng.integers(1, 5))
        S = [s for s in (1, 2, 4) if C % s == 0][int(rng.integers(0, 3)) % len([s for s in (1, 2, 4) if C % s == 0])]
        reqs = random_tiny_trace(rng, C=C, n_docs=6, max_doc_chunks=3, n_requests=12)
        cap = int(rng.integers(2, 10))
        W = int(rng.integers(0, 5))
        pattern = [None, [1, 0], [1, 1, 0]][case % 3]
        _run_both(reqs, C, S, cap, 4096, W, pattern)


def test_concurrent_plans_parity():
    """Several requests planned before any release (in flight together)."""
    rng = make_rng(77)
    for _ in range(50):
        reqs = random_tiny_trace(rng, C=2, n_docs=3, max_doc_chunks=2, n_requests=9)
        o, lib = _both(2, 2, 6, 4096, 2)
        for i, t in enumerate(reqs):
            o.submit(i, t)
            lib.submit(i, t)
        for b in range(0, 9, 3):
            for i in range(b, b + 3):
                pend = [j for j in range(i + 1, 9)][:2]
                _cmp_plan(o.match_prefix(i, pend), lib.match_prefix(i, pend))
            for i in range(b, b + 3):
                o.release(i, i % 2 == 0)
                lib.release(i, i % 2 == 0)
            assert o.leaf_list() == lib.leaf_list()
        lib.close()


def test_error_codes_match_oracle():
    o, lib = _both(4, 4, 4, 3, 2)
    toks = np.arange(9, dtype=np.uint32)

    def both(fn_o, fn_l):
        with pytest.raises(PlanError) as eo:
            fn_o()
        with pytest.raises(pcr.PcrError) as el:
            fn_l()
        assert eo.value.code == el.value.code

    both(lambda: o.match_prefix(5, []), lambda: lib.match_prefix(5, []))
    o.submit(0, toks)
    lib.submit(0, toks)
    both(lambda: o.submit(0, toks), lambda: lib.submit(0, toks))
    both(lambda: o.submit(1, toks, 10), lambda: lib.submit(1, toks, 10))
    both(lambda: o.match_prefix(0, [0]), lambda: lib.match_prefix(0, [0]))
    o.submit(1, toks)
    lib.submit(1, toks)
    both(lambda: o.match_prefix(0, [1, 1]), lambda: lib.match_prefix(0, [1, 1]))
    both(lambda: o.match_prefix(0, [7]), lambda: lib.match_prefix(0, [7]))
    both(lambda: o.release(0), lambda: lib.release(0))
    big = np.arange(13, dtype=np.uint32)
    o.submit(2, big)
    lib.submit(2, big)
    both(lambda: o.match_prefix(2, [0, 1]), lambda: lib.match_prefix(2, [0, 1]))
    _cmp_plan(o.match_prefix(0, [1, 2, 99]), lib.match_prefix(0, [1, 2, 99]))
    both(lambda: o.match_prefix(0, []), lambda: lib.match_prefix(0, []))
    lib.close()


def test_device_calls_rejected_on_host_ctx():
    lib = _host_ctx(4, 4, 4, 8, 0)
    lib.submit(0, np.arange(9, dtype=np.uint32))
    lib.match_prefix(0, [])
    with pytest.raises(pcr.PcrError) as e:
        lib.load_layer_kv(0, 0, None)
    assert e.value.code == "STATE"
    lib.close()


def test_store_roundtrip_host():
    lib = _host_ctx(8, 4, 3, 8, 0, L=2, Hq=4, Hkv=2, d=16)
    rec = np.arange(lib.slot_bytes // 2, dtype=np.uint16)
    lib.store_write(2, rec)
    assert np.array_equal(lib.store_read(2), rec)
    with pytest.raises(pcr.PcrError):
        lib.store_write(3, rec)
    lib.close()


def test_invalid_configs():
    with pytest.raises(pcr.PcrError) as e:
        pcr.Context(2, 3, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0)      # Hq % Hkv
    assert e.value.code == "INVAL"
    with pytest.raises(pcr.PcrError):
        pcr.Context(2, 4, 2, 64, 64, 48, 4, 0, device=-1, pool_bytes=0)     # S does not divide C
    with pytest.raises(pcr.PcrError):
        pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, rank=1, world=4)  # world !| Hkv
    with pytest.raises(pcr.PcrError):
        pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, load_mode=5)          # no such load path (0-4 since ABI v6)
    with pytest.raises(pcr.PcrError):
        pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, load_mode=4, load_ce_fraction=1.5)
    pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, load_mode=4, load_ce_fraction=0.5).close()
    with pytest.raises(pcr.PcrError):
        pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, shard_mode=2)         # no such sharding
    # context split: world need not divide Hkv, and every rank keeps all heads
    c = pcr.Context(2, 4, 2, 64, 64, 16, 4, 0, device=-1, pool_bytes=0, rank=3, world=4, shard_mode=1)
    assert c.slot_bytes == 2 * 2 * 2 * 64 * 64 * 2
    c.close()


def test_pcr_run_opts_layout_matches_header():
    """The binding's ctypes structs mirror include/pcr.h (ABI v7): field order and offsets that the
    C side reads (host_io / io_ring_layers in pcr_run_opts, load_ce_fraction in pcr_config)."""
    import ctypes
    assert [f for f, _ in pcr.PcrRunOpts._fields_][-5:] == ["mode", "host_io", "io_ring_layers", "partial_all",
                                                         "prefill_done_event"]
    assert pcr.PcrConfig.load_ce_fraction.offset == pcr.PcrConfig.load_mode.offset + 4
    assert pcr.PcrConfig.ssd_path.offset % ctypes.alignment(ctypes.c_void_p) == 0


def test_binding_struct_offsets_match_header(tmp_path):
    """Every field offset and struct size of the ctypes mirrors equals what a C compiler derives
    from include/pcr.h (gcc on the host): the binding cannot drift from the header."""
    import ctypes
    import os
    import shutil
    import subprocess
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    structs = {"pcr_config": pcr.PcrConfig, "pcr_plan": pcr.PcrPlan, "pcr_stats": pcr.PcrStats,
               "pcr_run_opts": pcr.PcrRunOpts}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "pcr.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "offsets.c"
    src.write_text("\n".join(lines))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "offsets"
    subprocess.run([gcc, "-std=c99", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        cls = structs[cname]
        got = ctypes.sizeof(cls) if field == "sizeof" else getattr(cls, field).offset
        assert got == int(val), (cname, field, got, val)
