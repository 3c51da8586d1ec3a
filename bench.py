"""bench.py — reuse-prefill throughput of the PCR hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload L8|M7|L70|T] [--ratio r]
                    [--mode overlap|sync] [--impl ours|reference]

One STEP = one RAG request through the whole hot path:
pcr_submit -> pcr_match_prefix (host plan, look-ahead LRU) -> pcr_run_prefill (per layer:
host->HBM gather of the cached prefix KV, suffix append, tcgen05 suffix attention; load(l+1)
overlapping attn(l) on two streams) -> pcr_release(commit).  Default workload = configs[1]
(L8: Llama-3-8B shape, 32 layers, 32/8 heads, d=128, 4 docs x 1k cached + 128-token query,
100% prefix hit, B=1).  value = context tokens (N1+N2) per second over K steps, whole job.

N > 1 (torchrun): KV heads are sharded across ranks (rank r owns heads [r*Hkv/N, (r+1)*Hkv/N),
its own store slice and host link); outputs are re-assembled by an NCCL all-gather.  The same
request is processed by all ranks, so per-GPU work shrinks with N: scaling = "strong".

--impl reference runs the fp64 CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import copy
import json
import socket
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (geometry preset, N1 docs tokens, query tokens)
    "L8": ("L8", 4096, 128),
    "M7": ("M7", 8192, 128),
    "L70": ("L70", 16384, 128),
    "T": ("T", 256, 64),
    "Z": ("L8", 0, 0),   # configs[4]: 1000-request Zipf trace (run_trace_z)
}


LOAD_MODES = {"sm": 0, "ce_runs": 1, "ce_blocks": 2, "tma": 3, "hybrid": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="L8", choices=list(WORKLOADS))
    ap.add_argument("--ratio", type=float, default=1.0, help="prefix hit ratio of the doc tokens (M7 sweep)")
    ap.add_argument("--mode", default="overlap", choices=["overlap", "sync", "only-up", "only-down"],
                    help="layer-wise overlap of loading (up) and, with --offload, offloading (down), P:703")
    ap.add_argument("--offload", action="store_true",
                    help="f1: offload the request's new cacheable chunks layer by layer on a third stream "
                         "(dropped at release so every step sees the same hit ratio)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0, help="CPU seconds for the oracle baseline sample")
    ap.add_argument("--no-target-point", action="store_true",
                    help="skip the M7 r=0.5 north_star sub-record of the default L8 line")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch-path check: bring up the ranks (gloo, no GPU), print them, exit")
    ap.add_argument("--gather-ctas", type=int, default=0, help="CTAs of the host->HBM gather (0 = library default)")
    ap.add_argument("--profile-steps", type=int, default=5, help="extra steps with per-layer events (after timing)")
    ap.add_argument("--window", type=int, default=4, help="look-ahead window W (Z trace)")
    ap.add_argument("--layer-body", action="store_true",
                    help="f3: stand-in layer body per layer (QKV / O projections + SwiGLU MLP GEMMs via "
                         "cuBLAS) around the attention, driven through the per-layer C-ABI calls")
    ap.add_argument("--store-frac", type=float, default=0.10, help="Z: DRAM store size / distinct chunks")
    ap.add_argument("--requests", type=int, default=1000, help="Z: requests in the trace")
    ap.add_argument("--rho-service-ms", type=float, default=0.0,
                    help="Z: service time (ms) that rho refers to (0 = this run's saturated-pass mean; set it "
                         "to compare configurations at the same arrival rate)")
    ap.add_argument("--no-reuse", action="store_true",
                    help="Z: nothing cacheable (every request recomputes its context: the no-PCR baseline)")
    ap.add_argument("--rho", default="", help="Z: comma list of loads (e.g. 0.5,0.8,0.95): extra passes with "
                                              "Poisson arrivals at rho x the measured service rate")
    ap.add_argument("--ssd-frac", type=float, default=0.0, help="Z: SSD tier size / distinct chunks (0 = none)")
    ap.add_argument("--ssd-path", default="/tmp/pcr_ssd_tier.bin", help="Z: SSD tier file")
    ap.add_argument("--z-windows", default="", help="Z sweep: comma list of look-ahead windows (one line per pass)")
    ap.add_argument("--z-store-fracs", default="", help="Z sweep: comma list of DRAM store fractions")
    ap.add_argument("--z-log", default="", help="Z: directory for per-pass plan logs (oracle replay)")
    ap.add_argument("--ce-frac", type=float, default=0.5, help="--load-mode hybrid: copy-engine share of the chunks")
    ap.add_argument("--shard", default="heads", choices=["heads", "context"],
                    help="how P GPUs (or --rank-slice P) split a request: KV heads (north_star) or the "
                         "context-split variant (chunk c -> rank c % P, partials merged)")
    ap.add_argument("--rank-slice", type=int, default=1,
                    help="single process doing the per-GPU work of rank 0 of a P-GPU KV-head-sharded run "
                         "(its head slice of the load and attention, no all-gather): a one-GPU estimate of "
                         "the per-rank critical path at P GPUs")
    ap.add_argument("--load-mode", default="sm", choices=list(LOAD_MODES),
                    help="a2 implementation: sm_100a 16-byte gather kernel (default), or the f4 baselines: "
                         "copy engines with one cudaMemcpyAsync per merged run (ce_runs) or per page image "
                         "(ce_blocks), TMA bulk copies, or the hybrid")
    return ap.parse_args()


def geometry(name):
    from pcrgen import PRESETS
    return PRESETS[name]


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML
    (nvidia-ml-py) polled every 10 ms from a thread, so even a sub-second timed region gets tens
    of samples; `nvidia-smi -lms 100` as the fallback."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index, pci_bus_id=None):
        self.index, self.pci = index, pci_bus_id
        self.proc = self.nvml = None
        self.lines, self.samples = [], []
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = (pynvml.nvmlDeviceGetHandleByPciBusId(self.pci) if self.pci
                 else pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self.nvml, self.h = pynvml, h
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                                          "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                                          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv = self.nvml
        while not self.stop_ev.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.samples.append((mhz, rs, time.perf_counter()))
            except Exception:
                pass
            self.stop_ev.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def begin(self):
        self.t_begin = time.perf_counter()

    def stop(self):
        if self.nvml:
            self.stop_ev.set()
            self.t.join(timeout=2)
            t0 = getattr(self, "t_begin", 0.0)
            inside = [(m, rs) for m, rs, ts in self.samples if ts >= t0]   # timed region only
            sm = [m for m, _ in inside]
            reasons = sorted({n for _, rs in inside for n, bit in self.REASONS if rs & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                    "samples": len(sm), "source": "nvml, 10 ms poll"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for (n, _), v in zip(self.REASONS, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 100"}


def pci_bus_id(torch, dev):
    try:
        pr = torch.cuda.get_device_properties(dev)
        return f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
    except Exception:
        return None


# ------------------------------------------------------------------------------ oracle leg
def oracle_sample(geo, N1, N2, hkv_loc, hq_loc, budget_s=15.0, seed=0, max_layers=None):
    """Time the oracle (as it stands) on a bounded sample of the workload: whole layers of
    load + append + fp64 suffix attention, until the budget is spent.  Returns
    (seconds per layer, layers sampled)."""
    from oracle.attention import bf16_bits_to_f64, suffix_attention_blocked
    from oracle.kvload import append_layer, load_layer
    from pcrgen import make_rng, randn_bf16
    rng = make_rng(seed)
    C, S, d = geo["C"], geo["S_pg"], geo["d"]
    N = N1 + N2
    n_chunks = N1 // C
    n_pages = -(-N // S)
    store = randn_bf16(rng, (n_chunks, 1, hkv_loc, 2, C, d))
    pool = np.zeros((1, n_pages, hkv_loc, 2, S, d), np.uint16)
    q = randn_bf16(rng, (N2, hq_loc, d))
    kn = randn_bf16(rng, (N2, hkv_loc, d))
    vn = randn_bf16(rng, (N2, hkv_loc, d))
    slots, pages = list(range(n_chunks)), list(range(n_pages))
    t0 = time.perf_counter()
    layers = 0
    while True:
        load_layer(pool, store, slots, pages, 0, N1, C, S)
        append_layer(pool, kn, vn, pages, 0, N1, S)
        kc = np.concatenate([store[c, 0, :, 0].transpose(1, 0, 2) for c in range(n_chunks)] + [kn]) if n_chunks else kn
        vc = np.concatenate([store[c, 0, :, 1].transpose(1, 0, 2) for c in range(n_chunks)] + [vn]) if n_chunks else vn
        suffix_attention_blocked(bf16_bits_to_f64(q), bf16_bits_to_f64(kc), bf16_bits_to_f64(vc), N1)
        layers += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_layers and layers >= max_layers) or layers >= geo["L"]:
            return el / layers, layers


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def metric_name(workload):
    return f"reuse-prefill tokens/s ({workload}: context tokens N1+N2 per second; TTFT in ttft_ms)"


def workload_config(args, geo, N1, N2, world=1, shard=1, ctx_split=False):
    """The `config` object both arms print (the workload, not the implementation)."""
    L, Hq, Hkv, d, C, S = geo["L"], geo["Hq"], geo["Hkv"], geo["d"], geo["C"], geo["S_pg"]
    load_bytes = 2 * N1 * (Hkv // shard) * d * 2
    if ctx_split:
        kind = "context split"
        return {"workload": f"{args.workload}: {L}L {Hq}/{Hkv} heads d={d}, N1={N1} cached (host DRAM) + "
                            f"N2={N2} computed, B=1, C={C}, S_pg={S}",
                "N1": N1, "N2": N2,
                "parallelism": f"{kind} x{world} (chunk c -> rank c % P, partials all-gathered and merged)"
                if world > 1 else f"rank 0 of a {kind} x{shard}, emulated on one GPU (its chunks' load, "
                                  f"attention of all rows to its keys, partial out; no all-gather/merge)",
                "l2": f"inputs > L2: {L * load_bytes / 2**20:.0f} MiB of prefix KV streamed from host per step"}
    return {"workload": f"{args.workload}: {L}L {Hq}/{Hkv} heads d={d}, N1={N1} cached (host DRAM) + "
                        f"N2={N2} computed, B=1, C={C}, S_pg={S}"
                        + (", +layer body (f3)" if getattr(args, "layer_body", False) else ""),
            "N1": N1, "N2": N2,
            "parallelism": f"kv-head shard x{world}" if world > 1 else (
                f"rank 0 of a kv-head shard x{shard}, emulated on one GPU (its head slice of load and "
                f"attention; no all-gather)" if shard > 1 else "single GPU"),
            "l2": f"inputs > L2: {L * load_bytes / 2**20:.0f} MiB of prefix KV streamed from host per step"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl_geo, n_doc, n_query = WORKLOADS[args.workload]
    geo = geometry(wl_geo)
    N1 = int(round(args.ratio * (n_doc // geo["C"]))) * geo["C"]
    N2 = n_doc - N1 + n_query
    per_step_budget = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(geo, N1, N2, geo["Hkv"], geo["Hq"], budget_s=0.0, max_layers=1)
    times = []
    for _ in range(args.steps):
        t_layer, _ = oracle_sample(geo, N1, N2, geo["Hkv"], geo["Hq"], budget_s=per_step_budget, max_layers=1)
        times.append(t_layer * geo["L"])
    t_step = statistics.mean(times)
    value = (N1 + N2) / t_step
    line = {
        "impl": "reference", "metric": metric_name(args.workload), "value": value,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, geo, N1, N2, world=max(1, args.gpus)),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": "1 of L layers per step (load + append + fp64 suffix attention, all heads), "
                                   "time x L"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def _hugepage_pinned(torch, nbytes, flags=0):
    """Anonymous mmap with MADV_HUGEPAGE, page-locked with cudaHostRegister: the same kind of host
    memory as the library's store (2 MiB pages: few IOMMU / GPU TLB translations per transfer).
    flags 3 = cudaHostRegisterMapped | Portable (device-readable, as host_io's gather reads it)."""
    import mmap
    huge = 2 << 20
    m = mmap.mmap(-1, nbytes + huge, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = np.frombuffer(m, dtype=np.uint8)
    off = (-base.ctypes.data) % huge          # a 2 MiB-aligned start: every 2 MiB range can be huge
    try:
        m.madvise(mmap.MADV_HUGEPAGE, off, nbytes)
    except Exception:
        pass
    a = base[off:off + nbytes]
    a[:] = 1
    t = torch.from_numpy(a)
    rc = torch._C._cudart.cudaHostRegister(t.data_ptr(), nbytes, flags)
    return (t, m) if int(rc) == 0 else (None, m)


def _anon_huge_frac(addrs):
    """Fraction of the given mappings' resident bytes on transparent huge pages (/proc/self/smaps):
    a diagnostic for the e2e host buffers (4 KiB pages read markedly slower from the GPU)."""
    try:
        size = huge = 0
        cur = None
        for line in open("/proc/self/smaps"):
            f = line.split()
            if "-" in f[0] and len(f) > 4 and ":" not in f[0]:
                lo, hi = (int(x, 16) for x in f[0].split("-"))
                cur = any(lo <= a < hi for a in addrs)
            elif cur and f[0] == "Rss:":
                size += int(f[1])
            elif cur and f[0] == "AnonHugePages:":
                huge += int(f[1])
        return huge / size if size else None
    except Exception:
        return None


def _host_buffer(torch, arr_or_shape, keep):
    """A page-locked host int16 tensor on hugepage-backed registered memory (falls back to torch's
    pinned allocator); `keep` collects the mappings to unregister later."""
    if isinstance(arr_or_shape, np.ndarray):
        shape, nbytes = arr_or_shape.shape, arr_or_shape.nbytes
    else:
        shape = tuple(arr_or_shape)
        nbytes = int(np.prod(shape)) * 2
    t, m = (None, None) if os.environ.get("PCR_BENCH_TORCH_PINNED") == "1" else _hugepage_pinned(torch, nbytes, flags=3)
    if t is None:
        out = torch.empty(shape, dtype=torch.int16).pin_memory()
    else:
        keep.append((t, m))
        out = t.view(torch.int16).view(shape)
    if isinstance(arr_or_shape, np.ndarray):
        out.copy_(torch.from_numpy(arr_or_shape.view(np.int16)))
    return out


def h2d_peak_gbs(torch, nbytes=256 << 20, reps=10):
    """Measured host->HBM copy-engine peak (the host-link roofline): best single 256 MiB
    cudaMemcpyAsync over `reps` tries from torch-pinned memory and from hugepage-backed registered
    memory (the store's kind); the larger is the link's demonstrated capability."""
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e9
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    hp, m = _hugepage_pinned(torch, nbytes)
    with torch.cuda.stream(s):
        for src in (h, hp):
            if src is None:
                continue
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                d.copy_(src, non_blocking=True)
                b.record(s)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
    if hp is not None:
        torch._C._cudart.cudaHostUnregister(hp.data_ptr())
    del h, hp, d
    try:
        m.close()
    except BufferError:
        pass
    return nbytes / (best * 1e-3) / 1e9


def measure(args, torch, dist, world, rank, local):
    """One workload (args.workload / args.ratio) through the hot path on this rank's GPU; returns
    the JSON line on rank 0 (None on the other ranks)."""
    from paper_2603_23049_b200 import MODE_SYNC, Context, comm_unique_id
    from pcrgen import make_rng, randn_bf16

    wl_geo, n_doc, n_query = WORKLOADS[args.workload]
    geo = geometry(wl_geo)
    L, Hq, Hkv, d, C, S = geo["L"], geo["Hq"], geo["Hkv"], geo["d"], geo["C"], geo["S_pg"]
    ctx_split = args.shard == "context"
    assert ctx_split or Hkv % world == 0, "KV-head sharding needs world | Hkv"
    shard = world
    if args.rank_slice > 1:
        assert world == 1 and (ctx_split or Hkv % args.rank_slice == 0), "--rank-slice P: one process, P | Hkv"
        shard = args.rank_slice
    hkv, hq = (Hkv, Hq) if ctx_split else (Hkv // shard, Hq // shard)
    N1 = int(round(args.ratio * (n_doc // C))) * C
    N = n_doc + n_query
    N2 = N - N1
    n_chunks = N1 // C
    # context split: this rank's chunks (depth c -> rank c % P) and whether it holds the suffix keys
    n_own = sum(1 for c in range(n_chunks) if c % shard == rank) if ctx_split else n_chunks
    suffix_here = (n_chunks % shard == rank) if ctx_split else True
    rng = make_rng(1000 + rank)

    # pool: room for 2 requests; store: the doc chunks (+ slack)
    pages_req = -(-N // S)
    n_pool_pages = 2 * pages_req + 8
    page_elems = L * hkv * 2 * S * d
    pool = torch.empty(n_pool_pages * page_elems, dtype=torch.int16, device="cuda")
    store_chunks = n_doc // C + 4
    load_mode = LOAD_MODES[args.load_mode]
    ctx = Context(L, Hq, Hkv, d, C, S, store_chunks, 4, device=local, pool=pool, rank=rank, world=shard,
                  gather_ctas=args.gather_ctas, load_mode=load_mode, load_ce_fraction=args.ce_frac,
                  shard_mode=1 if ctx_split else 0)

    # warm the DRAM store: commit a request whose first n_chunks chunks are the cached docs
    doc = make_rng(7).integers(0, 128256, n_doc, dtype=np.uint32)       # same tokens on every rank
    if n_chunks:
        ctx.submit(-1, np.concatenate([doc[:N1], [1]]).astype(np.uint32))
        warm = ctx.match_prefix(-1, [])
        assert warm["n_reserved"] == n_chunks
        # one N(0,1) record per 8 slots (rolled per slot): cheap to generate, finite bf16 values
        base = None
        for j, s in enumerate(warm["slots"]):
            if j % 8 == 0:
                base = randn_bf16(rng, (ctx.slot_bytes // 2,))
            ctx.store_write(s, np.roll(base, j))
        ctx.release(-1, True)
    query = make_rng(8).integers(0, 128256, n_query, dtype=np.uint32)
    toks = np.concatenate([doc, query])

    # suffix Q/K/V (device-resident for `value`; pinned host copies for `e2e`)
    def dev(a):
        return torch.from_numpy(a.view(np.int16)).cuda()
    q_h = randn_bf16(rng, (L, N2, hq, d))
    k_h = randn_bf16(rng, (L, N2, hkv, d))
    v_h = randn_bf16(rng, (L, N2, hkv, d))
    q_d, k_d, v_d = dev(q_h), dev(k_h), dev(v_h)
    out_d = torch.empty_like(q_d)
    # N > 1: the library re-assembles each layer's head-sharded output with an NCCL all-gather on
    # a comm stream, overlapped with the next layer (pcr_run_prefill_sharded)
    gathered, xs, lib_comm = None, None, False
    share_gpu = os.environ.get("PCR_BENCH_SHARE_GPU") == "1"   # functional N-rank check on one GPU
    part_d = None     # context split on one process: this rank's partials (the merge needs every rank)
    if ctx_split and world == 1:
        part_d = torch.empty((L, N2 * hq * (d + 1)), dtype=torch.float32, device="cuda")
    if world > 1:
        gathered = (torch.empty((L, world, N2 * hq * (d + 1)), dtype=torch.float32, device="cuda") if ctx_split else
                    torch.empty((L, world) + tuple(out_d.shape[1:]), dtype=out_d.dtype, device="cuda"))
        xs = torch.cuda.Stream()
        try:
            if share_gpu:
                raise RuntimeError("PCR_BENCH_SHARE_GPU: NCCL refuses two ranks on one GPU")
            uid = [comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.comm_init(uid[0])
            lib_comm = True
        except Exception as e:  # the same re-assembly through torch.distributed's NCCL, after the step
            print(f"rank {rank}: library NCCL communicator unavailable ({e}); using torch.distributed",
                  file=sys.stderr)
        ok = torch.tensor([1 if lib_comm else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        lib_comm = bool(ok.item())
    # the load stream gets the highest priority: its few gather CTAs are scheduled ahead of the
    # attention grid's CTAs whenever an SM slot frees up
    cs, ls = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    mode = {"overlap": 0, "sync": MODE_SYNC, "only-up": 2, "only-down": 3}[args.mode]
    os_ = torch.cuda.Stream() if args.offload else None
    assert not (args.offload and (world > 1 or args.layer_body)), "--offload: single GPU, no layer body"
    assert not (ctx_split and (args.layer_body or (world > 1 and not lib_comm))), \
        "--shard context: no layer body; N > 1 needs the library's NCCL communicator"
    req_counter = [0]
    match_us = []

    # f3 stand-in layer body: per layer, the suffix hidden state goes
    # through Wq/Wk/Wv projections (producing this layer's q, k_new, v_new), the PCR attention,
    # Wo and a SwiGLU MLP (Llama-3-8B widths, one random bf16 weight set shared by all layers).
    # The host->HBM load of layer l+1 runs on the load stream meanwhile.
    body = None
    if args.layer_body:
        assert world == 1, "--layer-body is single-GPU"
        dm, dff = 4096, 14336
        g = torch.Generator(device="cuda").manual_seed(5)
        wgt = lambda i, o: (torch.randn(i, o, device="cuda", generator=g, dtype=torch.bfloat16) / i ** 0.5)  # noqa: E731
        body = dict(wq=wgt(dm, hq * d), wk=wgt(dm, hkv * d), wv=wgt(dm, hkv * d), wo=wgt(hq * d, dm),
                    wg=wgt(dm, dff), wu=wgt(dm, dff), wd=wgt(dff, dm),
                    x=torch.randn(N2, dm, device="cuda", generator=g, dtype=torch.bfloat16))
        ev_ld = [torch.cuda.Event() for _ in range(L)]

    def run_with_layer_body(rid, out):
        b = body
        x = b["x"]
        ls.wait_stream(cs)
        for l in range(L):
            ctx.load_layer_kv(rid, l, ls)
            ev_ld[l].record(ls)
            with torch.cuda.stream(cs):
                qd = (x @ b["wq"]).view(N2, hq, d)
                kd = (x @ b["wk"]).view(N2, hkv, d)
                vd = (x @ b["wv"]).view(N2, hkv, d)
                cs.wait_event(ev_ld[l])
                ctx.prefill_attn_layer(rid, l, qd.view(torch.int16), kd.view(torch.int16), vd.view(torch.int16),
                                       out[l], cs)
                x = x + out[l].view(torch.bfloat16).view(N2, hq * d) @ b["wo"]
                x = x + (torch.nn.functional.silu(x @ b["wg"]) * (x @ b["wu"])) @ b["wd"]
        cs.wait_stream(ls)
        return None

    def step(q, k, v, out, times=False, load_events=None, step_mode=None, dev_events=None):
        """One request.  The caller's stream sync precedes pcr_release (pages are reused).
        dev_events: two events recorded on the compute stream just before the pipeline is enqueued
        and right after it (SURVEY 8(d) TTFT: the device pipeline, host planning reported apart)."""
        rid = req_counter[0]
        req_counter[0] += 1
        t0 = time.perf_counter()
        ctx.submit(rid, toks, n_cacheable=n_doc)
        plan = ctx.match_prefix(rid, [])
        match_us.append((time.perf_counter() - t0) * 1e6)
        assert plan["n1"] == N1, plan["n1"]
        if dev_events:
            dev_events[0].record(cs)
        if load_events:
            load_events[0].record(ls)
        if body is not None:
            t = run_with_layer_body(rid, out)
        elif world > 1 and lib_comm:
            t = ctx.run_prefill_sharded(rid, q, k, v, out, gathered, cs, ls, xs, mode=mode, layer_times=times)
        elif part_d is not None:
            t = ctx.run_prefill_ex(rid, q, k, v, None, cs, ls, offload_stream=os_, partial_all=part_d,
                                   mode=mode if step_mode is None else step_mode, layer_times=times)
        elif os_ is not None:
            t = ctx.run_prefill_ex(rid, q, k, v, out, cs, ls, offload_stream=os_,
                                   mode=mode if step_mode is None else step_mode, layer_times=times)
        else:
            t = ctx.run_prefill(rid, q, k, v, out, cs, ls, mode=mode if step_mode is None else step_mode,
                                layer_times=times)
            if world > 1 and not share_gpu:   # fallback re-assembly (rank-major [P][L][N2][Hq/P][d])
                with torch.cuda.stream(cs):
                    dist.all_gather_into_tensor(gathered.view(-1), out.view(-1))
        if load_events:
            load_events[1].record(ls)
        if dev_events:
            dev_events[1].record(cs)
        cs.synchronize()
        # The step is the hot path without the f1 offload (it would change the hit ratio from one
        # step to the next): newly reserved chunks are dropped, the cached prefix stays resident.
        # The full three-stream pipeline with commits is exercised by --workload Z.
        ctx.release(rid, False)
        return t

    if world > 1:
        dist.barrier()      # every rank measures its own host link at the same time: the concurrent peak
    peak_h2d_before = h2d_peak_gbs(torch)
    peaks_all = None
    if world > 1:
        peaks_all = [None] * world
        dist.all_gather_object(peaks_all, peak_h2d_before)
    for _ in range(args.warmup):
        step(q_d, k_d, v_d, out_d)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local, pci_bus_id(torch, local))
    clocks.start()
    launches0 = ctx.kernel_launches
    stats0 = ctx.stats
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clocks.begin()
    ev0.record(cs)
    ls.wait_event(ev0)
    step_ms, load_ms, dev_ms = [], [], []
    for _ in range(args.steps):
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l_a, l_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d_a, d_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record(cs)
        ls.wait_event(e_a)
        step(q_d, k_d, v_d, out_d, load_events=(l_a, l_b), dev_events=(d_a, d_b))
        e_b.record(cs)
        e_b.synchronize()
        step_ms.append(e_a.elapsed_time(e_b))
        load_ms.append(l_a.elapsed_time(l_b))
        dev_ms.append(d_a.elapsed_time(d_b))
    ev1.record(cs)
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    launches = ctx.kernel_launches - launches0
    if os.environ.get("PCR_BENCH_TIMELINE"):   # experiment (-DPCR_ATTN_TIMELINE=1 build): one more step's CTA timeline
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import ctypes
        from attn_timeline import read_tl, summarise
        lib = ctx.lib
        lib.pcr_debug_attn_timeline.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
        lib.pcr_debug_attn_timeline_clear()
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record(cs)
        ls.wait_event(e_a)
        step(q_d, k_d, v_d, out_d)
        e_b.record(cs)
        e_b.synchronize()
        print(json.dumps({"timeline_step_ms": e_a.elapsed_time(e_b)}), file=sys.stderr)
        summarise(read_tl(lib), L, "bench step")
    stats1 = ctx.stats
    ce_layers = stats1["ce_layer_loads"] - stats0["ce_layer_loads"]
    ce_copies_per_layer = (stats1["ce_copies"] - stats0["ce_copies"]) / max(1, ce_layers)
    clk = clocks.stop()
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        dist.barrier()

    # Per-kernel durations.  gather: inside a step the load stream runs the L gather launches
    # back to back (it never waits), so its busy time per step / L is the average launch
    # duration, measured over the timed steps with two events per step on that stream.
    # append+attention: per-layer events on the compute stream, in extra profiling steps.
    gather_ms = float(np.mean(load_ms)) / L
    if body is None:
        lt = np.array([step(q_d, k_d, v_d, out_d, times=True) for _ in range(max(1, args.profile_steps))])
        # layer 0's attention also waits for the first load (in-kernel with the streamed gather):
        # the in-pipeline attention time is the mean over layers 1..L-1
        attn_ms = float(lt[:, 1:, 1].mean()) if L > 1 else float(lt[:, :, 1].mean())
        gather_ms_evented = float(lt[:, :, 0].mean())
        offload_ms = float(lt[:, :, 2].mean()) if lt.shape[2] > 2 else None
        # the same kernels with nothing running beside them (SYNC order: gather, then attention)
        lt_iso, sync_ms = None, []
        if world == 1:
            lt_iso = []
            for _ in range(max(1, args.profile_steps)):
                e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_a.record(cs)
                lt_iso.append(step(q_d, k_d, v_d, out_d, times=True, step_mode=MODE_SYNC))
                e_b.record(cs)
                e_b.synchronize()
                sync_ms.append(e_a.elapsed_time(e_b))   # (includes the per-layer event reads)
            lt_iso = np.array(lt_iso)
        attn_ms_iso = float(lt_iso[:, :, 1].mean()) if lt_iso is not None else float("nan")
        gather_ms_iso = float(lt_iso[:, :, 0].mean()) if lt_iso is not None else float("nan")
        # the attention kernel's own speed: every layer's pcr_prefill_attn_layer back to back on the
        # compute stream (pool already loaded; PDL overlaps each launch with the one before, as in
        # the pipeline), nothing beside it -- the SYNC figures above also carry each launch's wait
        # for the gather before it
        attn_ms_b2b = float("nan")
        if part_d is None and os_ is None and not ctx_split:   # (each rank alone at P > 1: no collective)
            rid = req_counter[0]
            req_counter[0] += 1
            ctx.submit(rid, toks, n_cacheable=n_doc)
            ctx.match_prefix(rid, [])
            for l in range(L):
                ctx.load_layer_kv(rid, l, ls)
            ls.synchronize()
            reps = max(1, min(20, int(200 / max(1e-3, L * attn_ms_iso))))
            e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for rep in range(reps + 1):
                if rep == 1:
                    e_a.record(cs)
                for l in range(L):
                    ctx.prefill_attn_layer(rid, l, q_d[l], k_d[l], v_d[l], out_d[l], cs)
            e_b.record(cs)
            e_b.synchronize()
            attn_ms_b2b = e_a.elapsed_time(e_b) / (reps * L)
            ctx.release(rid, False)
    else:   # per-layer events are not recorded on the layer-body path
        attn_ms = gather_ms_evented = attn_ms_iso = gather_ms_iso = attn_ms_b2b = float("nan")
        sync_ms = []
        offload_ms = None

    sm_leg = None
    # e2e: the same step through the C-ABI with HOST buffers: q/k/v/out are page-locked host
    # tensors handed to pcr_run_prefill_ex(host_io=1); the library stages each layer's inputs
    # (H2D) and returns its output (D2H) on its own copy streams, overlapped with the pipeline.
    e2e = None
    if not args.no_e2e and part_d is None:   # (one rank of a context split has no whole output)
        # page-locked host buffers on hugepage-backed registered memory (2 MiB pages, like the store;
        # torch's 4 KiB pinned pages read slower from the GPU side)
        host_keep = []
        q_p = _host_buffer(torch, q_h, host_keep)
        k_p = _host_buffer(torch, k_h, host_keep)
        v_p = _host_buffer(torch, v_h, host_keep)
        res = gathered if world > 1 else None   # the step's result: full (re-assembled) output
        o_p = _host_buffer(torch, tuple(res.shape) if res is not None else tuple(q_p.shape), host_keep)
        host_io = world == 1 and body is None
        if not host_io:   # multi-rank / layer-body paths: copies around the device-buffer call
            q2, k2, v2, o2 = (torch.empty_like(q_d), torch.empty_like(k_d), torch.empty_like(v_d),
                              torch.empty_like(out_d))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(3, min(args.steps, 20))
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_e2e + 1)]
        # one untimed step first: the library allocates its host_io staging ring and D2H stream on
        # the first host_io call, and the host buffers' first device access maps them
        for i_e in range(-1, n_e2e):
            if i_e == 0:
                a.record(cs)
            if i_e >= 0:
                step_ev[i_e].record(cs)
            if host_io:
                rid = req_counter[0]
                req_counter[0] += 1
                ctx.submit(rid, toks, n_cacheable=n_doc)
                ctx.match_prefix(rid, [])
                ctx.run_prefill_ex(rid, q_p, k_p, v_p, o_p, cs, ls, mode=mode, host_io=True)
                cs.synchronize()
                ctx.release(rid, False)
                continue
            with torch.cuda.stream(cs):
                q2.copy_(q_p, non_blocking=True)
                k2.copy_(k_p, non_blocking=True)
                v2.copy_(v_p, non_blocking=True)
            ls.wait_stream(cs)
            step(q2, k2, v2, o2)
            with torch.cuda.stream(cs):
                o_p.copy_(res if res is not None else o2, non_blocking=True)
            cs.synchronize()
        step_ev[n_e2e].record(cs)
        b.record(cs)
        b.synchronize()
        e2e_ms = a.elapsed_time(b)
        e2e_steps = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(n_e2e)]
        if world > 1:
            tt = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        h2d_b, d2h_b = int(q_p.nbytes + k_p.nbytes + v_p.nbytes), int(o_p.nbytes)
        huge_frac = _anon_huge_frac([t_.data_ptr() for t_, _ in host_keep])
        del q_p, k_p, v_p, o_p
        for t_, _ in host_keep:
            torch._C._cudart.cudaHostUnregister(t_.data_ptr())
        e2e = {"value": n_e2e * N / (e2e_ms * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "steps": n_e2e,
               "host_hugepage_frac": huge_frac,
               "step_ms": {"median": statistics.median(e2e_steps), "min": min(e2e_steps), "max": max(e2e_steps),
                           "argmax": int(np.argmax(e2e_steps))},
               "path": "pcr_run_prefill_ex(host_io=1): each layer's q/k/v read by its gather launch from "
                       "page-locked (hugepage-registered) host buffers, its output returned by one cudaMemcpyAsync "
                       "on the library's D2H stream" if host_io
                       else "pinned-host copies around pcr_run_prefill (device buffers)"}

    n1_here = n_own * C                             # keys this rank loads (context split: its chunks)
    load_bytes = 2 * n1_here * hkv * d * 2          # algorithmic bytes per gather launch (one layer)
    attn_flops = 4 * hq * d * (N2 * n1_here + (N2 * (N2 + 1) // 2 if suffix_here else 0))
    peak_h2d_after = h2d_peak_gbs(torch)
    peak_h2d = max(peak_h2d_before, peak_h2d_after)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16_peak = peaks.get("bf16_tflops", 1590.0)
    bf16_src = "MEASURED_PEAKS.json bf16_tflops (burst)" if "bf16_tflops" in peaks else "fallback 1590 (B200_PROFILING.md)"
    gather_gbs = load_bytes / (gather_ms * 1e-3) / 1e9 if N1 else 0.0
    attn_tflops = attn_flops / (attn_ms * 1e-3) / 1e12 if attn_ms == attn_ms else None
    # two in-order streams, identical layers: T* = t_ld + (L-1) max(t_ld, t_at) + t_at
    ttft_pred = gather_ms + (L - 1) * max(gather_ms, attn_ms) + attn_ms if attn_tflops else None
    value = args.steps * N / (total_ms * 1e-3)
    # T*: the pipelined bound with every load and attention at its roofline
    t_ld_r = load_bytes / (peak_h2d * 1e9) * 1e3
    t_at_r = attn_flops / (bf16_peak * 1e12) * 1e3
    t_star = t_ld_r + (L - 1) * max(t_ld_r, t_at_r) + t_at_r if (t_ld_r + t_at_r) > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t_layer, n_l = oracle_sample(geo, n1_here, N2, hkv, hq, budget_s=args.cpu_budget_s)
        cpu = {"value": N / (t_layer * L), "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"{n_l} of {L} layers (pool load + append + fp64 suffix attention over all heads), "
                         f"extrapolated x{L}/{n_l}"}
    if rank != 0:
        ctx.close()
        return None
    # the dominant kernel by its own speed: in a load-bound pipeline the attention's in-pipeline time
    # includes its wait for the load (~ the load's pace), so it cannot decide
    attn_own = next((x for x in (attn_ms_b2b, attn_ms_iso, attn_ms) if x == x), float("nan"))
    dominant = "kv_gather" if N1 and (attn_own != attn_own or gather_ms >= attn_own) else "suffix_attn"
    # per-launch traffic of the dominant kernels from the committed ncu capture (profiles/)
    try:
        ncu_t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        ncu_t = {}
    if ce_layers:
        load_kernel = (f"kv_load on the copy engines (f4 baseline, load_mode {args.load_mode}): "
                       f"{ce_copies_per_layer:.0f} cudaMemcpyAsync per layer of "
                       f"{load_bytes / ce_copies_per_layer / 2**10:.0f} KiB")
    else:
        load_kernel = {4: f"kv_gather + copy engines ({args.ce_frac:.2f} of the chunks)", 3: "kv_gather_tma"}.get(
            load_mode, "kv_gather")
    # the streamed gather (one launch per request: OVERLAP loads, SM gather, head sharding) or one
    # kv_gather launch per layer; "per launch" below = per layer either way (streamed: its time / L)
    streamed = (load_mode == 0 and args.mode in ("overlap", "only-up") and not ctx_split and body is None
                and os.environ.get("PCR_STREAM_GATHER", "1") != "0")
    tr = ncu_t.get("gather_stream" if streamed else "gather", {}) if args.workload == "L8" and not ce_layers \
        and shard == 1 else {}
    per = L if streamed else 1
    rl_gather = {"bound": "host-link", "kernel": load_kernel + (" (streamed: one launch per request)" if streamed
                                                                 else ""),
                 "achieved": gather_gbs, "peak": peak_h2d, "unit": "GB/s", "frac": gather_gbs / peak_h2d,
                 "traffic": tr["dram_bytes"] / per if tr else None,
                 "traffic_pcie_read": tr["pcie_read_bytes"] / per if tr else None,
                 "traffic_note": "per layer, from the committed ncu --set full capture of this build "
                                 "(profiles/ncu_traffic.json): DRAM read+write bytes (the pool writes) and PCIe read "
                                 "bytes (incl. protocol; 1.094 x algorithmic: 128-byte read completions)",
                 "peak_source": f"live: cudaMemcpyAsync H2D, 256 MiB, best of 10 from torch-pinned and from "
                                f"hugepage-backed registered memory, max of a "
                                f"measurement before the warm-up ({peak_h2d_before:.1f}) and after the timed region "
                                f"({peak_h2d_after:.1f})",
                 "sm_read_ceiling_note": "SM-originated host reads top out at 51.1-51.5 GB/s on this link for every "
                                         "load width / TMA variant (tools/h2d_probe2.cu): 0.92 of the copy engine",
                 "algorithmic_bytes_per_launch": load_bytes, "avg_launch_ms": gather_ms}
    rl_sm = None
    if sm_leg is not None:
        sm_gbs = load_bytes / (sm_leg["avg_launch_ms"] * 1e-3) / 1e9
        rl_sm = {"bound": "host-link", "kernel": "kv_gather (sm_100a 16-byte gather kernel, load_mode sm)",
                 "achieved": sm_gbs, "peak": peak_h2d, "unit": "GB/s", "frac": sm_gbs / peak_h2d,
                 "traffic": ncu_t.get("gather", {}).get("pcie_read_bytes") if args.workload == "L8" else None,
                 "algorithmic_bytes_per_launch": load_bytes, "avg_launch_ms": sm_leg["avg_launch_ms"],
                 "ttft_ms": sm_leg["ttft_ms"], "steps": sm_leg["steps"],
                 "note": "the same steps re-timed with the SM gather kernel after the timed region"}
    rl_attn = None if attn_tflops is None else {
        "bound": "tensor", "kernel": "suffix_attn (suffix append fused; + split-KV combine at short suffixes)",
        "pipeline_regime": ("load-bound: achieved here is the load's pace; the kernel's own speed is 'isolated'"
                            if N1 and attn_ms_iso == attn_ms_iso and gather_ms >= min(attn_ms_iso, attn_ms_b2b)
                            else "attention-bound"),
        "achieved": attn_tflops, "peak": bf16_peak,
        "unit": "TFLOP/s", "frac": attn_tflops / bf16_peak,
        "frac_of_sustained": attn_tflops / peaks["bf16_tflops_sustained"] if "bf16_tflops_sustained" in peaks else None,
        "sustained_note": "MEASURED_PEAKS bf16_tflops_sustained (cuBLAS back to back for 4 s, SM clock ~1.26 GHz "
                          "under its power draw) -- the task's peak for a kernel inside a long step; frac uses the "
                          "burst figure because this kernel ran at the clocks in 'clocks', not at 1.26 GHz",
        "traffic": ncu_t.get("attn_M7_r05", {}).get("dram_bytes") if (args.workload, args.ratio, shard) == ("M7", 0.5, 1)
        else None,
        "peak_source": bf16_src,
        "algorithmic_flops_per_launch": attn_flops, "avg_launch_ms": attn_ms,
        "note": "attention (suffix append fused) per layer as it runs in the pipeline, layers 1..L-1: beside "
                "the gather in OVERLAP mode; with the streamed gather each attention first waits in-kernel for "
                "its layer's load, so in a load-bound workload (L8) this is the load's pace, not the kernel's; "
                "isolated = the kernel's own speed: every layer's attention launched back to back with nothing "
                "beside it (pool loaded beforehand); isolated_sync = the same launches in SYNC order, each one "
                "also waiting for the gather launch before it",
        "isolated": None if attn_ms_b2b != attn_ms_b2b else {
            "avg_launch_ms": attn_ms_b2b, "achieved": attn_flops / (attn_ms_b2b * 1e-3) / 1e12,
            "frac": attn_flops / (attn_ms_b2b * 1e-3) / 1e12 / bf16_peak},
        "isolated_sync": None if attn_ms_iso != attn_ms_iso else {
            "avg_launch_ms": attn_ms_iso, "achieved": attn_flops / (attn_ms_iso * 1e-3) / 1e12,
            "frac": attn_flops / (attn_ms_iso * 1e-3) / 1e12 / bf16_peak}}
    line = {
        "metric": metric_name(args.workload),
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) bf16 KV/Q, random token ids)",
        "config": workload_config(args, geo, N1, N2, world=world, shard=shard, ctx_split=ctx_split),
        "pipeline": {"mode": args.mode, "load_mode": args.load_mode, "offload": bool(args.offload)},
        "offload_ms_per_layer": offload_ms,
        "offload_bytes_per_layer": (2 * (n_doc - N1) * hkv * d * 2) if args.offload else None,
        "suffix_tokens_per_s": N2 / (statistics.median(step_ms) * 1e-3),
        # SURVEY §8(d) derived overlap metrics (SYNC = every op in order on one stream)
        "overlap": None if not sync_ms else {
            "sync_ttft_ms": statistics.median(sync_ms),
            "hidden_load_pct": 100 * (statistics.median(sync_ms) - statistics.median(step_ms)) / (L * gather_ms_iso)
            if N1 else None,
            "exposed_load_ms": statistics.median(step_ms) - L * attn_ms_iso,
            "contention_attn": attn_ms / attn_ms_iso,
            "note": "hidden load % = (SYNC - OVERLAP) / sum of isolated loads (SURVEY 8(d)); it can exceed 100 "
                    "because SYNC's attention launches (each after a gather, no PDL overlap) are slower than "
                    "OVERLAP's; exposed = OVERLAP - sum of SYNC-isolated append+attention; contention = "
                    "append+attention time beside the loads / SYNC-isolated"},
        "ttft_ms": statistics.median(step_ms), "ttft_ms_p90": float(np.percentile(step_ms, 90)),
        "ttft_device_ms": statistics.median(dev_ms), "ttft_device_ms_p90": float(np.percentile(dev_ms, 90)),
        "ttft_note": "ttft_ms = the whole step on the device clock: host pcr_submit + pcr_match_prefix "
                     "(match_prefix_us), the pipeline, the host's stream sync and pcr_release; ttft_device_ms "
                     "= SURVEY 8(d)'s TTFT: from just before the pipeline is enqueued to the end of the last "
                     "layer's attention (incl. the re-assembly at P > 1)",
        "ttft_device_over_t_star": statistics.median(dev_ms) / t_star if t_star else None,
        "ttft_pred_ms": ttft_pred, "sync_bound_ms": L * (gather_ms + attn_ms) if attn_tflops else None,
        "gather_ms_per_layer": gather_ms,
        "gather_ms_per_layer_evented": gather_ms_evented if attn_tflops else None,
        "attn_ms_per_layer": attn_ms if attn_tflops else None, "gather_ctas": args.gather_ctas or 8,
        "match_prefix_us": statistics.median(match_us),
        "gpu_launches": launches,
        "roofline": rl_gather if dominant == "kv_gather" else rl_attn,
        "roofline_gather": rl_gather,
        "roofline_attn": rl_attn,
        "t_star_ms": t_star, "ttft_over_t_star": statistics.median(step_ms) / t_star if t_star else None,
        "h2d_peak_concurrent_gbs": None if peaks_all is None else {
            "per_rank": peaks_all, "aggregate": float(sum(peaks_all)),
            "note": "each rank's cudaMemcpyAsync H2D peak, all ranks measuring at once after a barrier"},
        "roofline_gather_sm": rl_sm,
        "load_path": {"ce_layer_loads": ce_layers, "sm_layer_loads": stats1["sm_layer_loads"] - stats0["sm_layer_loads"],
                      "ce_copies_per_layer": ce_copies_per_layer if ce_layers else 0},
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    ctx.close()
    return line


def north_star_point(m7):
    """The north_star target point as a sub-record of the default line: M7 at r = 0.5,
    the SM gather sharing the GPU with the attention (OVERLAP)."""
    rg, ra = m7["roofline_gather"], m7["roofline_attn"]
    ov = m7.get("overlap") or {}
    return {"workload": m7["config"]["workload"], "ttft_ms": m7["ttft_ms"], "ttft_device_ms": m7.get("ttft_device_ms"),
            "load_gbs": rg["achieved"], "load_frac_of_h2d_peak": rg["frac"], "h2d_peak_gbs": rg["peak"],
            "attn_tflops_in_pipeline": ra["achieved"] if ra else None,
            "attn_frac_of_bf16_peak": ra["frac"] if ra else None, "bf16_peak_tflops": ra["peak"] if ra else None,
            "attn_frac_alone": (ra.get("isolated") or {}).get("frac") if ra else None,
            "attn_frac_of_bf16_sustained": ra.get("frac_of_sustained") if ra else None,
            "hidden_load_pct": ov.get("hidden_load_pct"), "t_star_ms": m7["t_star_ms"],
            "ttft_over_t_star": m7["ttft_over_t_star"], "clocks": m7["clocks"],
            "targets": {"load_frac": 0.8, "attn_frac": 0.5, "hidden_load_pct": 100.0},
            "note": "north_star: per-layer reused-KV load >= 80% of the measured host->HBM peak, fully hidden behind "
                    "suffix attention at >= 50% of bf16 tensor peak; T* = the pipelined bound with every load and "
                    "attention at its roofline (SURVEY §8(d))"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:   # launch-path check on CPU (tests): gloo, report the ranks that came up
        if world > 1:
            dist.init_process_group("gloo")
        ranks = [None] * world
        if world > 1:
            dist.all_gather_object(ranks, {"rank": rank, "local_rank": local, "pid": os.getpid()})
        else:
            ranks = [{"rank": 0, "local_rank": 0, "pid": os.getpid()}]
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    share_gpu = os.environ.get("PCR_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        # functional check of the N-rank path with every rank on GPU 0 (timings meaningless; NCCL
        # refuses two ranks on one device, so gloo carries the control collectives and the outputs
        # are not re-assembled)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = measure(args, torch, dist, world, rank, local)
    if (args.workload == "L8" and not args.no_target_point and args.rank_slice == 1 and args.shard == "heads"
            and not args.layer_body and not args.offload):
        sub = copy.copy(args)
        sub.workload, sub.ratio = "M7", 0.5
        sub.steps, sub.warmup, sub.profile_steps = max(5, min(args.steps, 10)), 3, 3
        sub.no_e2e = sub.no_cpu_baseline = True
        m7 = measure(sub, torch, dist, world, rank, local)
        if rank == 0:
            line["north_star_point"] = north_star_point(m7)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def poisson_arrivals(n, rho, service_ms, seed=5):
    """Arrival times (ms) of a Poisson process at rho x the measured service rate
    (SURVEY 8(d) preset Z: rho in {0.5, 0.8, 0.95})."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.cumsum(rng.exponential(service_ms / rho, n))


class VirtualQueue:
    """FIFO single server in virtual time over measured service times: request i starts at
    max(arrival_i, finish_{i-1}); its look-ahead window (Alg. 1, pending[:W]) holds the
    next W requests that have ARRIVED by then, so the window only helps when a queue forms."""

    def __init__(self, arrivals, window):
        self.a = np.asarray(arrivals, dtype=np.float64)
        self.w = window
        self.t = 0.0

    def start(self, i):
        self.t = max(self.t, float(self.a[i]))
        j = i + 1
        while j < min(len(self.a), i + 1 + self.w) and self.a[j] <= self.t:
            j += 1
        return list(range(i + 1, j))

    def finish(self, i, service_ms):
        self.t += service_ms
        return self.t - float(self.a[i])   # queueing + service


def _z_layer_body(torch, geo, max_n):
    """f3 stand-in layer body for the Z trace (same shapes as run_ours --layer-body)."""
    dm, dff = 4096, 14336
    hq, hkv, d = geo["Hq"], geo["Hkv"], geo["d"]
    g = torch.Generator(device="cuda").manual_seed(5)
    wgt = lambda i, o: (torch.randn(i, o, device="cuda", generator=g, dtype=torch.bfloat16) / i ** 0.5)  # noqa: E731
    return dict(wq=wgt(dm, hq * d), wk=wgt(dm, hkv * d), wv=wgt(dm, hkv * d), wo=wgt(hq * d, dm),
                wg=wgt(dm, dff), wu=wgt(dm, dff), wd=wgt(dff, dm),
                x=torch.randn(max_n, dm, device="cuda", generator=g, dtype=torch.bfloat16),
                ev_ld=[torch.cuda.Event() for _ in range(geo["L"])],
                ev_at=[torch.cuda.Event() for _ in range(geo["L"])])


def _z_request_with_body(torch, ctx, rid, n2, geo, body, out, cs, ls, os_, done=None):
    """One request through the per-layer C-ABI calls with the layer body around the attention:
    load(l) on ls || QKV projection on cs; attention(l); offload(l) on os_ || O projection + MLP.
    Only the N2 computed tokens go through the GEMMs (the reused prefix needs no hidden states)."""
    L, hq, hkv, d = geo["L"], geo["Hq"], geo["Hkv"], geo["d"]
    b = body
    x = b["x"][:n2]
    ls.wait_stream(cs)
    os_.wait_stream(cs)
    for l in range(L):
        ctx.load_layer_kv(rid, l, ls)
        b["ev_ld"][l].record(ls)
        with torch.cuda.stream(cs):
            qd = (x @ b["wq"]).view(n2, hq, d)
            kd = (x @ b["wk"]).view(n2, hkv, d)
            vd = (x @ b["wv"]).view(n2, hkv, d)
            cs.wait_event(b["ev_ld"][l])
            ctx.prefill_attn_layer(rid, l, qd.view(torch.int16), kd.view(torch.int16), vd.view(torch.int16),
                                   out[l], cs)
            b["ev_at"][l].record(cs)
            os_.wait_event(b["ev_at"][l])
            ctx.offload_layer_kv(rid, l, os_)
            x = x + out[l].view(torch.bfloat16).view(n2, hq * d) @ b["wo"]
            x = x + (torch.nn.functional.silu(x @ b["wg"]) * (x @ b["wu"])) @ b["wd"]
    if done is not None:
        done.record(cs)     # prefill complete (the last offloads may still run)
    cs.wait_stream(ls)
    cs.wait_stream(os_)


def _z_pass(args, torch, reqs, ndoc, cap, ssd_chunks, pool, bufs, queue=None, body=None, window=None):
    """One pass of the Z trace on a fresh Context (cold store).  queue=None: every request is
    waiting from the start (saturated queue, pending = next W); else a VirtualQueue.
    body: the f3 layer body around the attention (per-layer calls); args.no_reuse: nothing is
    cacheable (every request recomputes its whole context: the no-PCR baseline).
    --rank-slice P: the per-GPU work of rank 0 of a P-GPU KV-head-sharded run (its head slice of
    every chunk; the host decisions are the same on every rank).  Every pcr_match_prefix input
    (pending ids) and its decisions are logged in r["log"] for the oracle replay."""
    from paper_2603_23049_b200 import MODE_OVERLAP, Context
    geo = geometry("L8")
    L, Hq, Hkv, d, C, S = geo["L"], geo["Hq"], geo["Hkv"], geo["d"], geo["C"], geo["S_pg"]
    P = max(1, args.rank_slice)
    hq, hkv = Hq // P, Hkv // P
    W = args.window if window is None else window
    max_n = max(len(r) for r in reqs)
    t0 = time.perf_counter()
    ctx = Context(L, Hq, Hkv, d, C, S, cap, W, device=0, pool=pool, max_tokens=max_n, rank=0, world=P,
                  gather_ctas=args.gather_ctas, ssd_path=args.ssd_path if ssd_chunks else None,
                  ssd_chunks=ssd_chunks, load_mode=LOAD_MODES[args.load_mode], load_ce_fraction=args.ce_frac)
    t_pin = time.perf_counter() - t0
    q_d, k_d, v_d, o_d = bufs
    cs, ls, os_ = torch.cuda.Stream(), torch.cuda.Stream(priority=-1), torch.cuda.Stream()
    for i, (t, n) in enumerate(zip(reqs, ndoc)):
        ctx.submit(i, t, 0 if args.no_reuse else n)
    r = {"ttft": [], "step": [], "wall": [], "ttft_q": [], "pending": [], "hits": 0, "chunks": 0, "toks": 0,
         "n1s": [], "plan_us": [], "t_pin": t_pin, "log": []}
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(cs)
    for i in range(len(reqs)):
        pend = queue.start(i) if queue else list(range(i + 1, min(len(reqs), i + 1 + W)))
        r["pending"].append(len(pend))
        tp = time.perf_counter()
        plan = ctx.match_prefix(i, pend)
        r["plan_us"].append((time.perf_counter() - tp) * 1e6)
        r["log"].append({"i": i, "pend": pend, "nm": plan["n_matched"], "nr": plan["n_reserved"],
                         "slots": plan["slots"], "ev": [s_ for _, s_ in plan["evicted"]], "ssd": plan["n_from_ssd"]})
        n2 = plan["n2"]
        # contiguous [L][N2][H][d] views over the front of the max-size buffers
        q = q_d.view(-1)[: L * n2 * hq * d].view(L, n2, hq, d)
        k = k_d.view(-1)[: L * n2 * hkv * d].view(L, n2, hkv, d)
        v = v_d.view(-1)[: L * n2 * hkv * d].view(L, n2, hkv, d)
        o = o_d.view(-1)[: L * n2 * hq * d].view(L, n2, hq, d)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        done = torch.cuda.Event(enable_timing=True)
        done.record(cs)      # (creates the event; the library records it again)
        a.record(cs)
        ls.wait_event(a)
        os_.wait_event(a)
        if body is not None:
            _z_request_with_body(torch, ctx, i, n2, geometry("L8"), body, o, cs, ls, os_, done=done)
        else:
            ctx.run_prefill_ex(i, q, k, v, o, cs, ls, offload_stream=os_, mode=MODE_OVERLAP, prefill_done_event=done)
        b.record(cs)
        b.synchronize()
        r["ttft"].append(a.elapsed_time(done))     # prefill complete: the request's first token
        r["step"].append(a.elapsed_time(b))        # + the tail of its layer-wise offload
        r["wall"].append((time.perf_counter() - tp) * 1e3)   # host plan (+ on-demand SSD loads) + GPU
        ctx.release(i, True)
        if queue:
            r["ttft_q"].append(queue.finish(i, r["wall"][-1]))
        r["hits"] += plan["n_matched"]
        r["chunks"] += ndoc[i] // C
        r["toks"] += len(reqs[i])
        r["n1s"].append(plan["n1"])
    ev1.record(cs)
    torch.cuda.synchronize()
    r["total_ms"] = ev0.elapsed_time(ev1)
    r["launches"] = ctx.kernel_launches - launches0
    r["stats"] = ctx.stats
    ctx.close()
    return r


def _write_plan_log(path, header, log):
    """gzip JSON lines: the pass header, then one record per pcr_match_prefix call (its inputs and
    decisions) -- replayed through the oracle by tests/test_z_replay.py."""
    import gzip
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with gzip.open(path, "wt") as f:
        f.write(json.dumps(header) + "\n")
        for rec in log:
            f.write(json.dumps(rec, separators=(",", ":")) + "\n")


def run_trace_z(args):
    """configs[4]: the Zipf RAG trace end to end on one GPU (look-ahead LRU + layer overlap +
    layer-wise offload of new chunks on a third stream, committed at release).  One step = one
    request; value = trace context tokens / device time; TTFT per request from CUDA events.
    --rho r1,r2,...: after the saturated pass (which measures the mean service time), one more
    pass per rho with Poisson arrivals at rho x that service rate (virtual-time FIFO queue; TTFT
    then includes queueing).  --z-windows / --z-store-fracs: a sweep, one JSON line per pass
    (SURVEY §8(d) preset Z: W in {0, 2, 4, 6, 8} x store {10, 25, 50}%).  --z-log DIR: every pass's
    pcr_match_prefix inputs and decisions, for the oracle replay (tests/test_z_replay.py)."""
    import torch

    from pcrgen import make_rng, randn_bf16, zipf_trace
    torch.cuda.set_device(0)
    geo = geometry("L8")
    L, Hq, Hkv, d, C, S = geo["L"], geo["Hq"], geo["Hkv"], geo["d"], geo["C"], geo["S_pg"]
    P = max(1, args.rank_slice)
    hq, hkv = Hq // P, Hkv // P
    reqs, _, ndoc = zipf_trace(seed=4, n_requests=args.requests, C=C)
    distinct = set()
    for r, n in zip(reqs, ndoc):
        for c in range(n // C):
            distinct.add(r[: (c + 1) * C].tobytes())
    max_n = max(len(r) for r in reqs)
    pages_req = -(-max_n // S)
    page_elems = L * hkv * 2 * S * d
    n_pool_pages = 2 * pages_req + 1
    pool = torch.empty(n_pool_pages * page_elems, dtype=torch.int16, device="cuda")
    ssd_chunks = int(args.ssd_frac * len(distinct))
    rec = L * hkv * 2 * C * d * 2
    if ssd_chunks:
        # the tier file is pre-sized: refuse (loudly) rather than fill the disk
        free = shutil.disk_usage(os.path.dirname(os.path.abspath(args.ssd_path))).free
        if ssd_chunks * rec > 0.8 * free:
            sys.exit(f"bench: SSD tier of {ssd_chunks} x {rec >> 20} MiB = {ssd_chunks * rec / 1e9:.0f} GB does not "
                     f"fit in 80% of the {free / 1e9:.0f} GB free under {args.ssd_path}; lower --ssd-frac or --requests")
    rng = make_rng(11)
    bufs = tuple(torch.from_numpy(randn_bf16(rng, (L, max_n, h, d)).view(np.int16)).cuda() for h in (hq, hkv, hkv))
    bufs = bufs + (torch.empty_like(bufs[0]),)
    body = _z_layer_body(torch, geo, max_n) if args.layer_body else None
    windows = [int(x) for x in args.z_windows.split(",")] if args.z_windows else [args.window]
    fracs = [float(x) for x in args.z_store_fracs.split(",")] if args.z_store_fracs else [args.store_frac]
    rhos = [float(x) for x in args.rho.split(",")] if args.rho else []

    def header(W, cap, kind, rho=None, service_ms=None):
        return {"trace": "zipf_trace(seed=4)", "requests": len(reqs), "C": C, "S_pg": S, "L": L, "P": P,
                "window": W, "store_chunks": cap, "ssd_chunks": ssd_chunks, "n_pool_pages": n_pool_pages,
                "distinct_chunks": len(distinct), "pass": kind, "rho": rho, "rho_service_ms": service_ms,
                "no_reuse": bool(args.no_reuse)}

    def emit(r, W, cap, frac, clk, poisson=None):
        tt = np.array(r["ttft"])
        wall = r["wall"]
        line = {
            "metric": "Z trace: context tokens/s over the Zipf RAG requests (TTFT per request in ttft_ms_*)",
            "value": r["toks"] / (r["total_ms"] * 1e-3), "unit": "tokens/s", "n_gpus": 1, "steps": len(reqs),
            "warmup": 0, "ms_per_step": r["total_ms"] / len(reqs), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded Zipf(1.0) corpus of 1000 docs x 4-16 chunks, 2 docs + "
                                       "128-256 query tokens per request; random bf16 KV)",
            "config": {"workload": f"Z: L8 shape{f' (rank 0 of a KV-head shard x{P})' if P > 1 else ''}, W={W}, "
                                   f"store={cap} chunks ({frac:.0%} of {len(distinct)} distinct), "
                                   f"ssd={ssd_chunks} chunks, offload on"
                                   + (", +layer body (f3)" if body is not None else "")
                                   + (", NO REUSE (full recompute baseline)" if args.no_reuse else ""),
                       "requests": len(reqs), "window": W, "store_chunks": cap, "store_frac": frac,
                       "ssd_chunks": ssd_chunks, "rank_slice": P, "chunk_bytes": rec},
            "ttft_wall_ms_mean": float(np.mean(wall)), "ttft_wall_ms_p95": float(np.percentile(wall, 95)),
            "tier_stats": r["stats"],
            "ttft_ms_mean": float(tt.mean()), "ttft_ms_p50": float(np.percentile(tt, 50)),
            "ttft_ms_p95": float(np.percentile(tt, 95)), "ttft_ms_p99": float(np.percentile(tt, 99)),
            "ttft_note": "device time from the request's start to its prefill_done_event (last layer's attention; "
                         "first token); step_ms_* add the tail of its layer-wise offload",
            "step_ms_mean": float(np.mean(r["step"])), "step_ms_p95": float(np.percentile(r["step"], 95)),
            "chunk_hit_ratio": r["hits"] / max(1, r["chunks"]), "mean_n1_tokens": float(np.mean(r["n1s"])),
            "match_prefix_us_p50": float(np.percentile(r["plan_us"], 50)), "store_pin_s": r["t_pin"],
            "gpu_launches": r["launches"], "clocks": clk,
        }
        if poisson:
            line["poisson"] = poisson
            line["poisson_note"] = ("saturated pass first (every request waiting from t=0; its mean wall service "
                                    "time sets the rate), then one cold-store pass per rho with Poisson arrivals; "
                                    "ttft_ms_* there = queueing + service (virtual-time FIFO over measured service)")
        print(json.dumps(line), flush=True)

    for frac in fracs:
        cap = max(8, int(frac * len(distinct)))
        for W in windows:
            clocks = ClockSampler(0, pci_bus_id(torch, 0))
            clocks.start()
            clocks.begin()
            r = _z_pass(args, torch, reqs, ndoc, cap, ssd_chunks, pool, bufs, body=body, window=W)
            if args.z_log:
                _write_plan_log(os.path.join(args.z_log, f"z_P{P}_W{W}_store{round(frac * 100)}_ssd"
                                             f"{round(args.ssd_frac * 100)}_sat.jsonl.gz"), header(W, cap, "saturated"),
                                r["log"])
            service_ms = args.rho_service_ms or float(np.mean(r["wall"]))
            poisson = []
            for rho in rhos:
                arr = poisson_arrivals(len(reqs), rho, service_ms)
                rq = _z_pass(args, torch, reqs, ndoc, cap, ssd_chunks, pool, bufs, queue=VirtualQueue(arr, W),
                             body=body, window=W)
                if args.z_log:
                    _write_plan_log(os.path.join(args.z_log, f"z_P{P}_W{W}_store{round(frac * 100)}_ssd"
                                                 f"{round(args.ssd_frac * 100)}_rho{rho}.jsonl.gz"),
                                    header(W, cap, "poisson", rho, service_ms), rq["log"])
                tq = np.array(rq["ttft_q"])
                poisson.append({
                    "rho": rho, "rho_service_ms": service_ms, "arrival_rate_per_s": 1e3 * rho / service_ms,
                    "ttft_ms_mean": float(tq.mean()), "ttft_ms_p50": float(np.percentile(tq, 50)),
                    "ttft_ms_p95": float(np.percentile(tq, 95)), "ttft_ms_p99": float(np.percentile(tq, 99)),
                    "service_ms_mean": float(np.mean(rq["wall"])), "device_ttft_ms_mean": float(np.mean(rq["ttft"])),
                    "mean_pending": float(np.mean(rq["pending"])), "chunk_hit_ratio": rq["hits"] / max(1, rq["chunks"]),
                    "tier_stats": rq["stats"],
                })
            emit(r, W, cap, frac, clocks.stop(), poisson)



def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start N ranks (one process per GPU) with torchrun
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")   # NCCL's init lines (nranks) go to stderr
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd, env=env))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "Z":
        run_trace_z(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
