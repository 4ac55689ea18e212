"""Benchmark of the fused sparse decode step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]
    python bench.py --sweep table1|table2|configs     (rank 0, one GPU: JSON lines per point)

A "step" is one pass of the whole hot path (indexer scan -> exact top-k ->
gather-attend -> LSE merge) over one batch of decode
queries.

* N = 1 (default): BASELINE configs[2] (LOFT-shaped, `cfg3`: B=16, N=128K,
  S=50, Hq=32, Hkv=8, D=128, bf16 paged KV, 8-channel bf16 sketch).
* N > 1 (torchrun, one rank per GPU; default `cfg4`): BASELINE configs[3]
  (SWE-agentic-shaped, B=32 fixed, turn t of the 8K -> 128K trace, default
  t=66 = 128K), KV heads sharded over the ranks (rank r owns Hkv/N KV heads
  and their q-heads of every sequence).  Total work is
  fixed (strong scaling), no collective on the data path; the outputs are
  all-gathered once, outside the timed region, and rank 0 checks them
  bit for bit against the unsharded fused call.
* `--config cfg5` with N > 1: BASELINE configs[4], one 2^20-token sequence
  sequence-sharded over the ranks.

Prints ONE JSON line on rank 0.  Inputs are synthetic (workloads/), resident
in HBM.  Steps rotate among 4 query sets; when a step touches less than 4x the
L2 (126 MB) the L2 is flushed (a 512 MB write, outside the events) before
every timed step, otherwise the step's own traffic (902 MB at cfg3) evicts
the previous step's lines.  Every timed step is bracketed by CUDA events on
the launching stream: `value` = B * K / (sum of the K step times), with the
median / p10 / p90 of the per-step times beside it.  The step is captured in a
CUDA graph (the five PDL-chained kernels keep their programmatic edges) and
the graph is replayed; the eager (per-call) number is reported beside it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn µs/step & HBM GB/s vs roofline at N=128K, 50× sparsity; speedup vs dense"
SCALE = 1.0 / math.sqrt(128)
FALLBACK_HBM = 6650.0
L2_BYTES = 126 * 1024 * 1024


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            sel = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", sel], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def pct(xs, p):
    s = sorted(xs)
    if not s:
        return None
    i = min(len(s) - 1, max(0, int(round(p / 100.0 * (len(s) - 1)))))
    return s[i]


# --------------------------------------------------------------------------- timing
class Timer:
    """Per-step CUDA events on the launching (current) stream.  `flush` (a
    > L2 write) runs before a step, outside its events, when the step's inputs
    could otherwise be served from the previous step's L2 contents."""

    def __init__(self, dev, flush: bool):
        import torch
        self.torch = torch
        self.flush_buf = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev) if flush else None
        self.evict_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if flush else None

    def flush(self):
        # write 512 MB (> 4x L2), then read 256 MB so that the dirty lines are
        # written back here, outside the timed step, and L2 holds clean lines
        self.flush_buf.zero_()
        self.evict_buf.sum()

    def run(self, step, steps, warmup, world=1, dist=None, sampler=None):
        torch = self.torch
        for i in range(warmup):
            if self.flush_buf is not None:
                self.flush()
            step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if sampler:
            sampler.start()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(steps):
            if self.flush_buf is not None:
                self.flush()
            ev[2 * i].record()
            step(i)
            ev[2 * i + 1].record()
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        if world > 1:
            dist.barrier()
        per = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps)]
        total = sum(per)
        if world > 1:
            t = torch.tensor([total], device="cuda" if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return {"total_ms": total, "per_ms": per, "clocks": clocks}


def stats_us(per_ms):
    return {"median": statistics.median(per_ms) * 1e3, "p10": pct(per_ms, 10) * 1e3, "p90": pct(per_ms, 90) * 1e3,
            "mean": statistics.fmean(per_ms) * 1e3, "n": len(per_ms)}


def capture_graphs(fns, stream):
    """One CUDA graph per callable (captured on `stream`, which already owns
    its workspace from an eager warm-up call).  -> (graphs, None) or (None, why)."""
    import torch
    try:
        graphs = []
        for fn in fns:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fn()
            graphs.append(g)
        torch.cuda.synchronize()
        return graphs, None
    except Exception as e:  # capture unsupported: report eager timing only
        torch.cuda.synchronize()
        return None, f"{type(e).__name__}: {e}"[:200]


# --------------------------------------------------------------------------- oracle (cpu_baseline / reference arm)
def oracle_rows(case, cfg, rows, threads):
    """The fp64 oracle as it stands over (b, h) rows, split into (b, g) tasks
    run on `threads` host threads (numpy releases the GIL in its kernels; BLAS
    pinned to one thread per task).  Every task decodes its own (b, g) inputs
    from the stored bf16 bits (no decode cache reused across calls)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    G = cfg["Hq"] // cfg["Hkv"]
    tasks = {}
    for b, h in rows:
        tasks.setdefault((b, h // G), []).append((b, h))
    mode = "sketch" if cfg["sketch"] else "exact"

    def run(task_rows):
        inp = oracle.from_case(case)  # fresh: its lazily decoded K / V / sketch die with the task
        oracle.sparse_decode(inp, cfg["S"], SCALE, mode=mode, rows=task_rows)

    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    try:
        if ctx:
            ctx.__enter__()
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(run, list(tasks.values())))
        return time.perf_counter() - t0
    finally:
        if ctx:
            ctx.__exit__(None, None, None)


def host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg_name, cfg, n_seqs):
    """The fp64 oracle on host cores over a bounded sample (n_seqs full sequences)."""
    import workloads
    case = workloads.make_case(n_seqs, cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=cfg["sketch"],
                               seed=424242, device="cpu")
    rows = [(b, h) for b in range(n_seqs) for h in range(cfg["Hq"])]
    threads = min(host_threads(), n_seqs * cfg["Hkv"])
    dt = oracle_rows(case, cfg, rows, threads)
    return {"value": n_seqs / dt, "unit": "tokens/s", "cores": threads, "kind": "oracle",
            "sample": f"{n_seqs} full sequence(s) of {cfg_name} ({len(rows)} (b,h) rows at N={cfg['N']}), fp64 numpy "
                      f"oracle, one (b, KV head) task per thread, BLAS 1 thread per task, {dt:.2f} s"}


def run_reference(args):
    """--impl reference: the oracle (the only reference this paper has) on host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import workloads
    cfg_name = args.config or "cfg3"
    cfg = dict(workloads.CONFIGS[cfg_name])
    threads = min(host_threads(), cfg["Hkv"])
    case = workloads.make_case(1, cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=cfg["sketch"],
                               seed=424242, device="cpu")
    # each step = the Hq rows of one sequence, bounded so the whole run takes a few minutes
    rows = [(0, h) for h in range(cfg["Hq"])]
    for _ in range(args.warmup):
        oracle_rows(case, cfg, rows[: cfg["Hq"] // cfg["Hkv"]], 1)
    per = [oracle_rows(case, cfg, rows, threads) for _ in range(args.steps)]
    dt = sum(per)
    value = args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg_name, cfg, 1) + "; each step = the 32 (b,h) rows of ONE "
                       "sequence (a bounded sample of the B=16 batch)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                             "sample": f"one {cfg_name} sequence per step, {cfg['Hkv']} (b, KV head) tasks on "
                                       f"{threads} threads, fresh decode of the bf16 inputs every step"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------- helpers
def workload_name(cfg_name, cfg, world, sharded=None):
    base = (f"{cfg_name}: B={cfg['B']}, N={cfg['N']}, S={cfg['S']:g}, Hq={cfg['Hq']}, Hkv={cfg['Hkv']}, D=128, "
            f"page 16, {'bf16' if cfg['dtype'].is_floating_point and cfg['dtype'].itemsize == 2 else 'fp32'} KV, "
            + ((f"sketch C=8 {'fp8 e4m3' if 'float8' in str(cfg.get('sketch_dtype', '')) else 'bf16'}")
               if cfg["sketch"] else "exact scores"))
    if sharded:
        base += sharded
    return base


def union_rows(idx, counts, Hkv):
    import torch
    B, Hq, k = idx.shape
    x = idx.view(B, Hkv, (Hq // Hkv) * k).long()
    x = torch.where(x >= 0, x, torch.full_like(x, -1))
    s = x.sort(-1).values
    new = torch.ones_like(s, dtype=torch.bool)
    new[..., 1:] = s[..., 1:] != s[..., :-1]
    return int((new & (s >= 0)).sum().item())


def get_cfg(name):
    import workloads
    from workloads.gen import _cfg4_len
    if name in workloads.CONFIGS:
        return dict(workloads.CONFIGS[name])
    if name.startswith("cfg4_t"):  # any turn of the SWE-agentic trace
        t = int(name[len("cfg4_t"):])
        return dict(workloads.CONFIGS["cfg4_t66"], N=_cfg4_len(t))
    raise SystemExit(f"unknown config {name}")


def build_case(cfg, seed, dev):
    import workloads
    return workloads.make_case(cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["N"], dtype=cfg["dtype"], sketch=cfg["sketch"],
                               seed=seed, device=dev,
                               **({"sketch_dtype": cfg["sketch_dtype"]} if "sketch_dtype" in cfg else {}))


# --------------------------------------------------------------------------- sequence sharding (cfg5)
def run_seqshard(args, world, rank, dev):
    """BASELINE cfg5: one 2^20-token sequence, sequence-sharded over the ranks
    (SURVEY.md 8(e)): local top-k_b candidates with k_b from the GLOBAL length,
    all-gather of candidate scores, the global cut, local attend, all-gather of
    the normalised partials, LSE merge (paper_2605_24168_b200.parallel)."""
    import torch
    import torch.distributed as dist
    import workloads
    import paper_2605_24168_b200 as sd
    from paper_2605_24168_b200 import parallel as par
    from paper_2605_24168_b200 import roofline as RL

    cfg = dict(workloads.CONFIGS["cfg5"])
    NG, S = cfg["N"], cfg["S"]
    bounds = par.token_bounds(NG, world)
    n_loc = bounds[rank + 1] - bounds[rank]
    case = workloads.make_case(1, cfg["Hq"], cfg["Hkv"], n_loc, dtype=cfg["dtype"], sketch=True,
                               seed=9000 + rank, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(4242)  # the query is the same on every rank
    qs = [torch.randn(case.q.shape, generator=g, device=dev).to(case.q.dtype) for _ in range(4)]
    kv = sd.KVCache.from_case(case)
    sk = sd.SketchCache.from_case(case)
    glens = torch.tensor([NG], dtype=torch.int32, device=dev)
    k = sd.budget_k(S, NG)

    def step(i, q=None):
        backend = par.CudaSeqShardBackend(qs[i % 4] if q is None else q, kv, sk)
        return par.seqshard_decode(backend, glens, NG, S, SCALE, k)

    # survivors of this rank (the rows it must gather) for the byte model
    backend = par.CudaSeqShardBackend(qs[0], kv, sk)
    cs, ci = backend.local_topk(glens, NG, S, k)
    allc = par.all_gather_stack(cs)
    _, _, surv, scnt = sd.seqshard_cut_attend(qs[0], kv, glens, allc, ci, rank, S, scale=SCALE,
                                              return_survivors=True)
    surv_union = union_rows(surv, scnt, cfg["Hkv"])
    timer = Timer(dev, flush=False)
    r = timer.run(step, args.steps, args.warmup, world, dist, ClockSampler(dev.index))
    ms_step = r["total_ms"] / args.steps
    # end to end: the query from pinned host memory, the merged output back
    q_host = torch.stack([q.cpu() for q in qs]).pin_memory()
    out_host = torch.empty(case.q.shape, dtype=torch.float32).pin_memory()
    q_dev = torch.empty_like(qs[0])

    def e2e_step(i):
        q_dev.copy_(q_host[i % 4], non_blocking=True)
        o, _ = step(i, q_dev)
        out_host.copy_(o, non_blocking=True)

    r2 = timer.run(e2e_step, args.steps, 2, world, dist)
    ms_e2e = r2["total_ms"] / args.steps
    hbm, src = peaks()
    model = RL.sparse_step_bytes(1, cfg["Hq"], cfg["Hkv"], n_loc, k, union_rows_total=surv_union)
    t = torch.tensor([float(model["total_union"])], device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    achieved = float(t.item()) / (ms_step * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": 1000.0 / ms_step, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"cfg5: B=1, N={NG}, S={S:g}, Hq=32, Hkv=8, D=128, page 16, bf16 KV, sketch "
                                   f"C=8 bf16; sequence-sharded over {world} GPUs ({n_loc} tokens per rank)",
                       "global_batch": 1, "seq_len": NG, "sparsity": S, "k": k, "parallelism": f"seq-shard{world}",
                       "l2": "per-rank inputs 600+ MB > L2, 4 rotating queries"},
            "us_per_step": ms_step * 1e3, "step_us": stats_us(r["per_ms"]),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "peak_source": src,
                         "kernel": "per-rank step (local scan + top-k + cut + attend), bytes = the busiest rank's "
                                   "shard sketch + the GQA union of ITS survivors (measured)",
                         "algorithmic_bytes_per_launch": float(t.item())},
            "e2e": {"value": 1000.0 / ms_e2e, "unit": "tokens/s", "h2d_bytes_per_step": qs[0].numel() * 2,
                    "d2h_bytes_per_step": out_host.numel() * 4},
            "gpu_launches": None, "clocks": r["clocks"],
            "note": "exchange: two all-gathers per step (candidate scores, normalised partials) over "
                    + dist.get_backend()}))
    dist.barrier()
    return 0


# --------------------------------------------------------------------------- the fused step
def run_fused(args, world, rank, local, dev, dist):
    import torch
    import paper_2605_24168_b200 as sd
    from paper_2605_24168_b200 import parallel as par
    from paper_2605_24168_b200 import roofline as RL

    cfg_name = args.config or ("cfg3" if world == 1 else f"cfg4_t{args.turn}")
    cfg = get_cfg(cfg_name)
    S = cfg["S"]
    strong = cfg_name.startswith("cfg4") and world > 1
    sharded = None
    check = None
    if world == 1:
        import workloads
        case = workloads.config_case(cfg_name, device=dev) if cfg_name in workloads.CONFIGS else \
            build_case(cfg, 777, dev)
        q_full = None
    elif strong:
        # BASELINE configs[3]: one global B=32 batch, KV heads sharded over the ranks
        full = build_case(cfg, 4000 + args.turn, dev)
        sh = par.shard_heads(full.q, full.k_pages, full.v_pages, full.page_table, full.seq_lens,
                             full.sketch_pages, full.channel_ids, world=world, rank=rank)
        if rank == 0:  # the unsharded result, for the bitwise check of the gathered shards
            fkv, fsk = sd.KVCache.from_case(full), sd.SketchCache.from_case(full)
            ref_out, _ = sd.sparse_decode_fused(full.q, fkv, fsk, S=S, scale=SCALE)
            torch.cuda.synchronize()
            check = ref_out
            del fkv, fsk
        q_full = full.q
        from dataclasses import replace
        case = replace(full, q=sh.q, k_pages=sh.k_pages, v_pages=sh.v_pages, sketch_pages=sh.sketch_pages,
                       channel_ids=sh.channel_ids, Hq=sh.q.shape[1], Hkv=sh.k_pages.shape[2])
        del full
        torch.cuda.empty_cache()
        sharded = (f"; KV-head sharded over {world} GPUs (rank r owns KV heads [r*{cfg['Hkv'] // world}, "
                   f"(r+1)*{cfg['Hkv'] // world}) and their q-heads of all {cfg['B']} sequences), strong scaling")
    else:
        # weak scaling of cfg3 shapes (B = 16 N, Hkv / N heads per rank)
        if cfg["Hkv"] % world:
            raise SystemExit(f"--gpus {world} must divide Hkv={cfg['Hkv']}")
        cfg.update(B=cfg["B"] * world, Hkv=cfg["Hkv"] // world, Hq=cfg["Hq"] // world)
        case = build_case(cfg, 7000 + rank, dev)
        sharded = f"; weak scaling: B={cfg['B']}, each rank {cfg['Hkv']} KV heads (per-rank shard shown)"
        q_full = None

    kv = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, cfg["N"])
    sk = sd.SketchCache.from_case(case)
    B, Hq, Hkv = case.B, case.Hq, case.Hkv
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + (0 if strong else rank))
    R = 4
    extra = [torch.randn((B, q_full.shape[1] if strong else Hq, 128), generator=gen, device=dev).to(case.q.dtype)
             for _ in range(R - 1)]
    if strong:
        h0 = rank * Hq
        extra = [e[:, h0:h0 + Hq].contiguous() for e in extra]
    qs = [case.q] + extra
    out = torch.empty(case.q.shape, dtype=case.q.dtype, device=dev)
    lse = torch.empty(case.q.shape[:2], dtype=torch.float32, device=dev)

    # algorithmic bytes from the measured GQA union of the selected rows
    _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=SCALE, return_idx=True)
    E = union_rows(idx, cnt, Hkv)
    k = sd.budget_k(S, cfg["N"])
    model = RL.sparse_step_bytes(B, Hq, Hkv, cfg["N"], k, w=case.dtype.itemsize, exact=not cfg["sketch"],
                                 sketch_w=case.sketch_pages.element_size() if case.sketch_pages is not None else 2,
                                 union_rows_total=E)
    del idx, cnt
    sd.clear_device_error()
    sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=SCALE, out=out, lse=lse)
    fallback_rows = sd.read_stats()["fallback_rows"]
    clear_err = sd.read_device_error()

    # sharded outputs vs the unsharded call (validation only, untimed)
    shard_check = None
    if strong:
        gathered = par.HeadShardedDecoder.gather_outputs(out)
        if rank == 0:
            shard_check = {"bitwise_equal_to_unsharded": bool(torch.equal(gathered, check)),
                           "max_abs_diff": float((gathered.float() - check.float()).abs().max().item())}
        check = None

    flush = model["total_union"] < 4 * L2_BYTES
    timer = Timer(dev, flush)

    def eager(i):
        sd.sparse_decode_fused(qs[i % R], kv, sk, S=S, scale=SCALE, out=out, lse=lse)

    # CUDA graph of the step, one per rotating query (captured on a side stream
    # that owns its workspace from an eager warm-up)
    cap = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(cap):
        for i in range(R):
            eager(i)
    torch.cuda.synchronize()
    graphs, graph_err = (None, "disabled") if args.no_graph else capture_graphs(
        [(lambda i=i: eager(i)) for i in range(R)], cap)

    def replay(i):
        graphs[i % R].replay()

    sampler = ClockSampler(local)
    r_eager = timer.run(eager, args.steps, args.warmup, world, dist, None if graphs else sampler)
    r_graph = timer.run(replay, args.steps, args.warmup, world, dist, sampler) if graphs else None
    # the step launched both ways (same kernels): the faster total is the value
    main_r = r_graph if r_graph and r_graph["total_ms"] <= r_eager["total_ms"] else r_eager
    if main_r is r_eager and r_eager["clocks"] is None:
        main_r = dict(r_eager, clocks=r_graph["clocks"])
    ms_step = main_r["total_ms"] / args.steps
    value = B * 1000.0 / ms_step  # every rank serves all B sequences (its share of the heads)

    # end to end through the public API with pinned host buffers
    q_host = torch.stack([q.cpu() for q in qs]).pin_memory()
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    q_dev = torch.empty_like(case.q)

    def e2e(i):
        q_dev.copy_(q_host[i % R], non_blocking=True)
        sd.sparse_decode_fused(q_dev, kv, sk, S=S, scale=SCALE, out=out, lse=lse)
        out_host.copy_(out, non_blocking=True)

    r_e2e = timer.run(e2e, args.steps, args.warmup, world, dist)
    e2e_value = B * 1000.0 / (r_e2e["total_ms"] / args.steps)

    hbm, src = peaks()
    # dense decode on the same cache (speedup context)
    dense = None
    if not args.no_dense:
        rd = timer.run(lambda i: sd.dense_decode(qs[i % R], kv, scale=SCALE, out=out, lse=lse),
                       max(5, args.steps // 10), 2)
        dms = statistics.median(rd["per_ms"])
        dbytes = RL.dense_bytes(B, cfg["N"], Hkv, w=case.dtype.itemsize)
        dense = {"us_per_step": dms * 1e3, "hbm_gbs": dbytes / (dms * 1e-3) / 1e9,
                 "frac": dbytes / (dms * 1e-3) / 1e9 / hbm,
                 "speedup_sparse_vs_dense": dms / statistics.median(main_r["per_ms"])}

    # per-kernel durations (CUDA events between the fused call's kernels; this
    # serialises them, so it is a separate, untimed-for-value measurement)
    nt = 20
    phase_sum = {p: 0.0 for p in sd.api.FUSED_PHASES}
    for i in range(nt + 2):
        if flush:
            timer.flush()
        _, _, ph = sd.api.sparse_decode_fused_timed(qs[i % R], kv, sk, S=S, scale=SCALE, out=out, lse=lse)
        if i >= 2:
            for p2 in phase_sum:
                phase_sum[p2] += ph[p2] / nt
    phases_us = {p2: v * 1e3 for p2, v in phase_sum.items()}
    serial_us = sum(v for v in phases_us.values() if v > 0)

    step_achieved = model["total_union"] / (ms_step * 1e-3) / 1e9
    # dominant kernel: the gather-attend; algorithmic bytes per launch = the
    # GQA-union K/V rows of the step (512 B per union row) +
    # the queries / outputs
    attend_bytes = model["rows_union"] + model["io"]
    achieved = attend_bytes / (phases_us["attend"] * 1e-6) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp)).get(cfg_name if world == 1 else f"{cfg_name}_tp{world}")
        if tj:
            traffic = tj.get("kernels", {}).get("attend_union_ws_kernel")
    par_name = ("single-gpu" if world == 1 else f"kv-head-shard{world}")
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "bf16" if case.dtype == torch.bfloat16 else "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg_name, cfg, world, sharded), "global_batch": B,
                   "seq_len": cfg["N"], "sparsity": S, "k": k,
                   "l2": ("L2 flushed (512 MB write + 256 MB read) before every timed step" if flush else
                          f"inputs > L2: {model['total_union'] / 1e6:.0f} MB touched per step, 4 rotating queries"),
                   "launch": ("cuda-graph replay (5 PDL-chained kernels per step; faster than eager calls)"
                              if main_r is r_graph else
                              "eager C-ABI calls (5 PDL-chained kernels per step; faster than the graph replay "
                              f"{stats_us(r_graph['per_ms'])['median']:.1f} us)" if graphs else
                              f"eager C-ABI calls (graph capture: {graph_err})"),
                   "parallelism": par_name},
        "us_per_step": ms_step * 1e3,
        "step_us": stats_us(main_r["per_ms"]),
        "eager_step_us": stats_us(r_eager["per_ms"]),
        "graph_step_us": stats_us(r_graph["per_ms"]) if r_graph else None,
        "hbm_gbs": step_achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "peak_source": src,
                     "kernel": "attend_union_ws_kernel (GQA-union gather-attend)",
                     "algorithmic_bytes_per_launch": attend_bytes, "launch_us": phases_us["attend"],
                     "share_of_step": phases_us["attend"] / serial_us},
        "step_roofline": {"achieved": step_achieved, "frac": step_achieved / hbm,
                          "frac_median": model["total_union"] / (statistics.median(main_r["per_ms"]) * 1e-3) / 1e9
                          / hbm,
                          "algorithmic_bytes_per_step": model["total_union"],
                          "bytes_model": {k2: v for k2, v in model.items()}},
        "phases_us": {**phases_us, "note": "CUDA events between the kernels (serialised, no PDL overlap)"},
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": case.q.numel() * case.q.element_size(),
                "d2h_bytes_per_step": out.numel() * out.element_size(), "step_us": stats_us(r_e2e["per_ms"]),
                "path": "eager sd_sparse_decode_fused calls with the query copied from pinned host memory and the "
                        "output copied back inside every step"},
        "gpu_launches": args.steps * sd.api.LAUNCHES_PER_FUSED,
        "clocks": main_r["clocks"],
        "dense": dense,
        "device_error": clear_err,
        "fallback_rows": fallback_rows,
    }
    if shard_check is not None:
        line["shard_check"] = shard_check
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg_name, cfg, args.cpu_seqs)
    if rank == 0:
        print(json.dumps(line))


# --------------------------------------------------------------------------- sweeps (Table 1 / Table 2 layout)
PAPER_T1 = {1: [0.32, 0.63, 1.45, 2.58, 5.57, 10.25, 11.05, 11.14], 4: [0.33, 0.66, 1.64, 3.18, 7.45, 13.36, 24.25, 42.04],
            8: [0.38, 0.77, 1.90, 3.75, 8.88, 16.82, 29.64, 76.14], 16: [0.45, 0.89, 2.21, 4.35, 10.54, 20.09, 37.32, 76.77]}
T1_S = [2, 4, 10, 20, 50, 100, 200, 500]
PAPER_T2 = {"gqa": {1: [0.28, 0.56, 0.83, 1.12, 1.46, 1.65], 4: [0.32, 0.67, 1.06, 1.52, 2.11, 2.45],
                    8: [0.36, 0.75, 1.18, 1.68, 2.30, 2.66], 16: [0.41, 0.85, 1.31, 1.82, 2.46, 2.81]},
            "mha": {1: [0.91, 1.62, 2.18, 2.68, 3.14, 3.37], 4: [1.02, 1.86, 2.56, 3.17, 3.74, 4.00],
                    8: [1.12, 2.00, 2.71, 3.32, 3.86, 4.11], 16: [1.22, 2.13, 2.84, 3.43, 3.94, 4.17]}}
T2_S = [2, 5, 10, 20, 50, 100]


def run_sweep(args, dev):
    """Table 1 (backend only, given per-head indices) and Table 2
    (indexer-inclusive fused step) layouts at N=128K, plus the
    BASELINE configs not covered by the default line (cfg1, cfg2, cfg4 turns,
    cfg5 on one GPU).  Every point: median / p10 / p90 over `--steps` steps
    with the L2 flushed before each, dense decode on the same cache, the
    roofline fraction on the bytes the point must move."""
    import torch
    import workloads
    import paper_2605_24168_b200 as sd
    from paper_2605_24168_b200 import roofline as RL
    hbm, _ = peaks()
    timer = Timer(dev, flush=True)
    N = 131072
    steps, warm = args.steps, max(3, args.warmup)

    def emit(d):
        print(json.dumps(d), flush=True)

    def dense_us(q, kv):
        r = timer.run(lambda i: sd.dense_decode(q, kv, scale=SCALE), max(5, steps // 4), 2)
        return statistics.median(r["per_ms"]) * 1e3

    def fused_point(case, kv, sk, S, q_list, B, Hq, Hkv, Nn):
        out = torch.empty(case.q.shape, dtype=case.q.dtype, device=dev)
        lse = torch.empty(case.q.shape[:2], dtype=torch.float32, device=dev)
        _, _, idx, cnt = sd.sparse_decode_fused(case.q, kv, sk, S=S, scale=SCALE, return_idx=True)
        E = union_rows(idx, cnt, Hkv)
        k = sd.budget_k(S, Nn if isinstance(Nn, int) else max(Nn))
        model = RL.sparse_step_bytes(B, Hq, Hkv, Nn, k, w=case.dtype.itemsize, exact=sk is None,
                                     union_rows_total=E)
        sd.clear_device_error()
        r = timer.run(lambda i: sd.sparse_decode_fused(q_list[i % len(q_list)], kv, sk, S=S, scale=SCALE, out=out,
                                                       lse=lse), steps, warm)
        st = stats_us(r["per_ms"])
        return idx, cnt, model, st, sd.read_stats()["fallback_rows"], sd.read_device_error()

    which = args.sweep
    if which in ("table1", "table2"):
        layouts = [("gqa", 32, 8)] + ([("mha", 32, 32)] if which == "table2" else [])
        for lay, Hq, Hkv in layouts:
            for B in (1, 4, 8, 16):
                case = workloads.make_case(B, Hq, Hkv, N, seed=5000 + B, device=dev)
                kv, sk = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, N), \
                    sd.SketchCache.from_case(case)
                g = torch.Generator(device=dev)
                g.manual_seed(17)
                qs = [case.q] + [torch.randn(case.q.shape, generator=g, device=dev).to(case.q.dtype) for _ in range(3)]
                d_us = dense_us(case.q, kv)
                for j, S in enumerate(T1_S if which == "table1" else T2_S):
                    idx, cnt, model, st, fb, err = fused_point(case, kv, sk, float(S), qs, B, Hq, Hkv, N)
                    pt = {"sweep": which, "layout": lay, "B": B, "N": N, "S": S, "Hq": Hq, "Hkv": Hkv,
                          "k": sd.budget_k(float(S), N), "dense_us": d_us}
                    if which == "table1":
                        # backend only: weighted attention given per-head indices, per-head gathers
                        out = torch.empty(case.q.shape, dtype=case.q.dtype, device=dev)
                        r = timer.run(lambda i: sd.sparse_gather_attend(case.q, kv, idx, cnt, scale=SCALE, out=out),
                                      steps, warm)
                        b_st = stats_us(r["per_ms"])
                        per_head = model["rows_per_head"] + model["io"] + model["page_table"]
                        pt.update(backend_us=b_st, speedup_vs_dense=d_us / b_st["median"],
                                  paper_speedup_vs_flashinfer_h100=PAPER_T1[B][j],
                                  frac_per_head_bytes=per_head / (b_st["median"] * 1e-6) / 1e9 / hbm,
                                  frac_union_bytes=(model["rows_union"] + model["io"]) / (b_st["median"] * 1e-6)
                                  / 1e9 / hbm,
                                  fused_step_us=st["median"])
                    else:
                        pt.update(fused_us=st, speedup_vs_dense=d_us / st["median"],
                                  paper_speedup_vs_flashinfer_h100=PAPER_T2[lay][B][j],
                                  frac=model["total_union"] / (st["median"] * 1e-6) / 1e9 / hbm,
                                  bytes=model["total_union"], fallback_rows=fb, device_error=err)
                    emit(pt)
                    del idx, cnt
                del case, kv, sk, qs
                torch.cuda.empty_cache()
        return
    # the remaining BASELINE configs, one GPU each
    for name in (args.sweep_configs or "cfg1,cfg2_s10,cfg2_s50,cfg2_s100,cfg4_t0,cfg4_t33,cfg4_t66,cfg4_mixed,"
                                       "cfg3_fp8,cfg5").split(","):
        if name == "cfg4_mixed":
            # one batch of mixed lengths: sequence b at turn (t0 + 2b) mod 67 (SURVEY.md 8(d) cfg 4)
            from workloads.gen import _cfg4_len
            cfg = get_cfg("cfg4_t66")
            lens = [_cfg4_len((5 + 2 * b) % 67) for b in range(cfg["B"])]
            case = workloads.make_case(cfg["B"], 32, 8, lens, seed=4321, device=dev)
            Nn = lens
        else:
            cfg = get_cfg(name)
            case = build_case(cfg, 6000, dev)
            Nn = cfg["N"]
        kv = sd.KVCache(case.k_pages, case.v_pages, case.page_table, case.seq_lens, max(Nn) if isinstance(Nn, list) else Nn)
        sk = sd.SketchCache.from_case(case)
        g = torch.Generator(device=dev)
        g.manual_seed(17)
        qs = [case.q] + [torch.randn(case.q.shape, generator=g, device=dev).to(case.q.dtype) for _ in range(3)]
        S = cfg["S"]
        _, _, model, st, fb, err = fused_point(case, kv, sk, S, qs, case.B, case.Hq, case.Hkv, Nn)
        d_us = dense_us(case.q, kv)
        dbytes = RL.dense_bytes(case.B, Nn, case.Hkv, w=case.dtype.itemsize)
        emit({"sweep": "configs", "config": name, "B": case.B, "N": Nn if isinstance(Nn, int) else f"mixed {min(Nn)}..{max(Nn)}",
              "S": S, "Hq": case.Hq, "Hkv": case.Hkv, "fused_us": st, "tokens_per_s": case.B / (st["median"] * 1e-6),
              "bytes": model["total_union"], "frac": model["total_union"] / (st["median"] * 1e-6) / 1e9 / hbm,
              "dense_us": d_us, "dense_frac": dbytes / (d_us * 1e-6) / 1e9 / hbm, "speedup_vs_dense": d_us / st["median"],
              "fallback_rows": fb, "device_error": err, "l2": "flushed before every step"})
        del case, kv, sk, qs
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=None, help="cfg3 (N=1 default), cfg4_t<turn> (N>1 default), cfg5, ...")
    ap.add_argument("--turn", type=int, default=66, help="cfg4 turn for the N>1 default")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seqs", type=int, default=2, help="sequences in the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--sweep", choices=["table1", "table2", "configs"], default=None)
    ap.add_argument("--sweep-configs", default=None)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2605_24168_b200 as sd

    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # BENCH_SHARE_DEVICE=1 + BENCH_DIST_BACKEND=gloo: every rank on cuda:0 (a
    # smoke test of the multi-rank path on one GPU; not a scaling measurement)
    if os.environ.get("BENCH_SHARE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    sd.load_library()
    if args.sweep:
        if rank == 0:
            run_sweep(args, dev)
        return 0
    if args.config == "cfg5" and world > 1:
        return run_seqshard(args, world, rank, dev)
    run_fused(args, world, rank, local, dev, dist)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
