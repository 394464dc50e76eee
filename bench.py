#!/usr/bin/env python
"""Benchmark: full LCOM/CBO metric pass + move-method candidate sweep on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

One step = one pass of the hot path over the synthetic system resident in HBM:
metric pass (LCOM normalized, LCOM-CK, CBO, U rows) + threshold means + the
cohesion/coupling candidate sweep (every (method, destination) candidate
scored ungated, suggest_all ordered output) + for N > 1 the NCCL all-gather
of the per-shard suggestion lists. Metric: move-method candidates scored per
second, N_cand = Σ_u |used_classes(u)| over the whole system.

For N > 1 run under torchrun (one process per GPU): the metric pass is
replicated (no exchange), the sweep is sharded by cost-balanced contiguous
class ranges and the shard lists are all-gathered (counts, then padded
records); every rank ends with the full ordered list.

--impl reference times the reference CPU implementation (oracle/_ref, the
reference headers compiled in place; the C restatement oracle/liboracle.so
when that is absent) on the host cores, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # SURVEY.md §8d generator calls
    "c2": dict(seed=1, n_classes=1000, n_methods=10000, n_attributes=20000, k_max_calls=4, k_max_accesses=4,
               intra_class_bias=0.5),
    "c3": dict(seed=1, n_classes=10000, n_methods=100000, n_attributes=200000, k_max_calls=4, k_max_accesses=4,
               intra_class_bias=0.5, zipf_s=1.0),
    "c4": dict(seed=1, n_classes=100000, n_methods=1000000, n_attributes=2000000, k_max_calls=4,
               k_max_accesses=4, intra_class_bias=0.5),
    "c5": dict(seed=3, n_classes=5000, n_methods=2500000, n_attributes=320000, k_max_calls=4, k_max_accesses=32,
               intra_class_bias=0.9),
    # C4 shape at 8x the size (size scaling of one GPU; not a SURVEY config)
    "c4x8": dict(seed=1, n_classes=800000, n_methods=8000000, n_attributes=16000000, k_max_calls=4,
                 k_max_accesses=4, intra_class_bias=0.5),
}
WORKLOAD_NAMES = {
    "c2": "C2 synthetic 1k classes / 10k methods / 20k attributes",
    "c3": "C3 synthetic Zipf(s=1) 10k classes / 100k methods / 200k attributes",
    "c4": "C4 synthetic 100k classes / 1M methods / 2M attributes (metric pass + cohesion/coupling sweep)",
    "c5": "C5 dense-coupling 5k classes x 500 methods / 320k attributes",
    "c4x8": "C4 shape x8: 800k classes / 8M methods / 16M attributes",
}
DATA = "synthetic (the reference generate(), SURVEY.md §8d seeds; C3 Zipf ownership + the reference's draws)"
METRIC = "move-method candidates scored/sec (full LCOM+CBO recompute + cohesion/coupling sweep per step)"
UNIT = "candidates/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(sys_, cbo, n_sugg: int, rank_share: float = 1.0) -> dict:
    """Compulsory bytes per launch of each kernel: every array the kernel must
    touch, read or written once (DESIGN.md §4 derives each line), over the
    classes that kernel actually serves (the upload plan's kinds, restated
    here: CTA path M > 32 | A > 64 | member degree > 16; lean = the rest with
    ≤ 32 foreign edges; group = lean with member degree ≤ 8). m, c, a =
    methods, classes, attributes; E = call + access edges; nnz = Σ cbo (U row
    entries) of the kind; S = emitted suggestion records; the sweep kernels
    scale with the rank's share of methods."""
    m, c, a = sys_.n_methods, sys_.n_classes, sys_.n_attributes
    E = sys_.n_calls + sys_.n_accesses
    ms = int(m * rank_share)
    cbo = np.asarray(cbo, dtype=np.int64)
    nnz_u = int(cbo.sum())
    msz = np.diff(sys_.class_method_off).astype(np.int64)
    asz = np.diff(sys_.class_attr_off).astype(np.int64)
    deg = (np.diff(sys_.call_off) + np.diff(sys_.acc_off)).astype(np.int64)
    pos_cls = np.repeat(np.arange(c), msz)                 # class of each class-order position
    pdeg = deg[sys_.class_methods]
    maxdeg = np.zeros(c, np.int64)
    np.maximum.at(maxdeg, pos_cls, pdeg)
    # foreign edges per class (owner of the target != own class)
    own_of_method = np.empty(m, np.int64)
    own_of_method[sys_.class_methods] = pos_cls
    ce = np.repeat(np.arange(m), np.diff(sys_.call_off))
    ae = np.repeat(np.arange(m), np.diff(sys_.acc_off))
    fc = own_of_method[sys_.call_tgt] != own_of_method[ce]
    aown = np.empty(a, np.int64)
    aown[sys_.class_attrs] = np.repeat(np.arange(c), asz)
    fa = aown[sys_.acc_tgt] != own_of_method[ae]
    foreign = np.bincount(own_of_method[ce[fc]], minlength=c) + np.bincount(own_of_method[ae[fa]], minlength=c)
    large = (msz > 32) | (asz > 64) | (maxdeg > 16)
    lean = ~large & (foreign <= 32)
    big = ~large & ~lean
    group = lean & (maxdeg <= 8)

    def kind(sel):
        mem = np.repeat(sel, msz)
        return int(sel.sum()), int(msz[sel].sum()), int(asz[sel].sum()), int(pdeg[mem].sum()), int(cbo[sel].sum())

    c_l, m_l, a_l, e_l, n_l = kind(large)
    c_b, m_b, a_b, e_b, n_b = kind(big)
    c_n, m_n, a_n, e_n, n_n = kind(lean)
    c_g, m_g, a_g, e_g, n_g = kind(group)
    k = {
        # fused method + class pass of the lean classes: plan + edge ranges,
        # edge targets + member bytes, owner tables, records + headers, class
        # records + metrics, U rows
        "class_lean": 32 * c_n + 5 * e_n + 4 * m + 8 * a + 36 * m_n + 84 * c_n + 8 * n_n,
        # the same outputs from groups of lean classes per warp: plan, member
        # rows (offsets + class), edge targets, owner tables (method owner,
        # attr_info), records + headers, class records + metrics, U rows
        "class_group": 16 * c_g + 12 * m_g + 4 * e_g + 4 * m + 8 * a + 36 * m_g + 84 * c_g + 8 * n_g,
        # CTA path: member records + headers + own masks, plans / class
        # records / metrics, U rows (CSR rows only for overflowed records)
        "class_large": 44 * m_l + 93 * c_l + 8 * n_l,
        # method pass over the classes that are not lean
        "method": 64 * (m_l + m_b) + 8 * a + 4 * (e_l + e_b) + 4 * (c_l + c_b),
        # listed warp path (the big warp-path classes)
        "class_small": 44 * m_b + 93 * c_b + 8 * n_b,
        "thresholds": 12 * c,
        "score": 56 * ms + 64 * c + 4 * nnz_u,
        "offsets": 36 * ms + 12 * c,
        # emitters, method records, class records (origin + destination), records
        "write": 16 * n_sugg + 36 * n_sugg + 48 * n_sugg + 64 * n_sugg,
        # tensor-core LCOM-CK reads each member's own mask once
        "ck_mma": 8 * int(msz[(msz >= 128) & (msz <= 3328) & (asz <= 64)].sum()),
    }
    # the class pass: the CTA-path tiers, the listed warp path and the
    # tensor-core LCOM-CK, concurrent on their streams
    k["class_pass"] = k["class_large"] + k["class_small"] + k["ck_mma"]
    k["plan_kinds"] = {"large": c_l, "big": c_b, "lean": c_n, "group": c_g}
    # SURVEY.md §8d layout-independent totals, for reference
    b_in = 4 * (2 * (m + 1) + E + m + a)
    b_cls = 4 * ((c + 1) + m + (c + 1) + a) + 24 * c
    b_u = 4 * (c + 1) + 8 * nnz_u
    k["survey_metric_pass"] = b_in + b_cls + b_u + 20 * c
    k["survey_sweep"] = int(rank_share * b_in) + b_cls + b_u + 64 * n_sugg
    return k


def tensor_roofline(sys_, ck_us: float) -> dict:
    """k_ck_mma (classes with 128 ≤ M ≤ 3328 members and A ≤ 64 attributes): useful
    int8 operations = 2·64 per member pair (the dot product of two 64-byte 0/1 rows),
    executed = every 128×64×64 half-tile UMMA of the upper triangle."""
    msz = np.diff(sys_.class_method_off).astype(np.int64)
    asz = np.diff(sys_.class_attr_off).astype(np.int64)
    sel = (msz >= 128) & (msz <= 3328) & (asz <= 64)
    M = msz[sel]
    useful = float((2 * 64 * M * (M - 1) // 2).sum())
    T = (M + 127) // 128
    executed = float((T * (T + 1) * 2 * 128 * 64 * 64).sum())
    pk = ROOT / "profiles" / "r2_peaks.json"
    peak = json.loads(pk.read_text()).get("i8_mma_tops") if pk.exists() else None
    ach = useful / (ck_us * 1e-6) / 1e12
    return {"kernel": "ck_mma", "bound": "tensor", "unit": "TOPS (int8)", "achieved": ach,
            "executed": executed / (ck_us * 1e-6) / 1e12, "peak": peak,
            "frac": (ach / peak) if peak else None, "classes": int(sel.sum()),
            "peak_source": "profiles/r2_peaks.json (tools/peaks.cu: tcgen05.mma kind::i8 128x256x32, all SMs)",
            "note": "in situ (concurrent with k_class_large on its own stream); the drain of the TMEM accumulator "
                    "(one compare per pair) bounds it, not the tensor core"}


def cpp_dropin_e2e():
    """The C++ drop-in end to end (tools/e2e_cpp.cpp): the reference's SystemModel +
    DependencyTable -> gpu::parallel_class_metrics + gpu::compute_thresholds +
    gpu::suggest_all (free functions: one upload per call, as the reference takes
    the model by const& each time) and the same calls on one resident gpu::Engine;
    wall clock around complete calls (host vectors out), median of 10 steps."""
    exe = ROOT / "tools" / "_build" / "e2e_cpp"
    if not exe.exists():
        return {"unavailable": "tools/_build/e2e_cpp not built (needs the reference headers at build time)"}
    try:
        r = subprocess.run([str(exe), "--steps", "10", "--warmup", "3"], capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as exc:
        return {"unavailable": f"e2e_cpp failed: {exc}"}
    if "error" in d:
        return {"unavailable": d["error"]}
    cand = d["candidates"]
    return {"free_functions": {"ms_per_step": d["free_functions_ms"], "value": cand / (d["free_functions_ms"] / 1e3),
                               "unit": UNIT, "uploads_per_step": 2},
            "engine": {"ms_per_step": d["engine_ms"], "value": cand / (d["engine_ms"] / 1e3), "unit": UNIT,
                       "uploads_per_step": 1},
            "suggestions": d["suggestions"],
            "path": "reference generate() -> SystemModel/DependencyTable -> gpu.hpp (flattening to CSR, H2D, "
                    "metric pass, D2H, device means, sweep, D2H, std::vector<MoveSuggestion>)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons around the timed region (B200_PROFILING.md).

    Sampling starts before the warm-up (nvidia-smi needs ~0.1-0.3 s to emit its
    first row); `wait_for_samples` lets the caller extend the warm-up until it
    is live, and `summary` keeps the rows stamped inside the timed window
    (widened by one sampling interval on each side)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 20

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def _rows(self):
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 10:
                    rows.append(f)
        except OSError:
            pass
        return rows

    def wait_for_samples(self, n: int = 2, timeout_s: float = 3.0) -> bool:
        t = time.time()
        while self.proc and time.time() - t < timeout_s:
            if len(self._rows()) >= n:
                return True
            time.sleep(0.02)
        return False

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        self.wait_for_samples(len(self._rows()) + 1, 1.0)

    def summary(self) -> dict:
        import datetime
        rows = self._rows()
        sel = []
        slack = 2 * self.PERIOD_MS / 1e3
        for r in rows:
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.t0 is not None and self.t0 - slack <= ts <= (self.t1 or ts) + slack:
                sel.append(r)
        window = "timed region"
        if not sel and rows:
            sel, window = rows[-5:], "adjacent (timed region shorter than the sampling period)"
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[2]) for r in sel if r[2].replace(".", "").isdigit()]
        mx = [float(r[3]) for r in sel if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in sel for n, v in zip(names, r[6:10]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel), "window": window}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the reference compiled in place (oracle/_ref)
# ---------------------------------------------------------------------------

def host_cpu() -> dict:
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


class RefJob:
    """One step of the reference's own CPU path on the host cores, on the same
    workload: parallel_class_metrics + parallel_lcom_ck (parallel.hpp:149,164)
    with n_workers = all host threads, compute_thresholds (suggest.hpp:46),
    then the cohesion+coupling sweep — the reference's suggest_all is
    single-threaded, so its per-method body (detail::used_classes +
    detail::emit_for_method + what_if_move) runs on all host threads over the
    reference's detail::run_partitioned ranges and suggest_all's merge/sort
    follows ("reference logic, harness threads", SURVEY.md §8d item 4;
    oracle/ref_shim.cpp ref_sweep). The input comes from the reference's own
    generate() (no product library is loaded). `frac` < 1 sweeps every
    k-th method only (bounded sample) and is extrapolated by candidate
    count; the measured sample time is reported beside it."""

    def __init__(self, config: str):
        import oracle  # CPU baseline / reference arm only
        self.oracle = oracle
        if not oracle.ref_available():
            raise RuntimeError("oracle/_ref/libmmref.so missing (build() compiles it where /root/reference exists)")
        self.cfg = CONFIGS[config]
        t0 = time.perf_counter()
        self.R = oracle.ref_generate_model(**self.cfg)
        self.n_cand = self.R.candidates()
        self.gen_s = time.perf_counter() - t0
        self.threads = os.cpu_count() or 1
        self.n_methods = self.R.n_methods

    def step(self, frac: float = 1.0) -> dict:
        o = self.oracle
        t0 = time.perf_counter()
        lcom, ck, cbo = self.R.class_metrics(self.threads)
        t1 = time.perf_counter()
        thr = o.ref_thresholds(lcom, cbo)
        t2 = time.perf_counter()
        methods = None
        if frac < 1.0:
            k = max(1, int(round(1.0 / frac)))
            methods = np.arange(0, self.n_methods, k, dtype=np.uint32)
        recs, cand = self.R.sweep(lcom, cbo, abi_mask(), thr.lcom, thr.cbo, 0, False, methods=methods,
                                  n_workers=self.threads, dynamic=False)
        t3 = time.perf_counter()
        sweep_s = t3 - t2
        full_s = (t1 - t0) + (t2 - t1) + sweep_s * (self.n_cand / max(1, cand))
        return {"metric_pass_s": t1 - t0, "thresholds_s": t2 - t1, "sweep_s": sweep_s, "sweep_candidates": cand,
                "suggestions": len(recs), "full_job_s": full_s, "measured_s": t3 - t0,
                "extrapolated": methods is not None}

    def describe(self, r: dict) -> str:
        what = ("the full job" if not r["extrapolated"] else
                f"a sample (every {int(round(self.n_cand / max(1, r['sweep_candidates'])))}-th method's sweep, "
                f"{r['sweep_candidates']} of {self.n_cand} candidates, {r['measured_s']:.2f} s measured, "
                f"extrapolated by candidate count)")
        return (f"reference headers compiled in place (oracle/_ref, g++ -O3 -DNDEBUG): parallel_class_metrics + "
                f"parallel_lcom_ck on {self.threads} threads, compute_thresholds, cohesion+coupling sweep with the "
                f"reference's per-method code on {self.threads} threads (detail::run_partitioned) + suggest_all's "
                f"merge; input from the reference's generate(); {what}")


def abi_mask() -> int:
    return (1 << 1) | (1 << 2)  # MM_CRIT_COHESION | MM_CRIT_COUPLING (include/mmgpu.h)


def cpu_baseline(config: str, budget_s: float = 30.0) -> dict:
    """Bounded CPU baseline for our arm's line (rank 0, N=1): one full
    reference job when it fits the budget, else a method sample."""
    job = RefJob(config)
    frac = 1.0
    r = job.step(0.02)  # probe: 2 % of the sweep
    est = r["metric_pass_s"] + r["sweep_s"] * 50
    if est > budget_s:
        frac = max(0.001, min(1.0, (budget_s - r["metric_pass_s"]) / max(1e-9, r["sweep_s"] * 50)))
    r = job.step(frac)
    return {"value": job.n_cand / r["full_job_s"], "unit": UNIT, "cores": job.threads, "kind": "reference",
            "sample": job.describe(r), "host": host_cpu(), **r}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return  # the reference CPU path runs once, on rank 0
    job = RefJob(args.config)
    # size each step so the whole --steps K --warmup W run ends in a few minutes
    probe = job.step(0.02)
    full_est = probe["metric_pass_s"] + probe["sweep_s"] * 50
    budget = 180.0 / max(1, args.steps + args.warmup)
    frac = 1.0 if full_est <= budget else max(0.001, (budget - probe["metric_pass_s"]) / max(1e-9, probe["sweep_s"] * 50))
    for _ in range(args.warmup):
        job.step(frac)
    rs = [job.step(frac) for _ in range(args.steps)]
    t = float(np.mean([r["full_job_s"] for r in rs]))
    v = job.n_cand / t
    last = rs[-1]
    cb = {"value": v, "unit": UNIT, "kind": "reference", "cores": job.threads, "sample": job.describe(last),
          "host": host_cpu(), "measured_s_per_step": float(np.mean([r["measured_s"] for r in rs])),
          "extrapolated": last["extrapolated"], "suggestions": last["suggestions"]}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32+f64", "data": DATA, "config": bench_config(args.config, job.n_cand),
        "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "metric_pass_ms": float(np.mean([r["metric_pass_s"] for r in rs])) * 1e3,
    }), flush=True)


def bench_config(config: str, n_cand: int) -> dict:
    """The workload, identical on both arms (the driver compares them)."""
    return {"workload": WORKLOAD_NAMES[config], **CONFIGS[config], "candidates": n_cand,
            "l2": "inputs resident; L2 flushed between timed steps by a 256 MiB device write outside the events"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args) -> None:
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1308_4011_b200 import Engine, System, abi, plan_shards

    cfg = CONFIGS[args.config]
    t0 = time.time()
    s = System.generate(**cfg)
    n_cand = s.n_candidates()
    log(f"[rank {rank}] generated {args.config}: {s.n_classes} classes, {s.n_methods} methods, "
        f"{s.n_calls}+{s.n_accesses} edges, {n_cand} candidates in {time.time() - t0:.1f}s")
    bounds = plan_shards(s, world)
    shard = (int(bounds[rank]), int(bounds[rank + 1]))
    stream = torch.cuda.Stream(dev)  # all engine work and the timing events share this stream
    torch.cuda.set_stream(stream)
    eng = Engine(local, stream=stream.cuda_stream)
    eng.upload(s)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    def gather(n_local: int):
        """All-gather the shard lists (counts, then count-padded records) over NCCL."""
        from paper_1308_4011_b200.shard import allgather_records, device_records_tensor
        ptr, _ = eng.device_result()
        return allgather_records(device_records_tensor(ptr, n_local, dev), n_local)

    def step():
        # metric pass + thresholds + sweep: one CUDA-graph replay (mm_run)
        if world == 1:
            eng.run(thresholds=None)
            return None
        eng.run(thresholds=None, class_range=shard)
        return gather(eng.sweep_stats()["suggestions"])

    clocks = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # keep warming up (bounded) until the clock sampler is emitting rows
    t_w = time.time()
    while not clocks.wait_for_samples(2, 0.0) and time.time() - t_w < 3.0:
        step()
        torch.cuda.synchronize(dev)
    st = eng.sweep_stats()
    n_sugg_local = st["suggestions"]

    def timed(k):
        """k steps between per-step CUDA events on the engine's stream, L2
        flushed before each (outside the events); returns the per-step ms."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(k):
            flush.fill_(i)  # evict L2 (256 MiB write) outside the timed interval
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
            if eng_profiling[0]:
                eng.collect_timings()  # this replay's per-kernel event times (host sync outside the events)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return [a.elapsed_time(b) for a, b in evs]

    if world > 1:
        import torch.distributed as dist
    # (1) the product step, uninstrumented: value and ms_per_step
    eng_profiling = [False]
    clocks.mark_start()
    step_ms = timed(args.steps)
    # (2) the same K steps with a CUDA event pair around every kernel (graph
    # event nodes, ~10% slower): the per-kernel durations for the roofline
    eng.set_profiling(True)
    eng_profiling[0] = True
    for _ in range(2):
        step()  # re-capture with the timing nodes
    torch.cuda.synchronize(dev)
    eng.reset_kernel_stats()
    step_ms_prof = timed(args.steps)
    clocks.mark_end()
    clocks.__exit__(None, None, None)
    total_ms = float(sum(step_ms))
    kstats = eng.kernel_stats()
    eng.set_profiling(False)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n_cand / (ms_per_step / 1e3)

    # per-kernel averages over the timed region (events on the launching stream)
    kern = {k: {"launches": n, "avg_us": 1e3 * ms / n} for k, (n, ms) in kstats.items() if n}
    # spans that are not single kernels: class_pass brackets class_small + the
    # class_large tiers (counted there); ck_rows is k_ck_rows + k_ck_finalize
    kernels_per_span = {"class_pass": 0, "ck_rows": 2}
    gpu_launches = int(sum(n * kernels_per_span.get(k, 1) for k, (n, _) in kstats.items()))
    lcom, ck, cbo = eng.class_metrics_all()
    nnz_u = int(cbo.astype(np.int64).sum())
    share = 1.0 / world
    ab = algorithmic_bytes(s, cbo, n_sugg_local, share)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # the dominant unit per step: one kernel, or the class pass whose kernels overlap
    units = [k for k in kern if k in ab and k not in ("class_small", "class_large", "ck_mma")]
    dom = max(units, key=lambda k: kern[k]["avg_us"] * kern[k]["launches"])
    dom_bytes = ab[dom]
    dom_us = kern[dom]["avg_us"]
    achieved = dom_bytes / (dom_us * 1e-6) / 1e9
    traffic = args.traffic_bytes
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if traffic is None and tfile.exists():
        traffic = json.loads(tfile.read_text()).get(f"{args.config}:{dom}")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": dom_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6.65 TB/s"}
    # the tensor-core LCOM-CK of dense classes against the measured tcgen05 kind::i8
    # peak (tools/peaks.cu, profiles/r2_peaks.json)
    if "ck_mma" in kern:
        roofline["tensor"] = tensor_roofline(s, kern["ck_mma"]["avg_us"])
    # the metric pass: the lean-class kernel runs beside method + class pass when
    # both kinds of class exist, ahead of the class pass when every class is lean
    t_lean = kern.get("class_lean", {}).get("avg_us", 0.0)
    t_rest = sum(kern.get(k, {}).get("avg_us", 0.0) for k in ("method", "class_pass"))
    recompute_us = max(t_lean, t_rest) if "method" in kern else t_lean + t_rest

    # e2e through the public API: pinned host CSR -> H2D upload -> pass -> sweep -> D2H results
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, s, eng, dev, stream, n_cand, world, shard, gather if world > 1 else None)
        if e2e is not None and rank == 0 and world == 1 and args.config == "c4":
            e2e["cpp_dropin"] = cpp_dropin_e2e()

    cb = None
    ingest = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = cpu_baseline(args.config)
        if cb.get("suggestions") is not None and not cb.get("extrapolated") and world == 1:
            cb["same_list_length_as_gpu"] = int(cb["suggestions"]) == int(n_sugg_local)
        if args.config == "c4":
            ingest = ingest_bench(cfg)
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32+f64", "data": DATA,
            "config": bench_config(args.config, n_cand),
            "parallelism": f"dp{world} (class-range shards of the sweep, metric pass replicated, exact-count "
                           f"record exchange over NCCL)",
            "timing": "ms_per_step: K uninstrumented graph replays between CUDA events on the engine stream, max "
                      "over ranks; kernels: a second K-step pass with CUDA events around each kernel "
                      "(ms_per_step_instrumented)",
            "criteria": "cohesion+coupling, union, best-only, device mean thresholds",
            "roofline": roofline,
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
            "recompute_ms": recompute_us / 1e3,
            "sweep_ms": sum(kern.get(k, {}).get("avg_us", 0.0) for k in ("score", "offsets", "write")) / 1e3,
            "suggestions": int(n_sugg_local) if world == 1 else None,
            "kernels": kern,
            "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
            "ms_per_step_instrumented": float(np.mean(step_ms_prof)),
            "algorithmic_bytes": ab,
            "ingest": ingest,
        }
        print(json.dumps(out), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def ingest_bench(cfg):
    """Facts file -> device-ready CSR, host side, on this
    box: the config's canonical facts document (written by the product CLI's
    generator) parsed by mm_facts_load (C ABI, best of 3) against the
    reference's own parse_facts compiled in place (oracle/_ref/facts_parity
    --bench, the same C4 document; the reference single-threaded, ours with
    its parallel reader on min(16, cores) threads). Never fails the line."""
    import ctypes as C
    cli, harness = ROOT / "tools" / "_build" / "mmgpu", ROOT / "oracle" / "_ref" / "facts_parity"
    try:
        if not cli.exists():
            return {"unavailable": "tools/_build/mmgpu not built"}
        from paper_1308_4011_b200._lib import lib
        with tempfile.TemporaryDirectory() as d:
            path = Path(d) / "facts.json"
            subprocess.run([str(cli), "generate", "--classes", str(cfg["n_classes"]), "--methods", str(cfg["n_methods"]),
                            "--attributes", str(cfg["n_attributes"]), "--kmax-calls", str(cfg["k_max_calls"]),
                            "--kmax-accesses", str(cfg["k_max_accesses"]), "--intra-bias", str(cfg["intra_class_bias"]),
                            "--seed", str(cfg["seed"]), "--out", str(path)], check=True, timeout=300)
            size = path.stat().st_size
            best = float("inf")
            for _ in range(3):
                h = C.c_void_p()
                t0 = time.perf_counter()
                st = lib().mm_facts_load(str(path).encode(), C.byref(h))
                dt = time.perf_counter() - t0
                lib().mm_facts_free(h)
                if st != 0:
                    return {"error": f"mm_facts_load status {st}"}
                best = min(best, dt)
        threads = int(os.environ.get("MMGPU_FACTS_THREADS", min(16, os.cpu_count() or 1)))
        out = {"doc_mb": size / 1e6, "csr_load_s": best, "csr_mb_per_s": size / 1e6 / best, "threads": threads,
               "path": "mm_facts_load (file read + streaming parse + semantic checks + CSR)"}
        if harness.exists():
            r = subprocess.run([str(harness), "--bench"], capture_output=True, text=True, timeout=300)
            ref = json.loads(r.stdout.strip().splitlines()[-1])
            out["reference_parse_facts_s"] = ref["reference_parse_facts_s"]
            out["reference_kind"] = "reference parse_facts (nlohmann DOM + model walk), compiled in place, 1 thread"
            out["speedup_vs_reference"] = ref["reference_parse_facts_s"] / best
        return out
    except Exception as e:  # reported, never fatal
        return {"error": f"{type(e).__name__}: {e}"}


def run_e2e(args, s, eng, dev, stream, n_cand, world, shard, gather):
    import torch
    from paper_1308_4011_b200 import System
    # the step's inputs live in pinned host memory
    pinned = {}
    for f in ("method_owner", "attribute_owner", "class_method_off", "class_methods", "class_attr_off",
              "class_attrs", "call_off", "call_tgt", "acc_off", "acc_tgt"):
        a = getattr(s, f)
        t = torch.empty(a.size, dtype=torch.int32, pin_memory=True)
        t.numpy().view(np.uint32)[:] = a
        pinned[f] = t
    hs = System(s.n_classes, s.n_methods, s.n_attributes,
                **{f: t.numpy().view(np.uint32) for f, t in pinned.items()})
    # owner tables stay on the host: the device derives them from the
    # membership lists (mm_system contract), so they are not in the H2D bytes
    h2d = s.nbytes() - s.method_owner.nbytes - s.attribute_owner.nbytes
    d2h = [0]

    def e2e_step():
        eng.upload(hs, owner_tables=False)               # H2D from pinned host + device validation + plan
        eng.compute_metrics()
        if world == 1:
            lcom, ck, cbo = eng.class_metrics_async()      # D2H per-class metrics (pinned), under the sweep
            eng.sweep(thresholds=None, want_count=False)   # thresholds = device means of this pass
            recs = eng.suggestions(copy=False)             # D2H of the ordered list
            eng.synchronize()
        else:
            lcom, ck, cbo = eng.class_metrics_all(copy=False)
            eng.sweep(thresholds=None, class_range=shard, want_count=False)
            n_local = eng.sweep_stats()["suggestions"]
            allrec, counts = gather(n_local)
            recs = allrec.cpu().numpy()
        d2h[0] = lcom.nbytes + ck.nbytes + cbo.nbytes + (recs.nbytes if hasattr(recs, "nbytes") else 0)

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    torch.cuda.synchronize(dev)
    n = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(n):
        e2e_step()
    torch.cuda.synchronize(dev)
    dt = (time.perf_counter() - t0) / n
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    path = ("Engine.upload(pinned host CSR, owners derived on device) -> compute_metrics -> "
            "class_metrics_async (D2H under the sweep) -> sweep (device thresholds) -> suggestions (D2H)")
    out = {"value": n_cand / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h[0]),
           "ms_per_step": dt * 1e3, "steps": n, "latency_ms": dt * 1e3, "path": path}
    if world == 1 and not args.e2e_serial:
        # request pipelining, as a serving host runs it: several engines (
        # contexts with their own streams and device copies of the model),
        # each driven by its own host thread through the same public calls, so
        # one request's H2D overlaps the other's kernels and D2H (PCIe is full
        # duplex; the ctypes calls release the GIL). Every step still copies
        # its whole input from pinned host memory and reads its results back.
        import threading
        from paper_1308_4011_b200 import Engine
        extra = [Engine(dev.index if dev.index is not None else 0) for _ in range(max(1, args.e2e_engines) - 1)]
        engines = [eng] + extra
        counts = {}

        def request(e):
            e.upload(hs, owner_tables=False)
            e.compute_metrics()
            e.class_metrics_async()
            e.sweep(thresholds=None, want_count=False)
            recs = e.suggestions(copy=False)
            e.synchronize()
            counts[id(e)] = len(recs)

        for e in engines:
            request(e)
        n_each = max(2, min(args.steps, 10))
        gate = threading.Barrier(len(engines) + 1)

        def worker(e):
            gate.wait()
            for _ in range(n_each):
                request(e)

        ths = [threading.Thread(target=worker, args=(e,)) for e in engines]
        for th in ths:
            th.start()
        gate.wait()
        t0 = time.perf_counter()
        for th in ths:
            th.join()
        dtp = (time.perf_counter() - t0) / (len(engines) * n_each)
        for e in extra:
            e.close()
        if len(set(counts.values())) != 1:
            raise RuntimeError(f"pipelined e2e: engines disagree on the suggestion count {counts}")
        out.update({"value": n_cand / dtp, "ms_per_step": dtp * 1e3, "steps": len(engines) * n_each,
                    "serial_value": n_cand / dt, "engines": len(engines),
                    "path": path + f"; {len(engines)} engines on {len(engines)} host threads, requests pipelined "
                                   "(one request's H2D under another's kernels and D2H); latency_ms = one request alone"})
    return out


def ensure_world(args) -> None:
    """--gpus N means N ranks, one per GPU: under torchrun WORLD_SIZE must be
    N; run directly with N > 1 this process re-launches itself under
    torch.distributed.run (127.0.0.1) — or fails loudly when fewer than N GPUs
    are visible. Never a silent 1-GPU measurement."""
    _, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ:
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
        return
    if args.gpus <= 1:
        return
    if args.impl == "ours":
        import torch
        n_dev = torch.cuda.device_count()
        if n_dev < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {n_dev} CUDA device(s) are visible")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true", help="e2e without request pipelining (one engine)")
    ap.add_argument("--e2e-engines", type=int, default=3, help="engines (host threads) pipelining e2e requests")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from an ncu --set full capture")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    ensure_world(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
