"""A/B timing harness (development tool, not the bench): one config, several
environment variants, each in its own process; prints the step time (graph
replays between CUDA events) and the per-kernel event times.

    python tools/kbench.py --config c4 --steps 20 VAR=1,VAR2=0 ...   ('-' = no extra env)"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(config: str, steps: int):
    sys.path.insert(0, str(ROOT))
    import torch
    import bench
    from paper_1308_4011_b200 import Engine, System
    s = System.generate(**bench.CONFIGS[config])
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    e = Engine(0, stream=st.cuda_stream)
    e.upload(s)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    for _ in range(5):
        e.run(thresholds=None)
    torch.cuda.synchronize()

    def timed(prof):
        ts = []
        for i in range(steps):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            e.run(thresholds=None)
            b.record(st)
            if prof:
                e.collect_timings()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return ts

    plain = timed(False)
    e.set_profiling(True)
    for _ in range(2):
        e.run(thresholds=None)
    torch.cuda.synchronize()
    e.reset_kernel_stats()
    prof = timed(True)
    k = {n: round(1e3 * ms / c, 1) for n, (c, ms) in e.kernel_stats().items() if c}
    st_ = e.sweep_stats()
    print(json.dumps({"step_us": round(1e3 * sorted(plain)[len(plain) // 2], 1), "step_us_min": round(1e3 * min(plain), 1),
                      "prof_step_us": round(1e3 * sorted(prof)[len(prof) // 2], 1), "kernels_us": k,
                      "suggestions": st_["suggestions"]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("variants", nargs="*", default=["-"])
    a = ap.parse_args()
    if a.child:
        child(a.config, a.steps)
        return
    for v in a.variants:
        env = dict(os.environ)
        if v != "-":
            for kv in v.split(","):
                k, val = kv.split("=", 1)
                env[k] = val
        r = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--steps", str(a.steps)],
                           env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
        print(f"{a.config} [{v}] {line}", flush=True)


if __name__ == "__main__":
    main()
