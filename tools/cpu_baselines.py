"""CPU timing of the reference path (SURVEY.md 8d "CPU timing beside the GPU"),
all three modes, on this host (dev tool; oracle/ is the reference port):
  (i)   verification mode: config 1 (N=1024 H=256 I=688 V=4096, M=4), the f64
        SPEC restatement (sequential-K matmuls), single thread, best of 5;
  (ii)  the f32 port (oracle/mst_oracle.c) at Llama3-8B widths on a bounded
        token sample, one thread;
  (iii) the same on all host threads (OpenMP over output rows) — the bench's
        cpu_baseline / --impl reference arm.
Cost per token is independent of S, so (ii)/(iii) report tokens/s of the
sample.  Writes JSON lines to stdout."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from oracle import oracle

os.environ.setdefault("OMP_NUM_THREADS", "1")
c = oracle.make_inputs(1, 1024, 256, 688, 4096)
best = 1e30
for _ in range(5):
    t0 = time.perf_counter()
    out = oracle.block(c["X"], c["L"], c["Wg"], c["Wu"], c["Wd"], c["Wout"], 4, 4, round_bf16=False)
    best = min(best, time.perf_counter() - t0)
print(json.dumps({"mode": "(i) verification: config 1, f64 sequential-K, 1 thread, best of 5", "tokens": 1024,
                  "seconds": best, "tokens_per_s": 1024 / best, "loss": float(out["loss"])}), flush=True)
for nth, tokens in ((1, 32), (oracle.host_threads(), 256)):
    blk, _ = bench.cpu_block(tokens, 8, nth)
    blk.step()  # page-in
    t0 = time.perf_counter()
    loss = blk.step()
    dt = time.perf_counter() - t0
    print(json.dumps({"mode": f"({'ii' if nth == 1 else 'iii'}) f32 port at Llama3-8B widths, {nth} thread(s)",
                      "tokens": tokens, "seconds": dt, "tokens_per_s": tokens / dt,
                      "executed_tflops": tokens * bench.model_flops_per_token() / dt / 1e12, "loss": loss}), flush=True)
