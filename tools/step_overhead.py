"""Step-time decomposition at c3 (GPU box): device time per dynamic_step with and without per-kernel events,
the sum of the kernels' own times, and the host time per call -- the gap is launch/sync idle time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_14870_b200 as g
from paper_2103_14870_b200 import configs as cf

sim, mesh = cf.build_gpu(cf.get(sys.argv[1] if len(sys.argv) > 1 else "c3"))
K = 20
for prof in (False, True, False):
    sim.set_profiling(prof) if hasattr(sim, "set_profiling") else None
    for _ in range(3):
        sim.dynamic_step()
    sim.reset_kernel_times()
    sim.synchronize()
    sim.timer_record(0)
    t0 = time.perf_counter()
    for _ in range(K):
        sim.dynamic_step()
    t1 = time.perf_counter()
    sim.timer_record(1)
    ms = sim.timer_elapsed_ms(0, 1) / K
    kt = sim.kernel_times() if prof else {}
    ksum = sum(v["total_ms"] for v in kt.values()) / K
    print(f"profiling={prof}: device {ms:.4f} ms/step, host {1e3 * (t1 - t0) / K:.4f} ms/step"
          + (f", kernels {ksum:.4f} ms/step, gap {ms - ksum:.4f}" if prof else ""))
