"""Full-length trajectory parity of a BASELINE config: GPU path vs CPU oracle, step by step (GPU box).

Positions must agree within 1e-6 relative (north_star). Edge labels must agree exactly; a label that differs
is accepted only if the oracle's screening value for that edge lies within --flip-tol of the threshold (a
rounding-level flip caused by the CG's different summation order), after which the GPU state is re-seeded from
the oracle ("label-sync", SURVEY §7 hard part 7). Prints one JSON line.

  python tools/trajectory.py c2 [--steps 300]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2103_14870_b200 import configs as cf
from oracle.scenario import build_oracle, near_threshold_flips


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--flip-tol", type=float, default=1e-6)
    args = ap.parse_args()
    s = cf.get(args.config)
    steps = args.steps or s.steps
    gs, gm = cf.build_gpu(s)
    os_, om = build_oracle(s)
    X = om.arrays()["rest"]
    scale = np.abs(X).max()
    worst_u, worst_v, resyncs, flips, t_cpu, t_gpu = 0.0, 0.0, 0, 0, 0.0, 0.0
    cg_g, cg_o = 0, 0
    worst_flip, bad_flips = 0.0, 0
    for k in range(steps):
        u_pre = os_.get_state()["u"]
        t0 = time.perf_counter()
        a = os_.dynamic_step()
        t1 = time.perf_counter()
        b = gs.dynamic_step()
        t2 = time.perf_counter()
        t_cpu += t1 - t0
        t_gpu += t2 - t1
        cg_o += a.cg_iterations
        cg_g += b.cg_iterations
        ost, gst = os_.get_state(), gs.state()
        if not np.array_equal(gst.edge_damage, ost["zeta"]):
            diff = np.nonzero(gst.edge_damage != ost["zeta"])[0]
            # each differing label must be a near-threshold decision of the damage pass (oracle screening from the
            # pre-step state within --flip-tol x sigma_thres of the threshold); anything else fails the run
            ok, dist = near_threshold_flips(om, os_.mat, u_pre, s.r_d, s.sigma_thres, diff, args.flip_tol)
            worst_flip = max(worst_flip, dist)
            bad_flips += 0 if ok else len(diff)
            resyncs += 1
            flips += len(diff)
            gs.set_state(ost["u"], ost["v"], ost["zeta"], ost["chi"], ost["time"])
            continue
        worst_u = max(worst_u, np.abs(gst.displacements - ost["u"]).max() / scale)
        vs = max(1.0, np.abs(ost["v"]).max())
        worst_v = max(worst_v, np.abs(gst.velocities - ost["v"]).max() / vs)
    ost = os_.get_state()
    out = dict(config=s.name, tets=s.num_tets, steps=steps, max_rel_position_err=worst_u, max_rel_velocity_err=worst_v,
               label_resyncs=resyncs, flipped_labels=flips, flips_beyond_tol=bad_flips,
               max_flip_distance_rel=worst_flip, flip_tol=args.flip_tol, broken_edges=int(ost["zeta"].sum()),
               cg_iterations_gpu=cg_g, cg_iterations_oracle=cg_o, wall_s_oracle=t_cpu, wall_s_gpu=t_gpu,
               passed=bool(worst_u < 1e-6 and bad_flips == 0))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
