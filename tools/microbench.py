"""BASELINE.json configs[4]: kernel micro-benchmark sweep (GPU box).

Cubic 6-tet-per-hex grids n^3 (n = 26, 55, 94, 149 -> 1e5, 1e6, 5e6, 2e7 tets), node displacements uniform in
+-5% of the cell size (seeded), pre-damaged edge fractions 0 / 10 / 50 % (seeded), chi from the damage pass.
Per kernel: device time (CUDA events), algorithmic GB/s (SURVEY §8d byte formulas) and the fraction of the
measured HBM copy peak; next to it the CPU oracle's time for the same operation (sizes <= 1e6 tets).

  python tools/microbench.py [--sizes 26,55,94,149] [--reps 20] > profiles/r01_micro.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2103_14870_b200 as g

H = 0.01


def peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="26,55,94,149")
    ap.add_argument("--fractions", default="0,0.1,0.5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu-max-tets", type=int, default=1_100_000)
    args = ap.parse_args()
    pk = peak()
    for n in [int(x) for x in args.sizes.split(",")]:
        mesh = g.make_box_mesh((n * H,) * 3, (n, n, n))
        N, T, E = mesh.num_nodes(), mesh.num_tets(), mesh.num_edges()
        nd = 3 * N
        mat = g.MaterialParams.from_youngs(1e6, 0.3, 1000.0, 2e4, 0.0, g.STABLE_NEO_HOOKEAN)
        sim = g.Simulation(mesh, mat, g.SolverConfig(dt=1e-3))
        rng = np.random.default_rng(n)
        u = rng.uniform(-0.05 * H, 0.05 * H, (N, 3))
        Z = 9 * (N + 2 * E)
        info = sim.info()
        for frac in [float(x) for x in args.fractions.split(",")]:
            zeta = (rng.uniform(0, 1, E) < frac).astype(np.uint8)
            sim.set_state(displacements=u, velocities=np.zeros((N, 3)), edge_damage=zeta, element_chi=np.ones(T))
            sim.damage_pass()  # chi consistent with the pre-damage (compute_chi semantics)
            st = sim.state()
            try:
                sim.dynamic_step()  # assembles the system matrix for the SpMV timing
            except g.SolveError:
                pass  # random displacements can make A indefinite; the assembled matrix is all the SpMV needs
            sim.set_state(displacements=u, velocities=np.zeros((N, 3)), edge_damage=st.edge_damage,
                          element_chi=st.element_chi)
            sim.set_profiling(True)
            sim.reset_kernel_times()
            x = rng.uniform(-1, 1, nd)
            for _ in range(args.reps):
                sim.eval_forces()
                sim.set_state(edge_damage=st.edge_damage, element_chi=st.element_chi)
                sim.damage_pass()
                sim.spmv(x)
            kt = sim.kernel_times()
            sim.set_profiling(False)
            rows = {
                "force": ("forces", 16 * nd + 104 * T),
                "damage_stress": ("tet_stress", 16 * nd + 112 * T + 8 * E),
                "relabel": ("relabel", 2 * E),
                "chi": ("chi", 16 * T),
                # the symmetric SELL-32 format's bytes (every stored upper block once, the slot words, x gathered and y
                # written); the SURVEY scalar-CSR model 12Z + 4(n+1) + 16n is reported next to it (it overstates this
                # format's traffic: a "fraction" above 1 under it is not an HBM rate)
                "spmv": ("spmv", 72 * info["upper_blocks"] + 4 * info["spmv_slots"] + 48 * N),
            }
            survey_spmv = 12 * Z + 4 * (nd + 1) + 16 * nd
            out = {"n": n, "tets": T, "nodes": N, "edges": E, "predamage": frac, "peak_gbs": pk, "kernels": {}}
            for key, (name, nbytes) in rows.items():
                if name not in kt:
                    continue
                ms = kt[name]["total_ms"] / kt[name]["launches"]
                out["kernels"][key] = {"ms": ms, "GBps": nbytes / ms / 1e6, "frac_of_peak": nbytes / ms / 1e6 / pk,
                                       "algorithmic_bytes": nbytes}
                if key == "spmv":
                    out["kernels"][key]["survey_model_GBps"] = survey_spmv / ms / 1e6
            if T <= args.cpu_max_tets:
                from oracle import oracle as o
                om = o.Mesh.make_box((n * H,) * 3, (n, n, n))
                omat = o.material_from_youngs(1e6, 0.3, 1000.0, 2e4, 0.0, 0)
                chi = st.element_chi
                t0 = time.perf_counter()
                om.assemble_forces(omat, u, chi)
                t1 = time.perf_counter()
                sig = om.per_tet_cauchy(omat, u)
                scr, sf, deg = om.nonlocal_screen(u, sig, 0.0)
                o.update_damage(st.edge_damage, scr, 2e4)
                t2 = time.perf_counter()
                rp, cols, _ = om.pattern()
                vals = np.ones(len(cols))
                t3 = time.perf_counter()
                o.spmv_csr(rp, cols, vals, x)
                t4 = time.perf_counter()
                out["cpu_oracle_ms"] = {"force": 1e3 * (t1 - t0), "damage_pass": 1e3 * (t2 - t1),
                                        "spmv": 1e3 * (t4 - t3), "threads": o.num_threads()}
            print(json.dumps(out), flush=True)
        sim.close()


if __name__ == "__main__":
    main()
