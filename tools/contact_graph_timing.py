"""Contact step timing, host-driven detection vs one captured graph per step: the reference's
acceptance criterion #6 scene (two 7^3 cubes, 2000:1 mass ratio, n_max 25, 240 steps)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06321_b200 as V


def scene(precision):
    n = 7
    stiff = V.MaterialParams(mu=1e6, lam=1e7)
    light = V.generate_beam(n, n, n, 0.5 / (n - 1), density=10.0)
    rho_heavy = 2000.0 * light.masses.sum() / 0.4 ** 3
    heavy0 = V.generate_beam(n, n, n, 0.4 / (n - 1), density=rho_heavy)
    heavy = V.build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.5005], heavy0.tets, rho_heavy)
    bottom = np.flatnonzero(light.rest_positions[:, 2] < 1e-9)
    system = V.build_system([V.Body(light, stiff, k_d=0.01), V.Body(heavy, stiff, k_d=0.01)],
                            [V.FixedConstraint(int(i)) for i in bottom])
    params = V.SolverParams(h=1.0 / 120.0, n_max=25, a_ext=(0, 0, -9.8), precision=precision,
                            contact=V.ContactParams(k_c=1e7, mu_c=1.0, eps_v=1e-3, dcd_radius=0.008))
    return system, params


for precision in ("fp64", "fp32"):
    for mode in ("0", "1"):
        os.environ["VBD_CONTACT_GRAPH"] = mode
        system, params = scene(precision)
        state = V.make_state(system)
        V.step(state, params)  # first step (host path, sizes the capacities)
        V.step(state, params)
        _ = state.x
        t = time.perf_counter()
        for _ in range(240):
            V.step(state, params)
        _ = state.x
        dt = (time.perf_counter() - t) / 240 * 1e3
        info = state._ctx._info()
        print(f"{precision} contact graph={mode}: {dt:.3f} ms/step (wall, incl. the per-step result read); "
              f"graph steps {info.contact_graph_steps}, fallbacks {info.contact_graph_fallbacks}", flush=True)
