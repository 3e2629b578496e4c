"""Scene documents, frame files and the simulation runner (pkg/src/vbdsim/harness.py:95-691).

A scene is one JSON document: bodies from generators (beam, cube, chain, file) placed by a
rigid modelling transform, gravity, optional contact, constraints, solver settings, frame
count and output format.  ``parse_scene`` validates it with the reference's error contract:
structural problems (unknown key, wrong type, missing key, bad JSON) raise ``SchemaError``
carrying the key path; value-range problems raise ``ValueError`` prefixed with the same path.
Defaults follow harness.py:345-353 (h = 1/(60 S), n_max 10, n_col 4, ...).

``run_simulation`` steps the scene on the GPU.  The per-iteration metric columns (G, active
contact count, max penetration; harness.py:664-678) come from one device reduction per
iteration (``vbd_energy_metrics``) at the resident iterate, so x never leaves the device
between frames; ``metrics="off"`` runs each step as one CUDA graph instead.  Frames are read
back only when written.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from .backend import NAME as _BACKEND
from .errors import SchemaError
from .materials import MaterialParams
from .mesh import (TetMesh, build_spring_net, build_tet_mesh, generate_beam, generate_chain,
                   generate_cube, load_node_ele)
from .solver import ContactParams, SolverParams, make_state, metrics, step
from .system import Body, FixedConstraint, SubspaceConstraint, WorldBoxConstraint, build_system

METRICS_HEADER = "step,iteration,G,relative_loss,contact_count,max_penetration,wall_ms"
FRAME_FORMATS = ("bin", "obj")
_REQUIRED = object()


# ------------------------------------------------------------------------------------------
# typed reads with key paths (harness.py:120-172)

def _is_num(v):
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _as_number(v, path):
    if not _is_num(v):
        raise SchemaError(path, "expected a number")
    return float(v)


def _as_int(v, path):
    if not isinstance(v, int) or isinstance(v, bool):
        raise SchemaError(path, "expected an integer")
    return int(v)


def _as_vec3(v, path):
    if not isinstance(v, (list, tuple)) or len(v) != 3:
        raise SchemaError(path, "expected [x, y, z]")
    if not all(_is_num(c) for c in v):
        raise SchemaError(path, "expected numeric components")
    return tuple(float(c) for c in v)


def _as_str(v, path):
    if not isinstance(v, str):
        raise SchemaError(path, "expected a path string")
    return v


def _positive(v, path):
    if v <= 0.0:
        raise ValueError(f"{path}: must be positive")


def _nonneg(v, path):
    if v < 0.0:
        raise ValueError(f"{path}: must be >= 0")


def _at_least(k):
    def check(v, path):
        if v < k:
            raise ValueError(f"{path}: must be >= {k}")
    return check


class _Block:
    """One JSON object of the scene with its key path and allowed key set."""

    def __init__(self, d, path, allowed):
        if not isinstance(d, dict):
            raise SchemaError(path, "expected an object")
        for k in d:
            if k not in allowed:
                raise SchemaError(f"{path}.{k}", "unknown key")
        self.d, self.path = d, path

    def key(self, k):
        return f"{self.path}.{k}"

    def read(self, k, conv, default=_REQUIRED, check=None):
        if k not in self.d:
            if default is _REQUIRED:
                raise SchemaError(self.key(k), "missing required key")
            return default
        v = conv(self.d[k], self.key(k))
        if check is not None:
            check(v, self.key(k))
        return v

    def vec(self, k, default=_REQUIRED, each=None):
        v = self.read(k, _as_vec3, default)
        if each is not None and v is not None:
            for c in v:
                each(c, self.key(k))
        return v


# ------------------------------------------------------------------------------------------
# scene configuration

@dataclass
class ObjectConfig:
    generator: dict
    material: MaterialParams
    density: float
    translate: tuple
    rotate_deg: tuple
    scale: tuple
    velocity: tuple
    initial_stretch: tuple


@dataclass
class OutputConfig:
    format: str = "bin"
    every: int = 1


@dataclass
class SceneConfig:
    objects: list
    constraints: list
    solver: SolverParams
    frames: int
    output: OutputConfig


# generator kind -> [(key, converter, default, check)]  (harness.py:183-229)
_GENERATORS = {
    "beam": [("nx", _as_int, _REQUIRED, _at_least(2)), ("ny", _as_int, _REQUIRED, _at_least(2)),
             ("nz", _as_int, _REQUIRED, _at_least(2)), ("spacing", _as_number, _REQUIRED, _positive)],
    "cube": [("n", _as_int, _REQUIRED, _at_least(2)), ("edge", _as_number, _REQUIRED, _positive)],
    "chain": [("count", _as_int, _REQUIRED, _at_least(2)),
              ("spacing", _as_number, _REQUIRED, _positive),
              ("stiffness", _as_number, _REQUIRED, _positive),
              ("mass", _as_number, 1.0, _positive)],
    "file": [("node", _as_str, _REQUIRED, None), ("ele", _as_str, _REQUIRED, None)],
}

# constraint kind -> allowed keys (harness.py:272-276)
_CONSTRAINTS = {
    "fixed": {"kind", "object", "vertices", "box"},
    "subspace": {"kind", "object", "vertex", "basis", "anchor"},
    "world_box": {"kind", "object", "lo", "hi", "k_b"},
}

_SOLVER_KEYS = {"h", "S", "n_max", "n_col", "rho", "eps_det", "line_search", "init_mode",
                "threads", "precision"}


def _parse_generator(d, path):
    if not isinstance(d, dict):
        raise SchemaError(path, "expected an object")
    kind = d.get("kind")
    if kind not in _GENERATORS:
        raise SchemaError(f"{path}.kind", f"expected one of {sorted(_GENERATORS)}")
    fields = _GENERATORS[kind]
    b = _Block(d, path, {"kind"} | {f[0] for f in fields})
    out = {"kind": kind}
    for name, conv, default, check in fields:
        out[name] = b.read(name, conv, default, check)
    return out


def _parse_material(d, path):
    b = _Block(d, path, {"mu", "lambda", "k_d"})
    return MaterialParams(mu=b.read("mu", _as_number, check=_positive),
                          lam=b.read("lambda", _as_number, check=_positive),
                          k_d=b.read("k_d", _as_number, 0.0, _nonneg))


def _parse_object(d, i):
    path = f"objects[{i}]"
    b = _Block(d, path, {"generator", "material", "density", "translate", "rotate_deg", "scale",
                         "velocity", "initial_stretch"})
    if "generator" not in d:
        raise SchemaError(b.key("generator"), "missing required key")
    gen = _parse_generator(d["generator"], b.key("generator"))
    material = _parse_material(d["material"], b.key("material")) if "material" in d else None
    if material is None and gen["kind"] != "chain":
        raise SchemaError(b.key("material"), "missing required key")
    scale = d.get("scale", 1.0)
    if _is_num(scale):
        scale = (float(scale),) * 3
    else:
        scale = b.vec("scale", (1.0, 1.0, 1.0))
    for c in scale:
        _positive(c, b.key("scale"))
    return ObjectConfig(
        generator=gen, material=material,
        density=b.read("density", _as_number, 1000.0, _positive),
        translate=b.vec("translate", (0.0, 0.0, 0.0)),
        rotate_deg=b.vec("rotate_deg", (0.0, 0.0, 0.0)),
        scale=tuple(scale),
        velocity=b.vec("velocity", (0.0, 0.0, 0.0)),
        initial_stretch=b.vec("initial_stretch", None, each=_positive))


def _parse_constraint(d, i, n_objects):
    path = f"constraints[{i}]"
    if not isinstance(d, dict):
        raise SchemaError(path, "expected an object")
    kind = d.get("kind")
    if kind not in _CONSTRAINTS:
        raise SchemaError(f"{path}.kind", f"expected one of {sorted(_CONSTRAINTS)}")
    b = _Block(d, path, _CONSTRAINTS[kind])
    obj = d.get("object", "all" if kind == "world_box" else None)
    if not (kind == "world_box" and obj == "all"):
        if not isinstance(obj, int) or isinstance(obj, bool):
            raise SchemaError(b.key("object"), "expected an object index")
        if not 0 <= obj < n_objects:
            raise SchemaError(b.key("object"), f"object index out of range [0,{n_objects})")
    out = {"kind": kind, "object": obj}
    if kind == "fixed":
        if ("vertices" in d) == ("box" in d):
            raise SchemaError(path, "exactly one of vertices/box required")
        if "vertices" in d:
            v = d["vertices"]
            if not isinstance(v, list) or not all(isinstance(k, int) and not isinstance(k, bool)
                                                  for k in v):
                raise SchemaError(b.key("vertices"), "expected a list of vertex indices")
            out["vertices"] = [int(k) for k in v]
        else:
            box = d["box"]
            if not isinstance(box, list) or len(box) != 2:
                raise SchemaError(b.key("box"), "expected [lo, hi]")
            out["box"] = (_as_vec3(box[0], b.key("box.lo")), _as_vec3(box[1], b.key("box.hi")))
    elif kind == "subspace":
        out["vertex"] = b.read("vertex", _as_int)
        rows = d.get("basis")
        if not isinstance(rows, list) or len(rows) not in (1, 2):
            raise SchemaError(b.key("basis"), "expected 1 or 2 direction rows")
        for r in rows:
            if not isinstance(r, list) or len(r) != 3 or not all(_is_num(c) for c in r):
                raise SchemaError(b.key("basis"), "expected 3-vectors")
        out["basis"] = np.asarray(rows, dtype=np.float64).T  # (3, L) columns
        out["anchor"] = b.vec("anchor", None)
    else:
        out["lo"] = b.vec("lo")
        out["hi"] = b.vec("hi")
        out["k_b"] = b.read("k_b", _as_number, check=_positive)
    return out


def _parse_contact(d):
    b = _Block(d, "contact", {"k_c", "mu_c", "eps_v", "dcd_radius", "max_depth"})
    return ContactParams(k_c=b.read("k_c", _as_number, check=_positive),
                         mu_c=b.read("mu_c", _as_number, 0.0, _nonneg),
                         eps_v=b.read("eps_v", _as_number, 1e-2, _positive),
                         dcd_radius=b.read("dcd_radius", _as_number, 1e-3, _nonneg),
                         max_depth=b.read("max_depth", _as_number, None, _positive))


def _unit_interval(v, path):
    if not 0.0 <= v < 1.0:
        raise ValueError(f"{path}: must be in [0, 1)")


def _choice(options, message):
    def conv(v, path):
        if v not in options:
            raise SchemaError(path, message)
        return v
    return conv


def _parse_solver(d, gravity, contact):
    b = _Block(d, "solver", _SOLVER_KEYS)
    substeps = b.read("S", _as_int, 1, _at_least(1))
    return SolverParams(
        h=b.read("h", _as_number, 1.0 / (60.0 * substeps), _positive),
        substeps=substeps,
        n_max=b.read("n_max", _as_int, 10, _at_least(1)),
        n_col=b.read("n_col", _as_int, 4, _at_least(1)),
        rho=b.read("rho", _as_number, 0.0, _unit_interval),
        eps_det=b.read("eps_det", _as_number, 1e-10, _nonneg),
        line_search=b.read("line_search", _choice(("off", "local_backtracking"),
                                                  "expected 'off' or 'local_backtracking'"),
                           "off") == "local_backtracking",
        init_mode=b.read("init_mode", _choice(("prev_pos", "inertia", "inertia_accel", "adaptive"),
                                              "unknown warm start mode"), "adaptive"),
        a_ext=gravity,
        threads=b.read("threads", _as_int, 0, _at_least(0)),
        contact=contact,
        precision=b.read("precision", _choice(("fp64", "fp32"), "expected 'fp64' or 'fp32'"),
                         "fp64"))


def parse_scene(text: str) -> SceneConfig:
    """Parse and validate a scene JSON document (harness.py:377-412).  ``solver.precision``
    ("fp64" default, "fp32") is this package's one schema extension."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SchemaError("$", f"invalid JSON ({e})") from None
    top = _Block(doc, "$", {"objects", "gravity", "constraints", "contact", "solver", "frames",
                            "output"})
    objs = doc.get("objects")
    if not isinstance(objs, list) or not objs:
        raise SchemaError("$.objects", "expected a non-empty list")
    objects = [_parse_object(o, i) for i, o in enumerate(objs)]
    gravity = top.vec("gravity", (0.0, 0.0, 0.0))
    contact = _parse_contact(doc["contact"]) if "contact" in doc else None
    solver = _parse_solver(doc.get("solver", {}), gravity, contact)
    cons = doc.get("constraints", [])
    if not isinstance(cons, list):
        raise SchemaError("$.constraints", "expected a list")
    constraints = [_parse_constraint(c, i, len(objects)) for i, c in enumerate(cons)]
    frames = top.read("frames", _as_int, 60, _at_least(0))
    out = _Block(doc.get("output", {}), "output", {"format", "every"})
    fmt = out.read("format", _choice(FRAME_FORMATS, "expected 'bin' or 'obj'"), "bin")
    every = out.read("every", _as_int, 1, _at_least(1))
    return SceneConfig(objects, constraints, solver, frames, OutputConfig(fmt, every))


def serialize_scene(config: SceneConfig) -> str:
    """Inverse of parse_scene up to key order and defaults (harness.py:415-470); the text equals
    the reference's for scenes without the precision extension."""
    p = config.solver
    solver = {"h": p.h, "S": p.substeps, "n_max": p.n_max, "n_col": p.n_col, "rho": p.rho,
              "eps_det": p.eps_det, "line_search": "local_backtracking" if p.line_search else "off",
              "init_mode": p.init_mode, "threads": p.threads}
    if p.precision != "fp64":
        solver["precision"] = p.precision
    doc = {"objects": [], "gravity": list(p.a_ext), "constraints": [], "solver": solver,
           "frames": config.frames,
           "output": {"format": config.output.format, "every": config.output.every}}
    if p.contact is not None:
        c = p.contact
        doc["contact"] = {"k_c": c.k_c, "mu_c": c.mu_c, "eps_v": c.eps_v,
                          "dcd_radius": c.dcd_radius}
        if c.max_depth is not None:
            doc["contact"]["max_depth"] = c.max_depth
    for o in config.objects:
        od = {"generator": dict(o.generator), "density": o.density, "translate": list(o.translate),
              "rotate_deg": list(o.rotate_deg), "scale": list(o.scale),
              "velocity": list(o.velocity)}
        if o.material is not None:
            od["material"] = {"mu": o.material.mu, "lambda": o.material.lam, "k_d": o.material.k_d}
        if o.initial_stretch is not None:
            od["initial_stretch"] = list(o.initial_stretch)
        doc["objects"].append(od)
    for c in config.constraints:
        cd = {"kind": c["kind"], "object": c["object"]}
        if c["kind"] == "fixed":
            if "vertices" in c:
                cd["vertices"] = list(c["vertices"])
            else:
                cd["box"] = [list(c["box"][0]), list(c["box"][1])]
        elif c["kind"] == "subspace":
            cd["vertex"] = c["vertex"]
            cd["basis"] = np.asarray(c["basis"]).T.tolist()
            if c["anchor"] is not None:
                cd["anchor"] = list(c["anchor"])
        else:
            cd.update(lo=list(c["lo"]), hi=list(c["hi"]), k_b=c["k_b"])
        doc["constraints"].append(cd)
    return json.dumps(doc, indent=2, sort_keys=True)


# ------------------------------------------------------------------------------------------
# scene -> system (harness.py:475-575)

def rotation_matrix(rotate_deg) -> np.ndarray:
    """R = Rz Ry Rx for XYZ Euler angles in degrees (harness.py:475-484)."""
    ax, ay, az = np.radians(rotate_deg)

    def axis_rot(i, a):
        r = np.eye(3)
        j, k = (i + 1) % 3, (i + 2) % 3
        c, s = np.cos(a), np.sin(a)
        r[j, j], r[j, k], r[k, j], r[k, k] = c, -s, s, c
        return r

    return axis_rot(2, az) @ axis_rot(1, ay) @ axis_rot(0, ax)


def _geometry(o: ObjectConfig):
    g = o.generator
    kind = g["kind"]
    if kind == "beam":
        base = generate_beam(g["nx"], g["ny"], g["nz"], g["spacing"], o.density)
    elif kind == "cube":
        base = generate_cube(g["n"], g["edge"], o.density)
    elif kind == "file":
        base = build_tet_mesh(*load_node_ele(g["node"], g["ele"]), o.density)
    else:
        base = generate_chain(g["count"], g["spacing"], g["stiffness"], g["mass"])
    rot = rotation_matrix(o.rotate_deg)
    scale = np.asarray(o.scale)

    def place(p):
        return (np.asarray(p) * scale) @ rot.T + np.asarray(o.translate)

    if isinstance(base, TetMesh):
        geometry = build_tet_mesh(place(base.rest_positions), base.tets, o.density)
        rest = geometry.rest_positions
    else:  # springs keep their topology; rest lengths scale by the mean scale factor
        rows = np.column_stack([base.indices.astype(np.float64),
                                base.rest_length * np.mean(scale), base.stiffness])
        geometry = build_spring_net(place(base.particles), rows, base.masses)
        rest = geometry.particles
    x0 = np.array(rest)
    if o.initial_stretch is not None:
        c = rest.mean(axis=0)
        x0 = c + (x0 - c) * np.asarray(o.initial_stretch)
    v0 = np.broadcast_to(np.asarray(o.velocity), rest.shape).copy()
    return geometry, np.asarray(rest), x0, v0


def _scene_constraints(config, rests, offsets):
    out = []
    for c in config.constraints:
        kind, obj = c["kind"], c["object"]
        if kind == "world_box":
            span = range(offsets[-1]) if obj == "all" else range(offsets[obj], offsets[obj + 1])
            out.extend(WorldBoxConstraint(v, c["lo"], c["hi"], c["k_b"]) for v in span)
            continue
        base, n_local = offsets[obj], offsets[obj + 1] - offsets[obj]
        if kind == "fixed":
            if "vertices" in c:
                verts = c["vertices"]
                bad = [v for v in verts if not 0 <= v < n_local]
                if bad:
                    raise ValueError(f"constraints: vertex {bad[0]} outside object {obj} "
                                     f"with {n_local} vertices")
            else:
                lo, hi = (np.asarray(b) for b in c["box"])
                inside = ((rests[obj] >= lo) & (rests[obj] <= hi)).all(axis=1)
                verts = np.flatnonzero(inside).tolist()
            out.extend(FixedConstraint(base + v) for v in verts)
        else:
            v = c["vertex"]
            if not 0 <= v < n_local:
                raise ValueError(f"constraints: vertex {v} outside object {obj}")
            anchor = c["anchor"] if c["anchor"] is not None else rests[obj][v]
            out.append(SubspaceConstraint(base + v, c["basis"], anchor))
    return out


def scene_build(config: SceneConfig):
    """Compile a parsed scene into (system, state, params) (harness.py:521-574): the packed
    system is colour-partitioned on the device; the state starts host-side and is uploaded by
    the first step."""
    bodies, rests, x0, v0, offsets = [], [], [], [], [0]
    for o in config.objects:
        geometry, rest, x, v = _geometry(o)
        bodies.append(Body(geometry, o.material))
        rests.append(rest)
        x0.append(x)
        v0.append(v)
        offsets.append(offsets[-1] + len(x))
    system = build_system(bodies, _scene_constraints(config, rests, offsets),
                          device=config.solver.device)
    state = make_state(system, np.concatenate(x0), np.concatenate(v0))
    return system, state, config.solver


# ------------------------------------------------------------------------------------------
# frames (harness.py:580-621)

def export_frame(positions, faces, path) -> None:
    """Write one frame; the suffix picks the format.  ``.bin``: little-endian u32 nv, u32 nf,
    nv*3 f64 positions, nf*3 u32 face indices.  ``.obj``: text, repr-exact doubles, 1-based
    faces."""
    path = Path(path)
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    fac = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
    if path.suffix == ".bin":
        blob = b"".join((np.array([len(pos), len(fac)], dtype="<u4").tobytes(),
                         pos.astype("<f8").tobytes(), fac.astype("<u4").tobytes()))
        path.write_bytes(blob)
    elif path.suffix == ".obj":
        out = [f"v {a!r} {b!r} {c!r}" for a, b, c in pos.tolist()]
        out += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in fac.tolist()]
        path.write_text("\n".join(out) + "\n")
    else:
        raise ValueError(f"unknown frame format {path.suffix!r}")


def load_frame(path):
    """Read a frame written by export_frame: (positions (nv,3) f64, faces (nf,3) i64)."""
    path = Path(path)
    if path.suffix == ".bin":
        blob = path.read_bytes()
        nv, nf = (int(k) for k in np.frombuffer(blob, dtype="<u4", count=2))
        pos = np.frombuffer(blob, dtype="<f8", count=3 * nv, offset=8).reshape(-1, 3)
        fac = np.frombuffer(blob, dtype="<u4", count=3 * nf, offset=8 + 24 * nv).reshape(-1, 3)
        return pos.astype(np.float64), fac.astype(np.int64)
    if path.suffix == ".obj":
        pos, fac = [], []
        for line in path.read_text().splitlines():
            f = line.split()
            if f and f[0] == "v":
                pos.append([float(c) for c in f[1:4]])
            elif f and f[0] == "f":
                fac.append([int(c.split("/")[0]) - 1 for c in f[1:4]])
        return (np.asarray(pos, dtype=np.float64).reshape(-1, 3),
                np.asarray(fac, dtype=np.int64).reshape(-1, 3))
    raise ValueError(f"unknown frame format {path.suffix!r}")


def surface_faces(system) -> np.ndarray:
    """Boundary triangles of the tet bodies in global vertex ids (harness.py:627-630)."""
    if system.collision_mesh is None:
        return np.zeros((0, 3), dtype=np.int64)
    return system.collision_map[system.collision_mesh.surface_tris]


# ------------------------------------------------------------------------------------------
# runner (harness.py:637-691)

def _g(v) -> str:
    return repr(float(v))


def run_simulation(config: SceneConfig, out_dir, threads=None, frames=None, metrics_mode="iteration"):
    """Step the scene and write frame files plus ``metrics.csv``; returns a summary dict.

    ``metrics_mode="iteration"`` (default) records one CSV row per solver iteration as the
    reference does: G, the active contact count and the max penetration from one device
    reduction at the resident iterate, relative_loss = (G_n - G_last)/(G_1 - G_last) within the
    step (0 when the step made no progress), wall_ms since the step began.  ``"off"`` writes the
    header only and runs every step as one CUDA graph.  ``threads`` is accepted for API
    compatibility (the sweep runs on the GPU)."""
    if metrics_mode not in ("iteration", "off"):
        raise ValueError("metrics_mode must be 'iteration' or 'off'")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    system, state, params = scene_build(config)
    if threads is not None:
        params = replace(params, threads=threads)
    n_frames = config.frames if frames is None else frames
    faces = surface_faces(system)
    fmt, every = config.output.format, config.output.every
    t_start = time.perf_counter()
    export_frame(state.x, faces, out / f"frame_00000.{fmt}")
    written = 1
    csv_path = out / "metrics.csv"
    with open(csv_path, "w") as fh:
        fh.write(METRICS_HEADER + "\n")
        for frame in range(n_frames):
            for _ in range(params.substeps):
                if metrics_mode == "off":
                    step(state, params)
                    continue
                rows, t0 = [], time.perf_counter()

                def record(st, n):
                    g, nc, pen = metrics(st, params)
                    rows.append((st.step_index, n, g, nc, pen, (time.perf_counter() - t0) * 1e3))

                step(state, params, on_iteration=record)
                g_first, g_last = rows[0][2], rows[-1][2]
                span = g_first - g_last
                for s, n, g, nc, pen, ms in rows:
                    loss = (g - g_last) / span if span > 0 else 0.0
                    fh.write(f"{s},{n},{_g(g)},{_g(loss)},{nc},{_g(pen)},{ms:.3f}\n")
            if (frame + 1) % every == 0 or frame == n_frames - 1:
                export_frame(state.x, faces, out / f"frame_{frame + 1:05d}.{fmt}")
                written += 1
    return {"frames": n_frames, "steps": state.step_index, "frame_files": written,
            "backend": _BACKEND, "metrics": str(csv_path),
            "wall_s": round(time.perf_counter() - t_start, 3)}


CONVERGENCE_HEADER = "solver,iteration,G,relative_loss,wall_ms"


def run_convergence(config: SceneConfig, solvers, n_iters: int, out_csv=None, threads=None,
                    g_star=None):
    """Convergence study on the frozen first-step objective (harness.py:702-743) on the GPU.

    Builds the scene, runs DCD at x_t and the warm start once (device), then records a G trace
    per requested solver from the same start (``baselines.descend``: one device call per
    solver).  The reference's G* comes from Newton (harness.py:721-722), which is not provided:
    pass ``g_star``, else the lowest G of the recorded traces stands in for it
    (``g_star_method`` "min-trace"; VBD's fixed point is not G's minimiser, since damping is a
    force-level term, so a long VBD run is no substitute for Newton).  Writes
    solver,iteration,G,relative_loss,wall_ms rows when out_csv is given."""
    from . import baselines
    from .solver import _collision, _INPUTS, device_context, initialize
    names = list(solvers)
    if "newton" in names:
        raise NotImplementedError("newton is not provided by the b200 backend")
    bad = [n for n in names if n not in baselines.METHODS]
    if bad:
        raise ValueError(f"unknown solver {bad[0]!r}")
    system, state, params = scene_build(config)
    if threads is not None:
        params = replace(params, threads=threads)
    ctx = device_context(system, params.precision, params.device)
    _collision(ctx, system, params)
    state._bind(ctx)
    state._upload(_INPUTS)
    mesh = getattr(system, "collision_mesh", None)
    if params.contact is not None and mesh is not None and len(mesh.surface_tris):
        ctx.detect_contacts(0, cap=1)  # DCD at x_t -> the active contact set (harness.py:718)
    initialize(state, params)
    x0, y0 = state.x.copy(), state.y.copy()
    traces, losses = {}, {}
    for name in names:
        state.x, state.y = x0.copy(), y0.copy()
        p = params
        if name == "vbd-cheb" and p.rho == 0.0:
            p = replace(p, rho=0.95)
        traces[name] = baselines.descend(state, p, name, n_iters)
    method = "given"
    if g_star is None:
        g_star = min(float(np.nanmin(t.g)) for t in traces.values()) if traces else 0.0
        method = "min-trace"
    for name in names:
        try:
            losses[name] = baselines.relative_loss(traces[name].g, g_star)
        except Exception:
            losses[name] = np.zeros_like(traces[name].g)

    if out_csv is not None:
        with open(out_csv, "w") as fh:
            fh.write(CONVERGENCE_HEADER + "\n")
            for name in names:
                tr = traces[name]
                for k in range(len(tr.g)):
                    fh.write(f"{name},{k},{_g(tr.g[k])},{_g(losses[name][k])},{tr.wall_ms[k]:.3f}\n")
    return {"g_star": g_star, "g_star_method": method, "traces": traces, "relative_loss": losses}
