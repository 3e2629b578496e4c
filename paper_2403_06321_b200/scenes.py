"""The BASELINE.json configurations as device-generated scenes.

C1 cantilever    generate_beam(41,11,11,0.025), root x=0 fixed, mu=1e6 lam=1e7 kd=1e-6,
                 h=1/60, n_max=10, gravity, adaptive init
C2 extreme init  generate_cube(37,0.5) with x0 ~ U(bbox) (rng 0), mu=2e6 lam=1e7 kd=1e-6,
                 h=1/60, n_max=100, rho=0.95, no gravity
C3 twist beams   two generate_beam(3032,4,4,0.01), mu=5e4 lam=1e6 kd=1e-6, h=1/300,
                 n_max=100, rho=0.95, both ends clamped
C4 many objects  10,368 x generate_cube(15,0.3) on a 24x24x18 lattice (pitch 0.5 m), seeded
                 random rigid velocities, mu=1e6 lam=1e7 kd=1e-7, h=1/120, n_max=60, gravity
C5 large block   generate_beam(364,364,364,0.01) (48.2M v / 239.2M t), x=0 face fixed,
                 mu=2e6 lam=2e7 kd=1e-7, h=1/240, n_max=40, gravity
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .context import Beam, DeviceContext
from .dist import object_shard, slab_cuts

G = (0.0, 0.0, -9.8)


@dataclass(frozen=True)
class Config:
    name: str
    beams: tuple
    h: float
    n_max: int
    rho: float = 0.0
    a_ext: tuple = G
    substeps: int = 1
    sharding: str = "objects"   # "objects" | "slabs" | "replicas"
    random_init: bool = False
    rigid_velocity: float = 0.0  # scale of seeded random rigid velocities (C4)
    twist_rev_s: float = 0.0     # C3: clamped end planes rotate about the beam axis
    description: str = ""

    @property
    def num_vertices(self):
        return sum(b.num_vertices for b in self.beams)

    @property
    def num_tets(self):
        return sum(b.num_tets for b in self.beams)

    def step_params(self):
        return DeviceContext.step_params(self.h, self.n_max, self.rho, 1e-10, "adaptive",
                                         self.a_ext)


def _c4_beams(count=10368, n=15, edge=0.3, pitch=0.5, dims=(24, 24, 18)):
    out = []
    for k in range(count):
        i, j, l = k // (dims[1] * dims[2]), (k // dims[2]) % dims[1], k % dims[2]
        out.append(Beam(n, n, n, edge / (n - 1), 1e6, 1e7, 1e-7,
                        origin=(pitch * i, pitch * j, 1.0 + pitch * l)))
    return tuple(out)


def config(name: str, scale: float = 1.0) -> Config:
    """BASELINE config by name ('c1'..'c5'); ``scale`` < 1 shrinks C4/C5 for tests."""
    if name == "c1":
        return Config("c1", (Beam(41, 11, 11, 0.025, 1e6, 1e7, 1e-6, fix_min_x=True),),
                      1 / 60, 10, sharding="replicas",
                      description="cantilever generate_beam(41,11,11,0.025), root fixed")
    if name == "c2":
        return Config("c2", (Beam(37, 37, 37, 0.5 / 36, 2e6, 1e7, 1e-6),), 1 / 60, 100, 0.95,
                      (0.0, 0.0, 0.0), sharding="replicas", random_init=True,
                      description="extreme init: generate_cube(37,0.5), x0 ~ U(bbox) rng 0")
    if name == "c3":
        n = max(4, int(round(3032 * scale)))
        return Config("c3", (Beam(n, 4, 4, 0.01, 5e4, 1e6, 1e-6, fix_min_x=True, fix_max_x=True),
                             Beam(n, 4, 4, 0.01, 5e4, 1e6, 1e-6, origin=(0.0, 0.2, 0.0),
                                  fix_min_x=True, fix_max_x=True)),
                      1 / 300, 100, 0.95, (0.0, 0.0, 0.0), sharding="replicas", twist_rev_s=0.5,
                      description=f"two thin beams generate_beam({n},4,4,0.01), both ends "
                                  "clamped and twisted +-0.5 rev/s (kinematic x_t)")
    if name == "c4":
        count = max(1, int(round(10368 * scale)))
        return Config("c4", _c4_beams(count), 1 / 120, 60, sharding="objects",
                      rigid_velocity=1.0,
                      description=f"{count} x generate_cube(15,0.3) on a lattice")
    if name == "c5":
        n = max(4, int(round(364 * scale ** (1 / 3))))
        return Config("c5", (Beam(n, n, n, 0.01, 2e6, 2e7, 1e-7, fix_min_x=True),), 1 / 240, 40,
                      sharding="slabs", description=f"generate_beam({n},{n},{n},0.01), x=0 fixed")
    if name == "c5j":  # C5 with irregular rest shapes: one kind per entry, no entry dictionary
        n = max(4, int(round(364 * scale ** (1 / 3))))
        return Config("c5j", (Beam(n, n, n, 0.01, 2e6, 2e7, 1e-7, fix_min_x=True, jitter=0.1),),
                      1 / 240, 40, sharding="slabs",
                      description=f"generate_beam({n},{n},{n},0.01) with rest positions jittered "
                                  "+-10% of the spacing (irregular mesh), x=0 fixed")
    raise ValueError(f"unknown config {name!r}")


def end_planes(cfg: Config):
    """Original ids of the clamped end planes of every beam (x = first / last plane)."""
    ids, off = [], 0
    for b in cfg.beams:
        plane = b.ny * b.nz
        ids.append(off + np.arange(plane))
        ids.append(off + (b.nx - 1) * plane + np.arange(plane))
        off += b.num_vertices
    return ids


def twist_targets(cfg: Config, rest: np.ndarray, t: float):
    """Kinematic targets of the clamped ends at time t: the x = min plane of each beam turns
    by +2 pi f t and the x = max plane by -2 pi f t about the beam axis (
    the reference drives such BCs by rewriting x_t of fixed vertices, test_acceptance.py:471)."""
    idx, xyz = [], []
    planes = end_planes(cfg)
    for k, b in enumerate(cfg.beams):
        cy = b.origin[1] + 0.5 * b.spacing * (b.ny - 1)
        cz = b.origin[2] + 0.5 * b.spacing * (b.nz - 1)
        for side, sign in ((0, 1.0), (1, -1.0)):
            ids = planes[2 * k + side]
            th = sign * 2.0 * np.pi * cfg.twist_rev_s * t
            p = rest[ids].copy()
            dy, dz = p[:, 1] - cy, p[:, 2] - cz
            p[:, 1] = cy + np.cos(th) * dy - np.sin(th) * dz
            p[:, 2] = cz + np.sin(th) * dy + np.cos(th) * dz
            idx.append(ids)
            xyz.append(p)
    return np.concatenate(idx), np.concatenate(xyz)


def rigid_velocities(num_beams: int, scale: float, seed: int = 0):
    """Seeded random rigid (linear, angular) velocities per object, (num_beams, 6)."""
    rng = np.random.default_rng(seed)
    la = np.zeros((num_beams, 6))
    if scale:
        la[:, :3] = scale * rng.uniform(-1, 1, (num_beams, 3))
        la[:, 3:] = 4.0 * scale * rng.uniform(-1, 1, (num_beams, 3))
    return la


def build(cfg: Config, rank: int = 0, world: int = 1, precision: str = "fp32", device: int = 0):
    """This rank's DeviceContext for ``cfg`` (object shard, slab, or full replica)."""
    if world > 1 and cfg.sharding == "slabs":
        b = cfg.beams[0]
        cuts = slab_cuts(b.nx, world, int(b.fix_min_x), int(b.fix_max_x))
        ctx = DeviceContext.from_beams(list(cfg.beams), precision, device,
                                       slab=(cuts[rank], cuts[rank + 1]))
        return ctx, (cuts[rank], cuts[rank + 1])
    if world > 1 and cfg.sharding == "objects":
        lo, hi = object_shard(len(cfg.beams), rank, world)
        beams = list(cfg.beams[lo:hi])
        ctx = DeviceContext.from_beams(beams, precision, device)
        if cfg.rigid_velocity:
            ctx.set_beam_velocities(rigid_velocities(len(cfg.beams), cfg.rigid_velocity)[lo:hi])
        return ctx, (lo, hi)
    ctx = DeviceContext.from_beams(list(cfg.beams), precision, device)
    if cfg.rigid_velocity:
        ctx.set_beam_velocities(rigid_velocities(len(cfg.beams), cfg.rigid_velocity))
    if cfg.random_init:
        x = ctx.get_state(x=True)["x"]
        lo, hi = x.min(0), x.max(0)
        x0 = np.random.default_rng(0).uniform(lo, hi, size=x.shape)
        ctx.set_state(x=x0, x_t=x0)
    return ctx, None
