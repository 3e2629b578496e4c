/*
 * vbd_b200.h -- C ABI of the B200-native Vertex Block Descent hot path (libvbd_b200.so).
 *
 * Plain pointers and sizes only.  Every function returns VBD_OK (0) or a negative
 * VBD_ERR_* code; vbd_last_error() returns a thread-local message for the last failure.
 * Host arrays are C-contiguous, row-major, in the reference's original vertex numbering
 * ((N,3) float64 positions, int64 indices) exactly as the reference's System/SimState hold
 * them (/root/reference/pkg/src/vbdsim/_system.py:99-133, solver.py:88-108).
 *
 * Which reference interface each entry point replaces:
 *   vbd_ctx_create      <- the flat arrays the reference's Cython kernel borrows per call
 *                          (pkg/src/vbdsim/_native.pyx:525-575 SysData fill) -- compiled once
 *                          into the device layout instead of per call
 *   vbd_color_pass      <- backend.color_pass(system, carr, x, x_t, y, h, group, mode, ...)
 *                          (pkg/src/vbdsim/_native.pyx:513-589; protocol of _backend.py:13-32)
 *   vbd_step            <- vbdsim.step(state, params) (pkg/src/vbdsim/solver.py:291-324),
 *                          device-resident: K2 init, n_max x (colour passes, K3), K4 commit
 *   vbd_set_state /     <- SimState.x_t / v_t / v_prev / x / y (solver.py:88-108) crossing
 *   vbd_get_state          the host<->device boundary
 *   vbd_greedy_color    <- greedy_color(adjacency, order) (pkg/src/vbdsim/mesh.py:270-302)
 *   vbd_ctx_create_beams<- generate_beam/generate_cube + build_tet_mesh + build_system for
 *                          procedural scenes (harness.py:42-76, mesh.py:128-170,
 *                          _system.py:204-303), built on the device for 10^7..10^8-vertex scenes
 *   vbd_halo_*          <- (no reference counterpart: multi-GPU slab decomposition)
 */
#ifndef VBD_B200_H
#define VBD_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VBD_OK 0
#define VBD_ERR_ARG (-1)
#define VBD_ERR_CUDA (-2)
#define VBD_ERR_UNSUPPORTED (-3)
#define VBD_ERR_NODEVICE (-5)
#define VBD_ERR_INTERNAL (-6)

#define VBD_PREC_F32 0
#define VBD_PREC_F64 1

#define VBD_KIND_FREE 0
#define VBD_KIND_FIXED 1 /* _system.py:17 FIXED */
#define VBD_KIND_SUBSPACE 2 /* SubspaceConstraint (_system.py:38-53) */

#define VBD_INIT_PREV_POS 0 /* solver.py:25 INIT_MODES */
#define VBD_INIT_INERTIA 1
#define VBD_INIT_INERTIA_ACCEL 2
#define VBD_INIT_ADAPTIVE 3

typedef struct vbd_ctx vbd_ctx;

/* The reference System arrays (tets-only scenes).  Borrowed for the call only. */
typedef struct {
    int64_t num_vertices;
    int64_t num_tets;
    const int64_t* tets;        /* (T,4) */
    const double* tet_w;        /* (T,4,3) slot weight rows */
    const double* tet_vol;      /* (T,) */
    const double* tet_mu;       /* (T,) */
    const double* tet_lam;      /* (T,) */
    const double* tet_kd;       /* (T,) */
    const double* masses;       /* (N,) */
    const uint8_t* kind;        /* (N,) 0 free, 1 fixed; NULL = all free */
    const int64_t* t_off;       /* (N+1,) vertex->tet CSR, ascending tet id per vertex */
    const int64_t* t_id;        /* (4T,) */
    const int64_t* t_slot;      /* (4T,) */
    int64_t num_colors;
    const int64_t* color_off;   /* (C+1,) */
    const int64_t* color_verts; /* (N,) colour groups, concatenated */
    const double* rest_positions; /* (N,3) optional: spatial (Morton) order inside colours */
    /* spring nets (_system.py:117-123; NULL / 0 = none) */
    int64_t num_springs;
    const int64_t* springs;     /* (S,2) */
    const double* sp_l0;        /* (S,) */
    const double* sp_k;         /* (S,) */
    const double* sp_kd;        /* (S,) */
    /* constraints (_system.py:76-83; NULL = none): kind[v] == VBD_KIND_SUBSPACE marks
     * SubspaceConstraint vertices; box_k[v] > 0 an active WorldBoxConstraint */
    const int64_t* sub_dim;     /* (N,) */
    const double* sub_basis;    /* (N,3,2) */
    const double* sub_anchor;   /* (N,3) */
    const double* box_k;        /* (N,) */
    const double* box_lo;       /* (N,3) */
    const double* box_hi;       /* (N,3) */
} vbd_system_desc;

/* A procedural generate_beam(nx, ny, nz, spacing, density) body, rigidly translated. */
typedef struct {
    int64_t nx, ny, nz;
    double spacing;
    double density;
    double origin[3];
    double mu, lam, kd;
    int32_t fix_min_x; /* FixedConstraint on every vertex with (x - origin.x) < 1e-9 */
    int32_t fix_max_x; /* ... and on every vertex of the last x plane (clamped far end) */
    double jitter;     /* rest positions moved by a deterministic per-vertex offset in
                          [-jitter, jitter] x spacing (0 = the reference grid; the x = 0 plane
                          keeps x = 0): an irregular mesh with one rest shape per tet */
} vbd_beam_desc;

typedef struct {
    double h;
    int32_t n_max;
    int32_t init_mode;
    double rho;
    double eps_det;
    double a_ext[3];
    int32_t line_search; /* 17-trial local backtracking per vertex (_native.pyx:481-492) */
    int32_t reserved;
} vbd_step_params;

typedef struct {
    int32_t nonfinite;  /* 1 if a non-finite position was detected (step not committed) */
    int32_t step;       /* step (0-based, within this call) of the first detection */
    int32_t iteration;  /* iteration (1-based) of the first detection */
    int32_t reserved;
    int64_t vertex;     /* smallest original vertex id that was non-finite then */
} vbd_step_result;

typedef struct {
    int64_t num_vertices, num_solved, num_ghost, num_fixed;
    int64_t num_tets, num_entries;
    int64_t num_colors;
    int64_t color_count[64];   /* solved vertices per colour (first 64 colours) */
    int64_t device_bytes;
    int32_t precision;
    int32_t inplace;           /* 1 = colouring valid -> in-place colour sweeps */
    int32_t lanes_per_vertex;
    int32_t num_materials;
    int32_t layout;            /* 0 explicit entries (48 B fp32 / 96 B fp64), 1 compact (16 B +
                                  a table of distinct entry kinds; lossless) */
    int32_t entry_bytes;       /* bytes streamed per (vertex, tet) entry */
    int64_t num_entry_kinds;   /* compact layout: distinct (rows, volume, material) keys */
    int32_t tiles;             /* K1T tile pipeline: number of tiles (0 = off) */
    int32_t tile_nbr_cap;      /* max distinct neighbours of one tile */
    int64_t tile_slots;        /* K1T: 8-byte entry slots over all tiles (entries + padding) */
    int64_t tile_nbr_refs;     /* K1T: neighbour-list entries over all tiles */
    int32_t tile_lanes;        /* K1T: lanes per vertex */
    int32_t tile_stages;       /* K1T: shared-memory pipeline stages */
    int32_t tile_ent_cap;      /* K1T: entry slots of the largest tile (per-stage capacity) */
    int32_t tile_smem_bytes;   /* K1T: dynamic shared memory per CTA */
    int32_t resident;          /* K1R whole-step kernel (decided at the first step): 0 none,
                                  1 one cluster with position replicas, 2 grid-resident */
    int32_t resident_ctas;     /* K1R: CTAs (cluster size for 1, SMs for 2) */
    int64_t contact_graph_steps;     /* contact steps run as one captured graph */
    int64_t contact_graph_fallbacks; /* ... rolled back and redone on the host path (capacity) */
    int64_t class_vertices;    /* K1T: solved vertices swept in grid-class tiles */
    int32_t class_tiles;       /* K1T: grid-class tiles (one lane per vertex, register-resident
                                  neighbours) */
    int32_t class_records;     /* K1T: kind records staged per class position */
} vbd_ctx_info;

/* ---- context ---------------------------------------------------------------------------- */
int vbd_device_count(int* count);
int vbd_ctx_create(const vbd_system_desc* desc, int device, int precision, vbd_ctx** out);
int vbd_ctx_create_beams(const vbd_beam_desc* beams, int64_t num_beams, int64_t slab_lo,
                         int64_t slab_hi, int device, int precision, vbd_ctx** out);
int vbd_ctx_destroy(vbd_ctx* ctx);
int vbd_ctx_get_info(vbd_ctx* ctx, vbd_ctx_info* info);
int vbd_set_stream(vbd_ctx* ctx, void* cuda_stream); /* NULL = the context's own stream */
int vbd_get_stream(vbd_ctx* ctx, void** cuda_stream);
int vbd_get_colors(vbd_ctx* ctx, int64_t* color_of); /* (N,) original numbering */

/* ---- state (host <-> device, original numbering, (N,3) float64) ------------------------- */
int vbd_set_state(vbd_ctx* ctx, const double* x, const double* x_t, const double* v_t,
                  const double* v_prev, const double* y); /* NULL = leave unchanged */
int vbd_get_state(vbd_ctx* ctx, double* x, double* x_t, double* v_t, double* v_prev, double* y);
int vbd_set_beam_velocities(vbd_ctx* ctx, const double* lin_ang); /* (num_beams,6) rigid v */
/* kinematic boundary conditions: x_t (and x) of fixed vertices idx[0..n) (original ids) set to
 * xyz (n,3) before the next step -- how the reference drives clamped ends
 * (pkg/tests/test_acceptance.py:471-473 rewrites x/x_t of FixedConstraint vertices) */
int vbd_set_fixed_targets(vbd_ctx* ctx, int64_t n, const int64_t* idx, const double* xyz);

/* ---- the hot path ----------------------------------------------------------------------- */
int vbd_step(vbd_ctx* ctx, const vbd_step_params* params, int32_t n_steps, vbd_step_result* res);
int vbd_color_pass(vbd_ctx* ctx, double* x_inout, const double* x_t, const double* y, double h,
                   const int64_t* group, int64_t ng, int32_t mode, int32_t line_search,
                   double eps_det);

/* K2 only: y = inertia target and the warm start of solver.py:125-164 into x (no sweeps) */
int vbd_initialize(vbd_ctx* ctx, const vbd_step_params* params);

/* fine-grained step for multi-GPU slabs (halo exchange between colour passes) */
int vbd_step_begin(vbd_ctx* ctx, const vbd_step_params* params);
int vbd_step_color(vbd_ctx* ctx, int32_t color, int32_t iteration);
int vbd_step_iter_end(vbd_ctx* ctx, int32_t iteration);
int vbd_step_end(vbd_ctx* ctx, vbd_step_result* res);
int vbd_halo_count(vbd_ctx* ctx, int32_t side, int32_t color, int64_t* n_send, int64_t* n_recv);
int vbd_halo_pack(vbd_ctx* ctx, int32_t side, int32_t color, void* dev_buf);
int vbd_halo_unpack(vbd_ctx* ctx, int32_t side, int32_t color, const void* dev_buf);

/* fused P2P halo (B200 path): K1 stores each boundary vertex of the colour it just solved
 * straight into the neighbour's ghost slot (NVLink peer memory), and a device-side phase
 * barrier (flags in peer memory, st.release.sys / ld.acquire.sys) orders the phases of
 * neighbouring slabs; the whole step is one CUDA graph per rank with no host in the loop. */
int vbd_halo_ghost_blocks(vbd_ctx* ctx, int32_t side, int64_t* begin, int64_t* count, int64_t* boundary);
int vbd_halo_p2p_local(vbd_ctx* ctx, void** pos, void** flags); /* same-process peers */
int vbd_halo_p2p_export(vbd_ctx* ctx, void* pos_handle64, void* flags_handle64); /* cudaIpc */
int vbd_ipc_open(int device, const void* handle64, void** ptr);
int vbd_ipc_close(void* ptr);
int vbd_halo_p2p_connect(vbd_ctx* ctx, int32_t side, void* peer_pos, void* peer_flags,
                         const int64_t* peer_ghost_begin, const int64_t* peer_ghost_count);
                         /* peer_pos == NULL disconnects `side` (the other arguments are ignored) */
int vbd_step_p2p_launch(vbd_ctx* ctx, const vbd_step_params* params); /* asynchronous */
int vbd_step_p2p_finish(vbd_ctx* ctx, vbd_step_result* res);

/* ---- colouring (K5, device Jones-Plassmann == reference greedy) ------------------------- */
int vbd_greedy_color(int64_t n, const int64_t* noff, const int64_t* nids, const int64_t* order,
                     int device, int64_t* color_of, int64_t* num_colors);

/* ---- contacts ----------------------------------------------------------------------------- */
/* The contact set of subsequent colour passes / steps: the reference's ContactArrays
 * (_system.py:86-96, compile_contacts :306-333) in original numbering -- idx (C,4), gamma (C,4),
 * refresh (C,), normal (C,3), tangent (C,3,2), k_c (C,), cv_off (N+1), cv_cid, cv_slot -- and
 * the friction parameters mu_c, eps_v (eps_u = eps_v h).  count 0 clears it.  The colour pass
 * adds the penalty and friction terms of _native.pyx:351-399 (DCD anchors refreshed,
 * :134-172).  Detection (broad phase, DCD, CCD) stays with the caller. */
int vbd_set_contacts(vbd_ctx* ctx, int64_t count, const int64_t* idx, const double* gamma,
                     const uint8_t* refresh, const double* normal, const double* tangent,
                     const double* k_c, const int64_t* cv_off, const int64_t* cv_cid,
                     const int64_t* cv_slot, double mu_c, double eps_v);

/* Contact detection on the device for vbd_step (solver.py:241-324, contact.py): the collision
 * surface (outward triangles (S,3) and unique edges (E,2) of the merged tet bodies, original
 * ids), the hash cell (1.5 x median rest surface edge, contact.py:205-215) and ContactParams.
 * Each step then runs DCD at x_t, CCD every n_col iterations, aux-buffer colour passes and K3
 * without blending colliding vertices.  ntri 0 disables it. */
int vbd_set_collision(vbd_ctx* ctx, int64_t ntri, const int64_t* tris, int64_t nedge, const int64_t* edges,
                      double cell, double k_c, double mu_c, double eps_v, double dcd_radius,
                      int32_t has_max_depth, double max_depth, int32_t n_col);
/* one detection pass on the current state (which 0: DCD at x_t; 1: CCD x_t -> x), for tests:
 * count, and up to cap records (original ids, signed weights, normal, 1 = CCD) */
int vbd_detect_contacts(vbd_ctx* ctx, int32_t which, int64_t cap, int64_t* count, int64_t* idx,
                        double* gamma, double* normal, int32_t* ccd);
int vbd_get_colliding(vbd_ctx* ctx, uint8_t* flags); /* (N,) sticky colliding flags of the step */

/* ---- metrics ------------------------------------------------------------------------------ */
/* G(x) = 1/(2h^2) |x - y|_M^2 + E(x) at the current iterate (tets, springs, world boxes and the
 * penalty of the active contact set) -- baselines.energy / _assembly.variational_energy
 * (_assembly.py:78-82), the per-iteration metric of harness.run_simulation
 * (harness.py:664-678).  Synchronous. */
int vbd_energy(vbd_ctx* ctx, double h, double* G);
/* vbd_energy plus the other two per-iteration metric columns of harness.py:664-670 in the same
 * reduction: the active contact count (len(state.contact_set)) and the largest contact gap at
 * the iterate (max_penetration, solver.py:327-332; 0 without contacts).  Either may be NULL. */
int vbd_energy_metrics(vbd_ctx* ctx, double h, double* G, int64_t* contacts, double* max_gap);

/* ---- convergence traces ------------------------------------------------------------------- */
/* baselines.descend (baselines.py:152-189) for the sweep methods, on the device, on the frozen
 * objective of the current x and y (vbd_set_state; no detection updates): method 0 "vbd" (colour
 * sweeps), 1 "vbd-cheb" (colour sweeps + Chebyshev blend at rho), 2 "jacobi" (block_jacobi_step,
 * baselines.py:92-97: every vertex against the previous iterate) and 3 "gd" (gd_step, :100-104,
 * mode 1); jacobi and gd take the global backtracking line search toward the last checkpoint every
 * 8 iterations (:139-149, 180-183).  g[0..n_iters] = G per iteration (vbd_energy's value),
 * wall_ms[0..n_iters] (may be NULL) = cumulative device time since after G_0 (CUDA events).
 * x is left at the final iterate. */
int vbd_descend(vbd_ctx* ctx, int32_t method, int32_t n_iters, double h, double rho, double eps_det,
                int32_t line_search, double* g, double* wall_ms);

/* ---- measurement ------------------------------------------------------------------------ */
/* average device time of one colour-pass launch per colour over `reps` sweeps, colours in step
 * order (one CUDA event pair per launch on the context stream); ms has room for num_colors values */
/* Diagnostics (VBD_RES_DBG=8 at context creation): K1R's pass timeline of CTA 0 in the last
   step, 5 clock64 values per pass {start, last sweep end, last push end, barrier exit, the
   longest single group's sweep end -> push end}. */
int vbd_resident_timeline(vbd_ctx* ctx, int64_t* out, int64_t cap, int64_t* n);
int vbd_profile_color_pass(vbd_ctx* ctx, double h, int32_t reps, double* ms);

/* FMA-pipe peak of this device (the denominator of the FP32 / FP64 roofline): a kernel of
 * independent fused multiply-add chains on every SM (precision VBD_PREC_F32: packed fp32x2
 * FFMA2 when packed != 0, else scalar FFMA; VBD_PREC_F64: DFMA), run back to back for about
 * `seconds` (a burst when short, the power-capped sustained rate when long).  *tflops = 2 x FMAs
 * per second / 1e12 over the timed launches (CUDA events). */
int vbd_fma_peak(int device, int precision, int packed, double seconds, double* tflops);

const char* vbd_last_error(void);
const char* vbd_version(void);

#ifdef __cplusplus
}
#endif
#endif
