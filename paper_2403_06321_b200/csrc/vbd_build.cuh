// vbd_build.cuh -- one-off scene construction on the device:
//   * procedural beams/cubes (generate_beam, harness.py:42-76) incl. the orientation fix,
//     Dm^-1, volumes and slot-weight rows of build_tet_mesh / _slot_weight_rows
//     (mesh.py:128-170, _system.py:139-144);
//   * vertex->tet incidence (mesh.py:232-267) and lumped masses (mesh.py:161-162);
//   * distinct-neighbour CSR (_system.py:147-169) and the K5 Jones-Plassmann colouring whose
//     priority (-degree, index) reproduces greedy_color (mesh.py:270-302) bit-exactly;
//   * K6: the colour-major re-pack into the entry planes consumed by K1.
#pragma once
#include "vbd_common.cuh"
#include "vbd_grid_classes.cuh"

// ---------------------------------------------------------------------------------------
// procedural beams

struct BeamDev {
    long long nx, ny, nz;
    long long ax0, ax1;   // vertex planes generated: [ax0, ax1] inclusive (slab incl. ghosts)
    long long vbase;      // first local vertex id of this beam
    long long tbase;      // first local tet id
    long long gcell0;     // first global cell x index generated (cells [gcell0, ax1-1])
    double spacing, density;
    double origin[3];
    int mat;
    int fix_min_x;
    int fix_max_x;
    double jitter;  // fraction of spacing (vbd_beam_desc::jitter)
};

// deterministic jitter in [-1, 1) of (global vertex, axis): splitmix64 of the key
__device__ __forceinline__ double vertex_jitter(unsigned long long key)
{
    unsigned long long z = key + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

__constant__ int c_cell_even[5][4] = {{0, 3, 5, 6}, {1, 0, 3, 5}, {2, 0, 3, 6}, {4, 0, 5, 6}, {7, 3, 5, 6}};
__constant__ int c_cell_odd[5][4] = {{1, 2, 4, 7}, {0, 1, 2, 4}, {3, 1, 2, 7}, {5, 1, 4, 7}, {6, 2, 4, 7}};

__device__ __forceinline__ int find_beam(const BeamDev* b, int nb, long long key, bool by_tet)
{
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        long long base = by_tet ? b[mid].tbase : b[mid].vbase;
        if (base <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_gen_vertices(const BeamDev* __restrict__ beams, int nb, long long n,
                               double* __restrict__ pos, unsigned char* __restrict__ kind)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const BeamDev& B = beams[find_beam(beams, nb, v, false)];
    long long l = v - B.vbase;
    long long az = l % B.nz, ay = (l / B.nz) % B.ny, ax = B.ax0 + l / (B.nz * B.ny);
    // harness.py:50-51: spacing * (ix, iy, iz), then the rigid translation
    double px = B.spacing * (double)ax, py = B.spacing * (double)ay, pz = B.spacing * (double)az;
    if (B.jitter != 0.0) {  // irregular rest shapes; keyed by the global vertex (slabs agree)
        const unsigned long long g = (unsigned long long)((ax * B.ny + ay) * B.nz + az) * 3ull;
        const double a = B.jitter * B.spacing;
        if (ax > 0) px += a * vertex_jitter(g);
        py += a * vertex_jitter(g + 1);
        pz += a * vertex_jitter(g + 2);
    }
    pos[3 * v] = px + B.origin[0];
    pos[3 * v + 1] = py + B.origin[1];
    pos[3 * v + 2] = pz + B.origin[2];
    kind[v] = ((B.fix_min_x && px < 1e-9) || (B.fix_max_x && ax == B.nx - 1)) ? 1 : 0;
}

// Tets of the generated cells in global (cell-major, then pattern) order, with the
// orientation fix of mesh.py:147-152, Dm^-1 (mesh.py:158-159), |V| (mesh.py:147) and the
// slot-weight rows w_0 = -sum(Dm^-1 rows), w_{k+1} = row k (_system.py:139-144).
__global__ void k_gen_tets(const BeamDev* __restrict__ beams, int nb, long long T,
                           const double* __restrict__ pos, int* __restrict__ tets,
                           double* __restrict__ tet_w, double* __restrict__ vol,
                           int* __restrict__ tmat)
{
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const BeamDev& B = beams[find_beam(beams, nb, t, true)];
    long long l = t - B.tbase;
    long long cell = l / 5;
    int j = (int)(l % 5);
    long long ncz = B.nz - 1, ncy = B.ny - 1;
    long long cz = cell % ncz, cy = (cell / ncz) % ncy, cx = B.gcell0 + cell / (ncz * ncy);
    const int(*pat)[4] = ((cx + cy + cz) % 2 == 0) ? c_cell_even : c_cell_odd;
    long long vid[4];
    int cof[4][3];  // the corners' integer cell offsets
    for (int k = 0; k < 4; ++k) {
        int c = pat[j][k];
        int dx = c >> 2, dy = (c >> 1) & 1, dz = c & 1;
        cof[k][0] = dx;
        cof[k][1] = dy;
        cof[k][2] = dz;
        vid[k] = B.vbase + ((cx + dx - B.ax0) * B.ny + (cy + dy)) * B.nz + (cz + dz);
    }
    // columns = edges x_{k} - x_0, D[a*3+k].  On the regular grid the edges are formed from the
    // corners' integer offsets times the spacing (exact), not from differences of rounded
    // absolute positions: every cell of a shape then gets bitwise the same Dm^-1 and V, so an
    // fp64 grid has 40 entry kinds like fp32 (not ~40,000 last-bit variants).  The reference
    // differences positions (mesh.py:155-159); the two agree to ~1e-13 relative.  Jittered
    // meshes (irregular) difference the positions.
    double D[9];
    for (int k = 0; k < 3; ++k)
        for (int a = 0; a < 3; ++a)
            D[a * 3 + k] = B.jitter == 0.0 ? (double)(cof[k + 1][a] - cof[0][a]) * B.spacing
                                          : pos[3 * vid[k + 1] + a] - pos[3 * vid[0] + a];
    double det = D[0] * (D[4] * D[8] - D[5] * D[7]) - D[1] * (D[3] * D[8] - D[5] * D[6]) +
                 D[2] * (D[3] * D[7] - D[4] * D[6]);
    if (det < 0.0) {  // swap slots 1 and 2: [0, 2, 1, 3]
        long long tmp = vid[1]; vid[1] = vid[2]; vid[2] = tmp;
        for (int a = 0; a < 3; ++a) {
            double s = D[a * 3 + 0]; D[a * 3 + 0] = D[a * 3 + 1]; D[a * 3 + 1] = s;
        }
        det = -det;
    }
    double inv[9];
    inv[0] = (D[4] * D[8] - D[5] * D[7]) / det;
    inv[1] = (D[2] * D[7] - D[1] * D[8]) / det;
    inv[2] = (D[1] * D[5] - D[2] * D[4]) / det;
    inv[3] = (D[5] * D[6] - D[3] * D[8]) / det;
    inv[4] = (D[0] * D[8] - D[2] * D[6]) / det;
    inv[5] = (D[2] * D[3] - D[0] * D[5]) / det;
    inv[6] = (D[3] * D[7] - D[4] * D[6]) / det;
    inv[7] = (D[1] * D[6] - D[0] * D[7]) / det;
    inv[8] = (D[0] * D[4] - D[1] * D[3]) / det;
    for (int k = 0; k < 4; ++k) tets[4 * t + k] = (int)vid[k];
    double* w = tet_w + 12 * t;
    for (int b = 0; b < 3; ++b) {
        w[3 + b] = inv[b];
        w[6 + b] = inv[3 + b];
        w[9 + b] = inv[6 + b];
        w[b] = -((inv[b] + inv[3 + b]) + inv[6 + b]);
    }
    vol[t] = det / 6.0;
    tmat[t] = B.mat;
}

// ---------------------------------------------------------------------------------------
// incidence: keys = vertex of each (tet, slot), values = 4 t + s; a stable radix sort by key
// gives the reference's lexsort((eids, verts)) order (mesh.py:243-250).

__global__ void k_inc_keys(const int* __restrict__ tets, long long n4, int* __restrict__ keys,
                           unsigned* __restrict__ vals, int* __restrict__ count)
{
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n4) return;
    int v = tets[k];
    keys[k] = v;
    vals[k] = (unsigned)k;
    atomicAdd(count + v, 1);
}

// lumped masses rho V / 4 accumulated in ascending tet order per vertex (mesh.py:161-162)
__global__ void k_mass_gather(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                              const double* __restrict__ vol, const int* __restrict__ tmat,
                              const double* __restrict__ density_of_mat, long long n,
                              double* __restrict__ mass)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    double m = 0.0;
    for (long long k = off[v]; k < off[v + 1]; ++k) {
        long long t = inc[k] >> 2;
        m = m + (density_of_mat[tmat[t]] * vol[t]) / 4.0;
    }
    mass[v] = m;
}

// ---------------------------------------------------------------------------------------
// distinct neighbours from the incidence (per-vertex sort + unique in registers/local mem)

#define VBD_MAX_NBR_CAND 384

__device__ int gather_neighbours(long long v, const long long* off, const unsigned* inc,
                                 const int* tets, int* cand)
{
    int c = 0;
    for (long long k = off[v]; k < off[v + 1] && c + 3 <= VBD_MAX_NBR_CAND; ++k) {
        long long t = inc[k] >> 2;
        for (int s = 0; s < 4; ++s) {
            int u = tets[4 * t + s];
            if (u != v) cand[c++] = u;
        }
    }
    // insertion sort (small) then unique
    for (int i = 1; i < c; ++i) {
        int x = cand[i], j = i - 1;
        while (j >= 0 && cand[j] > x) { cand[j + 1] = cand[j]; --j; }
        cand[j + 1] = x;
    }
    int u = 0;
    for (int i = 0; i < c; ++i)
        if (u == 0 || cand[u - 1] != cand[i]) cand[u++] = cand[i];
    return u;
}

__global__ void k_nbr_count(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                            const int* __restrict__ tets, long long n, int* __restrict__ cnt,
                            int* __restrict__ overflow)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    if ((off[v + 1] - off[v]) * 3 > VBD_MAX_NBR_CAND) atomicExch(overflow, 1);
    int cand[VBD_MAX_NBR_CAND];
    cnt[v] = gather_neighbours(v, off, inc, tets, cand);
}

__global__ void k_nbr_fill(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                           const int* __restrict__ tets, long long n, const long long* __restrict__ noff,
                           int* __restrict__ nids)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    int cand[VBD_MAX_NBR_CAND];
    int c = gather_neighbours(v, off, inc, tets, cand);
    for (int i = 0; i < c; ++i) nids[noff[v] + i] = cand[i];
}

// ---------------------------------------------------------------------------------------
// K5: Jones-Plassmann colouring with the greedy order as priority.  Vertex u precedes v iff
// rank(u) < rank(v), rank = position in lexsort((index, -degree)) (mesh.py:277-278) or a
// caller-given order.  A vertex is coloured once all preceding neighbours are, with the
// smallest colour they do not use -- exactly what the sequential greedy assigns.

__device__ __forceinline__ bool precedes(long long u, long long v, const long long* noff,
                                         const long long* rank)
{
    if (rank) return rank[u] < rank[v];
    long long du = noff[u + 1] - noff[u], dv = noff[v + 1] - noff[v];
    return du > dv || (du == dv && u < v);
}

__global__ void k_jp_init(const long long* __restrict__ noff, const int* __restrict__ nids,
                          const long long* __restrict__ rank, long long n, int* __restrict__ pending,
                          int* __restrict__ color, int* __restrict__ frontier, int* __restrict__ fcount)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    int p = 0;
    for (long long k = noff[v]; k < noff[v + 1]; ++k)
        if (precedes(nids[k], v, noff, rank)) ++p;
    pending[v] = p;
    color[v] = -1;
    if (p == 0) frontier[atomicAdd(fcount, 1)] = (int)v;
}

__global__ void k_jp_round(const long long* __restrict__ noff, const int* __restrict__ nids,
                           const long long* __restrict__ rank, const int* __restrict__ fin,
                           const int* __restrict__ fin_count, int* __restrict__ pending,
                           int* __restrict__ color, int* __restrict__ fout, int* __restrict__ fout_count,
                           unsigned long long* __restrict__ colored, int* __restrict__ overflow)
{
    const int cnt = *fin_count;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < cnt; idx += gridDim.x * blockDim.x) {
        const int v = fin[idx];
        unsigned long long used[4] = {0ull, 0ull, 0ull, 0ull};
        for (long long k = noff[v]; k < noff[v + 1]; ++k) {
            int u = nids[k];
            if (precedes(u, v, noff, rank)) {
                int c = color[u];
                if (c < 256) used[c >> 6] |= 1ull << (c & 63);
                else atomicExch(overflow, 1);
            }
        }
        int c = 0;
        while (c < 256 && ((used[c >> 6] >> (c & 63)) & 1ull)) ++c;
        if (c >= 256) atomicExch(overflow, 1);
        color[v] = c;
        atomicAdd(colored, 1ull);
        for (long long k = noff[v]; k < noff[v + 1]; ++k) {
            int u = nids[k];
            if (precedes(v, u, noff, rank))
                if (atomicSub(pending + u, 1) == 1) fout[atomicAdd(fout_count, 1)] = u;
        }
    }
}

// a colouring is valid for in-place sweeps iff no tet repeats a colour (oracles.py:175-181)
__global__ void k_check_coloring(const int* __restrict__ tets, long long T, const int* __restrict__ color,
                                 int* __restrict__ bad)
{
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= T) return;
    int c0 = color[tets[4 * t]], c1 = color[tets[4 * t + 1]], c2 = color[tets[4 * t + 2]],
        c3 = color[tets[4 * t + 3]];
    if (c0 == c1 || c0 == c2 || c0 == c3 || c1 == c2 || c1 == c3 || c2 == c3) atomicExch(bad, 1);
}

// ---------------------------------------------------------------------------------------
// K6: colour-major order and entry packing

__device__ __forceinline__ unsigned long long spread3(unsigned long long x)
{
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// 63-bit Morton code of the quantised rest position (21 bits per axis)
__global__ void k_morton_keys(const double* __restrict__ pos, long long n, double lx, double ly,
                              double lz, double scale, unsigned long long* __restrict__ keys,
                              int* __restrict__ ids)
{
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    double q[3] = {(pos[3 * v] - lx) * scale, (pos[3 * v + 1] - ly) * scale, (pos[3 * v + 2] - lz) * scale};
    unsigned long long c[3];
    for (int k = 0; k < 3; ++k) {
        double t = q[k] < 0.0 ? 0.0 : (q[k] > 2097151.0 ? 2097151.0 : q[k]);
        c[k] = (unsigned long long)t;
    }
    keys[v] = spread3(c[0]) << 2 | spread3(c[1]) << 1 | spread3(c[2]);
    ids[v] = (int)v;
}

__global__ void k_iota(int* __restrict__ a, long long n)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

// Sort key of the colour-major order:
//   category (2 b: 0 solved, 1 ghost, 2 fixed) | colour (12 b) | class (4 b) | rounds (8 b) | low 32
// solved: class 0 / 1 = slab boundary vertex facing the left / right neighbour, 2 = interior;
// ghost: class 0 / 1 = ghost plane on the left / right.  Boundary and ghost blocks are ordered
// by vertex id (so a rank's boundary block matches the neighbour's ghost block element for
// element); interior vertices by (rounds = ceil(d/W), spatial rank i -> order0[i]); vertices of
// a grid-class instance (vinst, K1T class tiles) by (0x80 | instance, spatial rank), so each
// (colour, instance) is one contiguous run.
// halo: 0 none, 1 boundary-left, 2 boundary-right, 3 ghost-left, 4 ghost-right (may be null)
__global__ void k_order_keys(const long long* __restrict__ off, const unsigned char* __restrict__ kind,
                             const unsigned char* __restrict__ halo, const int* __restrict__ color,
                             const int* __restrict__ order0, long long n, int W,
                             unsigned long long* __restrict__ keys, const signed char* __restrict__ vinst = nullptr)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = order0[i];
    const unsigned hv = halo ? halo[v] : 0u;
    unsigned long long cat = kind[v] == 1 ? 2ull : (kind[v] == 3 ? 1ull : 0ull);
    unsigned long long c = (unsigned long long)(color[v] < 0 ? 0 : color[v]) & 0xfffull;
    unsigned long long cls, r = 0ull, low;
    if (cat == 0) {
        cls = hv == 1 ? 0ull : (hv == 2 ? 1ull : 2ull);
        if (cls == 2) {
            long long d = off[v + 1] - off[v];
            r = (unsigned long long)min((d + W - 1) / W, 0x7fLL);
            if (vinst && vinst[v] >= 0) r = 0x80ull | (unsigned long long)vinst[v];  // K1T class tiles
            low = (unsigned long long)i;
        } else {
            low = (unsigned long long)v;
        }
    } else {
        cls = (cat == 1 && hv == 4) ? 1ull : 0ull;
        low = (unsigned long long)v;
    }
    keys[i] = (cat << 56) | (c << 44) | (cls << 40) | (r << 32) | low;
}

__device__ __forceinline__ bool key_is_rank(unsigned long long k)
{
    return (k >> 56) == 0ull && ((k >> 40) & 0xfull) == 2ull;
}

__global__ void k_perm_from_keys(const unsigned long long* __restrict__ keys,
                                 const int* __restrict__ order0, long long n, int* __restrict__ perm,
                                 int* __restrict__ inv)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    const long long low = (long long)(k & 0xffffffffull);
    int o = key_is_rank(k) ? order0[low] : (int)low;
    perm[i] = o;
    inv[o] = (int)i;
}

__global__ void k_degree_new(const long long* __restrict__ off, const int* __restrict__ perm,
                             long long nsolve, long long* __restrict__ deg)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nsolve) return;
    int o = perm[i];
    deg[i] = off[o + 1] - off[o];
}

template <typename R>
__global__ void k_pack_entries(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                               const int* __restrict__ tets, const double* __restrict__ tet_w,
                               const double* __restrict__ vol, const int* __restrict__ tmat,
                               const int* __restrict__ perm, const int* __restrict__ inv,
                               const long long* __restrict__ eoff, long long nsolve,
                               typename PlaneT<R>::T* __restrict__ planes, long long E,
                               int* __restrict__ bad_volume);

template <>
__global__ void k_pack_entries<float>(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                                      const int* __restrict__ tets, const double* __restrict__ tet_w,
                                      const double* __restrict__ vol, const int* __restrict__ tmat,
                                      const int* __restrict__ perm, const int* __restrict__ inv,
                                      const long long* __restrict__ eoff, long long nsolve,
                                      float4* __restrict__ planes, long long E,
                                      int* __restrict__ bad_volume)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nsolve) return;
    int o = perm[i];
    long long base = eoff[i];
    for (long long k = off[o]; k < off[o + 1]; ++k, ++base) {
        unsigned val = inc[k];
        long long t = val >> 2;
        int s = (int)(val & 3u);
        int ks[3], j = 0;
        for (int q = 0; q < 4; ++q)
            if (q != s) ks[j++] = q;
        unsigned n[3];
        double w[9];
        for (j = 0; j < 3; ++j) {
            n[j] = (unsigned)inv[tets[4 * t + ks[j]]];
            for (int b = 0; b < 3; ++b) w[3 * j + b] = tet_w[12 * t + 3 * ks[j] + b];
        }
        // fp32 layout recomputes V from |det W| = 1/(6V): verify the inputs agree
        double d = w[0] * (w[4] * w[8] - w[5] * w[7]) - w[1] * (w[3] * w[8] - w[5] * w[6]) +
                   w[2] * (w[3] * w[7] - w[4] * w[6]);
        double vr = 1.0 / (6.0 * fabs(d));
        if (!(fabs(vr / vol[t] - 1.0) < 1e-5)) atomicExch(bad_volume, 1);
        unsigned m = (unsigned)tmat[t];
        unsigned u0 = n[0] | ((m & 7u) << VBD_ID_BITS);
        unsigned u1 = n[1] | (((m >> 3) & 7u) << VBD_ID_BITS);
        unsigned u2 = n[2] | (((m >> 6) & 7u) << VBD_ID_BITS);
        planes[base] = make_float4(__uint_as_float(u0), __uint_as_float(u1), __uint_as_float(u2),
                                   (float)w[0]);
        planes[E + base] = make_float4((float)w[1], (float)w[2], (float)w[3], (float)w[4]);
        planes[2 * E + base] = make_float4((float)w[5], (float)w[6], (float)w[7], (float)w[8]);
    }
}

template <>
__global__ void k_pack_entries<double>(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                                       const int* __restrict__ tets, const double* __restrict__ tet_w,
                                       const double* __restrict__ vol, const int* __restrict__ tmat,
                                       const int* __restrict__ perm, const int* __restrict__ inv,
                                       const long long* __restrict__ eoff, long long nsolve,
                                       double2* __restrict__ planes, long long E,
                                       int* __restrict__ bad_volume)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nsolve) return;
    int o = perm[i];
    long long base = eoff[i];
    for (long long k = off[o]; k < off[o + 1]; ++k, ++base) {
        unsigned val = inc[k];
        long long t = val >> 2;
        int s = (int)(val & 3u);
        int ks[3], j = 0;
        for (int q = 0; q < 4; ++q)
            if (q != s) ks[j++] = q;
        int n[3];
        double w[9];
        for (j = 0; j < 3; ++j) {
            n[j] = inv[tets[4 * t + ks[j]]];
            for (int b = 0; b < 3; ++b) w[3 * j + b] = tet_w[12 * t + 3 * ks[j] + b];
        }
        reinterpret_cast<int4*>(planes)[base] = make_int4(n[0], n[1], n[2], tmat[t]);
        planes[E + base] = make_double2(w[0], w[1]);
        planes[2 * E + base] = make_double2(w[2], w[3]);
        planes[3 * E + base] = make_double2(w[4], w[5]);
        planes[4 * E + base] = make_double2(w[6], w[7]);
        planes[5 * E + base] = make_double2(w[8], vol[t]);
    }
    (void)bad_volume;
}

// per-vertex material (solved vertices, colour-major order) when all incident tets agree
__global__ void k_vertex_material(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                                  const int* __restrict__ tmat, const int* __restrict__ perm,
                                  long long nsolve, int* __restrict__ vmat, int* __restrict__ mixed)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nsolve) return;
    int o = perm[i];
    int m = 0;
    for (long long k = off[o]; k < off[o + 1]; ++k) {
        int mk = tmat[inc[k] >> 2];
        if (k == off[o]) m = mk;
        else if (mk != m) atomicExch(mixed, 1);
    }
    vmat[i] = m;
}

template <typename R>
__global__ void k_mass_new(const double* __restrict__ mass_orig, const int* __restrict__ perm,
                           long long n, R* __restrict__ mass)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) mass[i] = (R)mass_orig[perm[i]];
}

// ---------------------------------------------------------------------------------------
// compact layout (entry kinds): lossless dictionary of the explicit entries' rest data.
// The key of an entry is the exact bit pattern of everything but its neighbour ids:
//   fp32: the nine fp32 slot-weight rows + material id (10 words)
//   fp64: the nine fp64 rows + V (20 words) + material id
// Structured grids and instanced objects have few distinct keys (a 5-tet grid: 10 rest
// shapes x 4 slots), so the 48/96-byte entry becomes one int4 {n0, n1, n2, kind}.

template <typename R> struct KindKey;
template <> struct KindKey<float> {
    static constexpr int KW = 10;
    static __device__ __forceinline__ void get(const float4* __restrict__ pl, long long E, long long k,
                                               unsigned* key, int* n)
    {
        const float4 a = pl[k], b = pl[E + k], c = pl[2 * E + k];
        const unsigned u0 = __float_as_uint(a.x), u1 = __float_as_uint(a.y), u2 = __float_as_uint(a.z);
        n[0] = (int)(u0 & VBD_ID_MASK);
        n[1] = (int)(u1 & VBD_ID_MASK);
        n[2] = (int)(u2 & VBD_ID_MASK);
        key[0] = __float_as_uint(a.w);
        key[1] = __float_as_uint(b.x); key[2] = __float_as_uint(b.y);
        key[3] = __float_as_uint(b.z); key[4] = __float_as_uint(b.w);
        key[5] = __float_as_uint(c.x); key[6] = __float_as_uint(c.y);
        key[7] = __float_as_uint(c.z); key[8] = __float_as_uint(c.w);
        key[9] = (u0 >> VBD_ID_BITS) | ((u1 >> VBD_ID_BITS) << 3) | ((u2 >> VBD_ID_BITS) << 6);
    }
};
template <> struct KindKey<double> {
    static constexpr int KW = 21;
    static __device__ __forceinline__ void get(const double2* __restrict__ pl, long long E, long long k,
                                               unsigned* key, int* n)
    {
        const int4 a = reinterpret_cast<const int4*>(pl)[k];
        n[0] = a.x; n[1] = a.y; n[2] = a.z;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const uint4 v = reinterpret_cast<const uint4*>(pl)[(q + 1) * E + k];
            key[4 * q] = v.x; key[4 * q + 1] = v.y; key[4 * q + 2] = v.z; key[4 * q + 3] = v.w;
        }
        key[20] = (unsigned)a.w;
    }
};

template <int KW> __device__ __forceinline__ unsigned kind_hash(const unsigned* key)
{
    unsigned h = 0x9e3779b9u;
#pragma unroll
    for (int i = 0; i < KW; ++i) {
        unsigned x = key[i] * 0xcc9e2d51u;
        x = (x << 15) | (x >> 17);
        h ^= x * 0x1b873593u;
        h = ((h << 13) | (h >> 19)) * 5u + 0xe6546b64u;
    }
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    return h;
}

// slots: 0 = empty, else (representative entry index + 1)
template <typename R>
__device__ __forceinline__ long long kind_find(const typename PlaneT<R>::T* __restrict__ pl, long long E,
                                               unsigned long long* slots, unsigned mask, const unsigned* key,
                                               long long k, bool insert, int* count, int cap, int* overflow)
{
    constexpr int KW = KindKey<R>::KW;
    const unsigned h = kind_hash<KW>(key);
    for (unsigned probe = 0; probe <= mask; ++probe) {
        const unsigned s = (h + probe) & mask;
        unsigned long long cur = *(volatile unsigned long long*)(slots + s);
        if (cur == 0) {
            if (!insert) return -1;
            cur = atomicCAS(slots + s, 0ull, (unsigned long long)(k + 1));
            if (cur == 0) {
                if (atomicAdd(count, 1) >= cap) atomicExch(overflow, 1);
                return s;
            }
        }
        unsigned rk[KW];
        int rn[3];
        KindKey<R>::get(pl, E, (long long)cur - 1, rk, rn);
        bool eq = true;
#pragma unroll
        for (int i = 0; i < KW; ++i) eq = eq && rk[i] == key[i];
        if (eq) return s;
        if (insert && *(volatile int*)overflow) return -1;
    }
    if (insert) atomicExch(overflow, 1);
    return -1;
}

template <typename R>
__global__ void k_kind_insert(const typename PlaneT<R>::T* __restrict__ pl, long long E,
                              unsigned long long* slots, unsigned mask, int* count, int cap, int* overflow)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < E;
         k += (long long)gridDim.x * blockDim.x) {
        if (*(volatile int*)overflow) return;
        unsigned key[KindKey<R>::KW];
        int n[3];
        KindKey<R>::get(pl, E, k, key, n);
        kind_find<R>(pl, E, slots, mask, key, k, true, count, cap, overflow);
    }
}

template <typename R>
__global__ void k_kind_emit(const typename PlaneT<R>::T* __restrict__ pl, long long E,
                            unsigned long long* slots, unsigned mask, const int* __restrict__ slot_kind,
                            int4* __restrict__ out, int* missing)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < E;
         k += (long long)gridDim.x * blockDim.x) {
        unsigned key[KindKey<R>::KW];
        int n[3];
        KindKey<R>::get(pl, E, k, key, n);
        const long long s = kind_find<R>(pl, E, slots, mask, key, k, false, nullptr, 0, nullptr);
        if (s < 0) {
            atomicExch(missing, 1);
            continue;
        }
        out[k] = make_int4(n[0], n[1], n[2], slot_kind[s]);
    }
}

// keys of the representatives, kind-major
template <typename R>
__global__ void k_kind_keys(const typename PlaneT<R>::T* __restrict__ pl, long long E,
                            const long long* __restrict__ rep, int nk, unsigned* __restrict__ keys)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nk) return;
    int n[3];
    KindKey<R>::get(pl, E, rep[i], keys + (long long)i * KindKey<R>::KW, n);
}

// kind records (KindRec) for the current material table (refreshed when h changes)
template <typename R>
__global__ void k_kind_records(const unsigned* __restrict__ keys, int nk, const Material<R>* __restrict__ mats,
                               typename PlaneT<R>::T* __restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nk) return;
    constexpr int KW = KindKey<R>::KW;
    const unsigned* key = keys + (long long)i * KW;
    R w[9], V;
    if constexpr (sizeof(R) == 4) {
        for (int j = 0; j < 9; ++j) w[j] = __uint_as_float(key[j]);
        V = volume_from_rows(reinterpret_cast<const float*>(w));
    } else {
        for (int j = 0; j < 9; ++j) w[j] = __hiloint2double((int)key[2 * j + 1], (int)key[2 * j]);
        V = __hiloint2double((int)key[19], (int)key[18]);
    }
    const Material<R> m = mats[key[KW - 1]];
    R r[KindRec<R>::NR];
    ec_terms<R>(w, V, m.mu, m.lam, m.gamma, r);
    r[9] = m.dsc;
    r[10] = m.opd;
    r[11] = m.gamma;
    for (int j = 0; j < 9; ++j) r[12 + j] = w[j];
    r[21] = V;
    r[22] = m.mu;
    r[23] = m.lam;
    R* o = reinterpret_cast<R*>(out + (long long)i * KindRec<R>::Q);
    for (int j = 0; j < KindRec<R>::NR; ++j) o[j] = r[j];
}

// rest edges of every kind (fp32 displacement state): W^-1 of the key's three fp32 rows
__global__ void k_kind_edges(const unsigned* __restrict__ keys, int nk, float4* __restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nk) return;
    const unsigned* key = keys + (long long)i * KindKey<float>::KW;
    float w[9];
    for (int j = 0; j < 9; ++j) w[j] = __uint_as_float(key[j]);
    rest_edges_from_rows(w, out + 3LL * i);
}

__global__ void k_max_degree(const long long* __restrict__ eoff, long long n, int* out)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) atomicMax(out, (int)(eoff[i + 1] - eoff[i]));
}

// Rest-edge sign pattern of an entry (vertex role sl of tet t): E = W^-1 over the other three
// slot rows, column j = (w_{j+1} x w_{j+2}) / det W; each component's sign {-, 0, +} -> digit
// {0, 1, 2}, code = sum digit(E_j[k]) 3^(3 j + k) (< 3^9).  Zero below 1e-9 of the largest
// cofactor (a structured grid's axis-aligned edges).  tools/gen_grid_classes.py computes the
// same code from rest positions.
__device__ __forceinline__ unsigned entry_code(const double* __restrict__ w12, int sl)
{
    double w[9];
    int j = 0;
    for (int q = 0; q < 4; ++q) {
        if (q == sl) continue;
        for (int b = 0; b < 3; ++b) w[3 * j + b] = w12[3 * q + b];
        ++j;
    }
    double cr[9], m = 0.0;
    for (int c = 0; c < 3; ++c) {
        const double* a = w + 3 * ((c + 1) % 3);
        const double* b = w + 3 * ((c + 2) % 3);
        cr[3 * c + 0] = a[1] * b[2] - a[2] * b[1];
        cr[3 * c + 1] = a[2] * b[0] - a[0] * b[2];
        cr[3 * c + 2] = a[0] * b[1] - a[1] * b[0];
    }
    for (int i = 0; i < 9; ++i) m = fmax(m, fabs(cr[i]));
    const double det = w[0] * cr[0] + w[1] * cr[1] + w[2] * cr[2];
    const double tol = 1e-9 * m;
    unsigned code = 0, p = 1;
    for (int i = 0; i < 9; ++i, p *= 3) {
        const unsigned d = fabs(cr[i]) <= tol ? 1u : ((cr[i] > 0.0) == (det > 0.0) ? 2u : 0u);
        code += d * p;
    }
    return code;
}

// the kind hash of an entry (the exact rest data + material the layouts deduplicate)
template <typename R>
__device__ __forceinline__ unsigned entry_kind_hash(const double* __restrict__ tet_w, const double* __restrict__ vol,
                                                    const int* __restrict__ tmat, long long t, int sl)
{
    unsigned key[KindKey<R>::KW];
    int j = 0;
    for (int q = 0; q < 4; ++q) {
        if (q == sl) continue;
        for (int b = 0; b < 3; ++b) {
            const double w = tet_w[12 * t + 3 * q + b];
            if constexpr (sizeof(R) == 4) {
                key[3 * j + b] = __float_as_uint((float)w);
            } else {
                key[2 * (3 * j + b)] = (unsigned)__double2loint(w);
                key[2 * (3 * j + b) + 1] = (unsigned)__double2hiint(w);
            }
        }
        ++j;
    }
    if constexpr (sizeof(R) == 8) {
        key[18] = (unsigned)__double2loint(vol[t]);
        key[19] = (unsigned)__double2hiint(vol[t]);
    }
    key[KindKey<R>::KW - 1] = (unsigned)tmat[t];
    return kind_hash<KindKey<R>::KW>(key);
}

// Entry order within a vertex: by the entry's rest-edge sign pattern (entry_code), then by a
// hash of its kind key (the exact rest data the layouts deduplicate), ties in ascending (tet,
// slot) order.  Interior vertices of one class of a structured grid then list the same kinds
// in the same order -- independent of spacing and material -- so the lanes of a K1T
// quarter-warp (same entry position, 8 vertices) read the same kind record (smem broadcast),
// and K1T's class tiles can address the entries' neighbours by compile-time indices
// (vbd_grid_classes.cuh).  Every layout is packed from this one order, so they stay bitwise equal.
template <typename R>
__global__ void k_inc_kind_keys(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                                const double* __restrict__ tet_w, const double* __restrict__ vol,
                                const int* __restrict__ tmat, long long n, unsigned long long* __restrict__ keys,
                                int by_code = 1)
{
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    for (long long k = off[v]; k < off[v + 1]; ++k) {
        const unsigned val = inc[k];
        const long long t = val >> 2;
        const int sl = (int)(val & 3u);
        const unsigned h = entry_kind_hash<R>(tet_w, vol, tmat, t, sl);
        if (!by_code) {  // (VBD_ENTRY_ORDER=hash: the kind hash alone; no class tiles)
            keys[k] = ((unsigned long long)v << 32) | h;
            continue;
        }
        const unsigned code = entry_code(tet_w + 12 * t, sl);
        keys[k] = ((unsigned long long)v << 32) | ((unsigned long long)code << 17) | (h & 0x1ffffu);
    }
}

// Grid-class detection (original vertex order, after the entry sort): a vertex is of class c
// (vbd_grid_classes.cuh) when its entry count, every entry's pattern code and the neighbour
// identity implied by the class's local indices all match.  out_key = (c + 1) << 32 | a hash of
// its entries' kind hashes (the class instance: the same kinds at every position), else 0.
template <typename R>
__global__ void k_vertex_class(const long long* __restrict__ off, const unsigned* __restrict__ inc,
                               const int* __restrict__ tets, const double* __restrict__ tet_w,
                               const double* __restrict__ vol, const int* __restrict__ tmat, long long n,
                               unsigned long long* __restrict__ out_key)
{
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const long long e0 = off[v];
    const int d = (int)(off[v + 1] - e0);
    unsigned long long res = 0ull;
    for (int c = 0; c < VBD_GC_N && !res; ++c) {
        const int b = vbd_gc_beg[c];
        if (d != vbd_gc_beg[c + 1] - b) continue;
        int loc[VBD_GC_MAXNL];
        for (int i = 0; i < VBD_GC_MAXNL; ++i) loc[i] = -1;
        bool ok = true;
        unsigned h = 0x811c9dc5u;
        for (int q = 0; q < d && ok; ++q) {
            const unsigned val = inc[e0 + q];
            const long long t = val >> 2;
            const int sl = (int)(val & 3u);
            if (entry_code(tet_w + 12 * t, sl) != vbd_gc_code[b + q]) {
                ok = false;
                break;
            }
            int r = 0;
            for (int q4 = 0; q4 < 4; ++q4) {
                if (q4 == sl) continue;
                const int id = tets[4 * t + q4];
                const int li = vbd_gc_nbr[3 * (b + q) + r];
                if (loc[li] < 0) loc[li] = id;
                else if (loc[li] != id) ok = false;
                ++r;
            }
            h = (h ^ entry_kind_hash<R>(tet_w, vol, tmat, t, sl)) * 0x01000193u;
        }
        if (ok) res = ((unsigned long long)(c + 1) << 32) | h;
    }
    out_key[v] = res;
}

// the distinct nonzero class keys into a small open-addressing table (cap slots, 0 = empty);
// *overflow set when more than cap distinct keys
__global__ void k_class_keys_insert(const unsigned long long* __restrict__ key, long long n,
                                    unsigned long long* __restrict__ table, int cap, int* __restrict__ overflow)
{
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const unsigned long long k = key[v];
    if (!k) return;
    unsigned s = (unsigned)((k * 0x9e3779b97f4a7c15ull) >> 40) % (unsigned)cap;
    for (int p = 0; p < cap; ++p, s = (s + 1) % (unsigned)cap) {
        unsigned long long cur = *(volatile unsigned long long*)(table + s);
        if (cur == k) return;
        if (cur == 0ull) {
            cur = atomicCAS(table + s, 0ull, k);
            if (cur == 0ull || cur == k) return;
        }
    }
    atomicExch(overflow, 1);
}

// per vertex: its class instance (index of its key in the host-sorted key list), or -1
__global__ void k_class_instance(const unsigned long long* __restrict__ key, long long n,
                                 const unsigned long long* __restrict__ sorted, int nkeys, signed char* __restrict__ inst)
{
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const unsigned long long k = key[v];
    int r = -1;
    for (int i = 0; i < nkeys && k; ++i)
        if (sorted[i] == k) r = i;
    inst[v] = (signed char)r;
}
