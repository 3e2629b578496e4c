// vbd_common.cuh -- shared types and device math for the B200 VBD hot path.
//
// Layout summary (see DESIGN.md for the byte accounting):
//   * vertices are renumbered colour-major: [free vertices sorted by (colour, rounds, id)]
//     [ghosts (halo copies, multi-GPU slabs)] [fixed vertices]; the colour pass for colour c
//     is one contiguous range [cbeg[c], cend[c]).
//   * per-vertex state is one array per field (x, x_t, y, v_t, v_prev, Chebyshev history),
//     each an array of R4 = float4/double4 so a neighbour gather is one 16/32-byte load.
//   * the vertex->tet adjacency is a CSR over free vertices in that order; entry k of vertex
//     i describes one incident tet *relative to i*: the three other vertex ids n_j and the
//     three matching slot-weight rows w_j = Dm^-T rows (reference tet_w, _system.py:139-144),
//     so that F = sum_j (x_{n_j} - x_i) w_j^T and i's own row is w_i = -(w_0 + w_1 + w_2).
//     Entries are stored as 16-byte planes (struct-of-arrays): one LDG.128 per plane per
//     lane, fully coalesced for consecutive entries.
//       fp32: 3 planes = 48 B/entry  {n0|m, n1|m, n2|m, w0} {w1..w4} {w5..w8}
//             (material id in the top 3 bits of each id; V = 1/(6|det W|) recomputed)
//       fp64: 6 planes = 96 B/entry  {n0,n1,n2,mat} {w0,w1} {w2,w3} {w4,w5} {w6,w7} {w8,V}
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define VBD_MAX_MATERIALS 512
#define VBD_ID_BITS 29
#define VBD_ID_MASK ((1u << VBD_ID_BITS) - 1u)

template <typename R> struct Vec4;
template <> struct Vec4<float> { typedef float4 T; };
template <> struct Vec4<double> { typedef double4 T; };

// Per-material constants for one step size h (host computes gamma = 1 + mu/lam exactly as
// the reference does per tet, _native.pyx:291; dsc = kd/h, _native.pyx:309).
template <typename R> struct Material {
    R mu, lam, gamma, dsc, opd;  // opd = 1 + dsc
};

// number of 16-byte planes per entry
template <typename R> struct EntryPlanes;
template <> struct EntryPlanes<float> { static constexpr int P = 3; };
template <> struct EntryPlanes<double> { static constexpr int P = 6; };

struct StepFlag {  // first non-finite (step, iteration, vertex) as a 64-bit min key
    static __host__ __device__ inline unsigned long long key(unsigned step, unsigned iter,
                                                             unsigned vertex) {
        return ((unsigned long long)(step & 0xffffu) << 48) |
               ((unsigned long long)(iter & 0xffffu) << 32) | (unsigned long long)vertex;
    }
    static constexpr unsigned long long NONE = ~0ull;
};

// ---------------------------------------------------------------------------------------
// entry access

// V = 1 / (6 |det W|): |det| of the three non-own slot-weight rows equals |det Dm^-1|
// (fp32 layouts recompute the rest volume instead of storing it)
// Every product is pinned (explicit fma / mul.rn, never re-contracted by the compiler) so the
// explicit layout (recomputed in K1) and the compact layout's kind table (computed once in
// k_kind_records) round identically.
__device__ __forceinline__ float volume_from_rows(const float* w)
{
    const float m1 = __fmaf_rn(w[4], w[8], -__fmul_rn(w[5], w[7]));
    const float m2 = __fmaf_rn(w[3], w[8], -__fmul_rn(w[5], w[6]));
    const float m3 = __fmaf_rn(w[3], w[7], -__fmul_rn(w[4], w[6]));
    const float d = __fmaf_rn(w[2], m3, __fmaf_rn(-w[1], m2, __fmul_rn(w[0], m1)));
    return __fdividef(1.0f / 6.0f, fabsf(d));
}

// fp32 displacement state: positions are stored as u = x - X (rest), so an
// edge is e_j = E_j + (u_nj - u_i) with the REST edges E = W^-1 (F = E W = I at rest; column
// j of W^-1 is (w_{j+1} x w_{j+2}) / det W over the entry's three other slot rows).  E is a
// function of the fp32 rows only, in fp32 with every operation pinned, so the kind table
// (k_kind_edges, once) and the explicit layout (per entry, per pass: ~30 instructions) agree
// bitwise.  out: E_0 (xyz), E_1, E_2 as 3 float4 (w = 0).
__device__ __forceinline__ void rest_edges_from_rows(const float* w, float4* out)
{
    float cr[3][3];  // cr[j] = w_{j+1} x w_{j+2}
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const float* a = w + 3 * ((j + 1) % 3);
        const float* b = w + 3 * ((j + 2) % 3);
        cr[j][0] = __fmaf_rn(a[1], b[2], -__fmul_rn(a[2], b[1]));
        cr[j][1] = __fmaf_rn(a[2], b[0], -__fmul_rn(a[0], b[2]));
        cr[j][2] = __fmaf_rn(a[0], b[1], -__fmul_rn(a[1], b[0]));
    }
    const float det = __fmaf_rn(w[2], cr[0][2], __fmaf_rn(w[1], cr[0][1], __fmul_rn(w[0], cr[0][0])));
    const float inv = __fdiv_rn(1.0f, det);
#pragma unroll
    for (int j = 0; j < 3; ++j)
        out[j] = make_float4(__fmul_rn(cr[j][0], inv), __fmul_rn(cr[j][1], inv), __fmul_rn(cr[j][2], inv), 0.0f);
}

// e_j = E_j + (p_j - x_i) (displacement state, has) or p_j - x_i (absolute state)
template <typename R>
__device__ __forceinline__ void edge3(const typename Vec4<R>::T& p, const R* xi, const float4& ex, bool has, R* e)
{
    e[0] = p.x - xi[0];
    e[1] = p.y - xi[1];
    e[2] = p.z - xi[2];
    if (has) {
        e[0] = (R)ex.x + e[0];
        e[1] = (R)ex.y + e[1];
        e[2] = (R)ex.z + e[2];
    }
}

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename R> struct Entry;

template <> struct Entry<float> {
    int n[3];
    int mat;
    float w[9];
    float V;
    static __device__ __forceinline__ Entry load(const float4* __restrict__ planes, long long E,
                                                 long long k) {
        Entry e;
        float4 a = __ldg(planes + k);
        float4 b = __ldg(planes + E + k);
        float4 c = __ldg(planes + 2 * E + k);
        unsigned u0 = __float_as_uint(a.x), u1 = __float_as_uint(a.y), u2 = __float_as_uint(a.z);
        e.n[0] = (int)(u0 & VBD_ID_MASK);
        e.n[1] = (int)(u1 & VBD_ID_MASK);
        e.n[2] = (int)(u2 & VBD_ID_MASK);
        e.mat = (int)((u0 >> VBD_ID_BITS) | ((u1 >> VBD_ID_BITS) << 3) | ((u2 >> VBD_ID_BITS) << 6));
        e.w[0] = a.w;
        e.w[1] = b.x; e.w[2] = b.y; e.w[3] = b.z; e.w[4] = b.w;
        e.w[5] = c.x; e.w[6] = c.y; e.w[7] = c.z; e.w[8] = c.w;
        e.V = volume_from_rows(e.w);
        return e;
    }
};

template <> struct Entry<double> {
    int n[3];
    int mat;
    double w[9];
    double V;
    static __device__ __forceinline__ Entry load(const double2* __restrict__ planes, long long E,
                                                 long long k) {
        Entry e;
        int4 a = __ldg(reinterpret_cast<const int4*>(planes) + k);
        e.n[0] = a.x; e.n[1] = a.y; e.n[2] = a.z; e.mat = a.w;
        double2 p1 = __ldg(planes + E + k), p2 = __ldg(planes + 2 * E + k),
                p3 = __ldg(planes + 3 * E + k), p4 = __ldg(planes + 4 * E + k),
                p5 = __ldg(planes + 5 * E + k);
        e.w[0] = p1.x; e.w[1] = p1.y; e.w[2] = p2.x; e.w[3] = p2.y; e.w[4] = p3.x;
        e.w[5] = p3.y; e.w[6] = p4.x; e.w[7] = p4.y; e.w[8] = p5.x; e.V = p5.y;
        return e;
    }
};

template <typename R> struct PlaneT;
template <> struct PlaneT<float> { typedef float4 T; };
template <> struct PlaneT<double> { typedef double2 T; };

// ---------------------------------------------------------------------------------------
// Per-entry Stable Neo-Hookean force/Hessian + Rayleigh damping of _native.pyx:283-317
// (F, cofactor and J of _native.pyx:175-198):
//   f  -= V (mu F w + lam (J - gamma) C w) + dsc He (x_i - x_t,i)
//   H  += (1 + dsc) He,  He = V (lam (C w)(C w)^T + mu |w|^2 I)
// with w the vertex's own slot-weight row.  Only F w and C w are needed, never F itself.
// Write the edges e_j = x_{n_j} - x_i as the columns of E and the other three slot rows
// as the rows of W (F = E W, reference tet_w, _system.py:139-144).  Then
//   F w = E s,          s_j = w_j . w
//   C w = cof(E) q,     q = cof(W) w            (cof(E W) = cof(E) cof(W))
//   J   = det(E) det(W)
// and cof(E) q = (q0 e1 - q1 e0) x e2 + q2 (e0 x e1), det(E) = e2 . (e0 x e1).
// s, q, det W, V lam and V mu |w|^2 depend only on the rest shape and material: ec_terms()
// computes them (once per entry kind in the compact layout, per entry in the explicit one)
// and tet_contrib_ec() is ~60 FP instructions per entry instead of ~130 for the F-form.
//
// Every multiply-add is written out (fma / mul_rn are never re-contracted by the compiler),
// so all K1 variants -- explicit or compact entries, global or shared-memory staging -- round
// identically and give bitwise equal results.
// H is kept as 6 unique entries (xx, xy, xz, yy, yz, zz).

template <typename R> __device__ __forceinline__ R dot3(const R* a, const R* b)
{
    return fma(a[2], b[2], fma(a[1], b[1], mul_rn(a[0], b[0])));
}
template <typename R> __device__ __forceinline__ void cross3(const R* a, const R* b, R* c)
{
    c[0] = fma(a[1], b[2], -mul_rn(a[2], b[1]));
    c[1] = fma(a[2], b[0], -mul_rn(a[0], b[2]));
    c[2] = fma(a[0], b[1], -mul_rn(a[1], b[0]));
}

// With r = sqrt(V lam) folded into q, det W and gamma, the Hessian block is (r C w)(r C w)^T
// and the force term r (J - gamma) (r C w): per entry kind
//   t[0..2] = V mu s,  t[3..5] = r q,  t[6] = r det W,  t[7] = r gamma,  t[8] = V mu |w|^2
template <typename R>
__device__ __forceinline__ void ec_terms(const R* __restrict__ w, R V, R mu, R lam, R gamma, R* __restrict__ t)
{
    R wo[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) wo[b] = -((w[b] + w[3 + b]) + w[6 + b]);  // own row
    const R vmu = mul_rn(V, mu);
    const R r = sqrt(mul_rn(V, lam));
#pragma unroll
    for (int j = 0; j < 3; ++j) t[j] = mul_rn(vmu, dot3(w + 3 * j, wo));
    R c[3];
    cross3(w + 3, w + 6, c);
    t[3] = mul_rn(r, dot3(c, wo));
    t[6] = mul_rn(r, dot3(w, c));
    cross3(w + 6, w, c);
    t[4] = mul_rn(r, dot3(c, wo));
    cross3(w, w + 3, c);
    t[5] = mul_rn(r, dot3(c, wo));
    t[7] = mul_rn(r, gamma);
    t[8] = mul_rn(vmu, dot3(wo, wo));
}

// DAMP = false: one material per vertex -- the undamped block is accumulated (H and the
// scalar sum sv of V mu |w|^2) and the caller applies damping once per vertex.
// ~50 FP instructions per entry (the F-form needs ~130).
template <typename R, bool DAMP>
__device__ __forceinline__ void tet_contrib_ec(const R* __restrict__ e0, const R* __restrict__ e1,
                                               const R* __restrict__ e2, const R* __restrict__ t, R dsc, R opd,
                                               const R* __restrict__ dx, R* __restrict__ f,
                                               R* __restrict__ H, R& sv)
{
    R u[3], c[3], k[3], cw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = fma(t[3], e1[a], -mul_rn(t[4], e0[a]));
    cross3(e0, e1, c);
    cross3(u, e2, k);
#pragma unroll
    for (int a = 0; a < 3; ++a) cw[a] = fma(t[5], c[a], k[a]);  // r C w
    const R vc = fma(t[6], dot3(e2, c), -t[7]);                  // r (J - gamma)
    if (DAMP) {
        R g[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)  // V (mu F w + lam (J - gamma) C w)
            g[a] = fma(vc, cw[a], fma(t[2], e2[a], fma(t[1], e1[a], mul_rn(t[0], e0[a]))));
        R he[6];
        he[0] = fma(cw[0], cw[0], t[8]);
        he[1] = mul_rn(cw[0], cw[1]);
        he[2] = mul_rn(cw[0], cw[2]);
        he[3] = fma(cw[1], cw[1], t[8]);
        he[4] = mul_rn(cw[1], cw[2]);
        he[5] = fma(cw[2], cw[2], t[8]);
        const R hd[3] = {fma(he[2], dx[2], fma(he[1], dx[1], mul_rn(he[0], dx[0]))),
                         fma(he[4], dx[2], fma(he[3], dx[1], mul_rn(he[1], dx[0]))),
                         fma(he[5], dx[2], fma(he[4], dx[1], mul_rn(he[2], dx[0])))};
#pragma unroll
        for (int a = 0; a < 3; ++a) f[a] = f[a] - fma(dsc, hd[a], g[a]);
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] = fma(opd, he[q], H[q]);
    } else {
#pragma unroll
        for (int a = 0; a < 3; ++a)  // f -= V (mu F w + lam (J - gamma) C w), one FFMA per term
            f[a] = fma(-vc, cw[a], fma(-t[2], e2[a], fma(-t[1], e1[a], fma(-t[0], e0[a], f[a]))));
        H[0] = fma(cw[0], cw[0], H[0]);
        H[1] = fma(cw[0], cw[1], H[1]);
        H[2] = fma(cw[0], cw[2], H[2]);
        H[3] = fma(cw[1], cw[1], H[3]);
        H[4] = fma(cw[1], cw[2], H[4]);
        H[5] = fma(cw[2], cw[2], H[5]);
        (void)sv;  // V mu |w|^2 (t[8]) is summed once per vertex at pack time (k_vertex_sv)
    }
}

// ---------------------------------------------------------------------------------------
// compact layout ("entry kinds"): an entry is one int4 {n0, n1, n2, kind} (16 B) and the
// per-kind constants live in a small table (L1/L2-resident).  Lossless: kinds are
// deduplicated on the exact bits of the explicit entry (rows, volume, material), and both
// layouts derive the constants with ec_terms, so they produce bitwise identical results.
// Record (24 R): [0..8] ec_terms, [9] dsc, [10] opd, [11] gamma  (the sweep reads these 12)
//                [12..20] w0..w8, [21] V, [22] mu, [23] lam     (local energy / line search)
template <typename R> struct KindRec {
    static constexpr int NR = 24;
    static constexpr int HOT = 12;
    static constexpr int Q = NR * (int)sizeof(R) / 16;    // 16-byte chunks per record
    static constexpr int QH = HOT * (int)sizeof(R) / 16;  // chunks the sweep loads
};

struct EntryK {
    int n[3];
    int kind;
    static __device__ __forceinline__ EntryK load(const int4* __restrict__ ent, long long k)
    {
        // the entry stream is touched once per pass: keep it out of L1 (positions and the
        // kind table live there)
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(ent + k));
        EntryK e;
        e.n[0] = v.x; e.n[1] = v.y; e.n[2] = v.z; e.kind = v.w;
        return e;
    }
};

// load the first NQ 16-byte chunks of kind record `kind` into r (R[4*NQ*16/sizeof(R)/4])
template <typename R, int NQ>
__device__ __forceinline__ void load_kind(const typename PlaneT<R>::T* __restrict__ kinds, int kind, R* r)
{
    typedef typename PlaneT<R>::T PL;
    const PL* p = kinds + (long long)kind * KindRec<R>::Q;
    constexpr int PER = 16 / (int)sizeof(R);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const PL v = __ldg(p + q);
        const R* vr = reinterpret_cast<const R*>(&v);
#pragma unroll
        for (int j = 0; j < PER; ++j) r[q * PER + j] = vr[j];
    }
}

// Guarded 3x3 block solve of _native.pyx:465-479 on the symmetric H (6 unique entries):
// skip (delta = 0) when |det| <= eps_det * (tr/3)^3.  mode 1 = diagonal GD (_native.pyx:431-434).
template <typename R>
__device__ __forceinline__ void block_solve(const R* f, const R* H, R eps_det, int mode, R* d)
{
    d[0] = d[1] = d[2] = R(0);
    if (mode == 1) {
        if (H[0] != R(0)) d[0] = f[0] / H[0];
        if (H[3] != R(0)) d[1] = f[1] / H[3];
        if (H[5] != R(0)) d[2] = f[2] / H[5];
        return;
    }
    // full symmetric matrix [H0 H1 H2; H1 H3 H4; H2 H4 H5] (products pinned, see above)
    const R a0 = fma(H[3], H[5], -mul_rn(H[4], H[4]));
    const R a1 = fma(H[2], H[4], -mul_rn(H[1], H[5]));
    const R a2 = fma(H[1], H[4], -mul_rn(H[2], H[3]));
    const R a4 = fma(H[0], H[5], -mul_rn(H[2], H[2]));
    const R a5 = fma(H[2], H[1], -mul_rn(H[0], H[4]));
    const R a8 = fma(H[0], H[3], -mul_rn(H[1], H[1]));
    const R det = fma(H[2], a2, fma(H[1], a1, mul_rn(H[0], a0)));
    const R tr = mul_rn((H[0] + H[3] + H[5]), R(1) / R(3));
    if (fabs(det) > mul_rn(mul_rn(mul_rn(eps_det, tr), tr), tr)) {
        const R inv = R(1) / det;  // one IEEE division per vertex
        d[0] = mul_rn(fma(a2, f[2], fma(a1, f[1], mul_rn(a0, f[0]))), inv);
        d[1] = mul_rn(fma(a5, f[2], fma(a4, f[1], mul_rn(a1, f[0]))), inv);
        d[2] = mul_rn(fma(a8, f[2], fma(a5, f[1], mul_rn(a2, f[0]))), inv);
    }
}

// inertia term (_native.pyx:278-281) and the hoisted Rayleigh damping of one material per
// vertex (_native.pyx:309-317 summed over the vertex's tets), pinned like tet_contrib_core
template <typename R>
__device__ __forceinline__ void vertex_terms(R* f, R* H, const R* dx, const R* xi, R y0, R y1, R y2,
                                             R mih2, bool damp, R dsc, R opd)
{
    if (damp) {
        const R hd0 = fma(H[2], dx[2], fma(H[1], dx[1], mul_rn(H[0], dx[0])));
        const R hd1 = fma(H[4], dx[2], fma(H[3], dx[1], mul_rn(H[1], dx[0])));
        const R hd2 = fma(H[5], dx[2], fma(H[4], dx[1], mul_rn(H[2], dx[0])));
        f[0] = f[0] - mul_rn(dsc, hd0);
        f[1] = f[1] - mul_rn(dsc, hd1);
        f[2] = f[2] - mul_rn(dsc, hd2);
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] = mul_rn(H[q], opd);
    }
    f[0] = fma(mih2, y0 - xi[0], f[0]);
    f[1] = fma(mih2, y1 - xi[1], f[1]);
    f[2] = fma(mih2, y2 - xi[2], f[2]);
    H[0] = H[0] + mih2;
    H[3] = H[3] + mih2;
    H[5] = H[5] + mih2;
}

template <typename R> __device__ __forceinline__ bool finite3(R a, R b, R c)
{
    return isfinite(a) && isfinite(b) && isfinite(c);
}

// ---------------------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-stream-
// serialization attribute may start while its predecessor drains; griddepcontrol.wait blocks
// until the predecessor grid has completed and its writes are visible, so everything before it
// must read constant data only.  Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// shared-memory address / mbarrier helpers (bulk-copy staging)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// the waiting warp is suspended (not spinning on issue slots) until the phase completes or
// the hint expires
#ifndef VBD_MBAR_SUSPEND_NS
#define VBD_MBAR_SUSPEND_NS 1000000u
#endif
__device__ __forceinline__ void mbar_wait_parity(unsigned bar, unsigned phase)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(bar), "r"(phase), "r"(VBD_MBAR_SUSPEND_NS) : "memory");
}


// ---------------------------------------------------------------------------------------
// tet_contrib_ec<float, false> with the x/y components of each 3-vector packed as fp32x2
// (FFMA2 / FMUL2 / FADD2 on sm_100; a scalar operand is broadcast to both halves).  The x/y
// pair of a position comes straight from its 16-byte shared-memory load; each component
// executes exactly the scalar operation sequence (round-to-nearest per component;
// x - a b == x + (-a) b), so results are bitwise those of tet_contrib_ec.  Cross products and
// the volume term stay scalar.  f is (f0, f1) + f2; H is (H0, H3), (H2, H4), H1, H5.
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

struct AccXY {
    float2 f01;    // f0, f1
    float f2;
    float2 h03;    // H0, H3
    float2 h24;    // H2, H4
    float h1, h5;
    __device__ __forceinline__ void zero()
    {
        f01 = h03 = h24 = make_float2(0.f, 0.f);
        f2 = h1 = h5 = 0.f;
    }
};

// the displacement difference u_k - u_i of one neighbour (x/y packed), formed once per
// neighbour by the class-tile sweep (the same operation tet_contrib_ec_xy does per use)
struct DiffXY {
    float2 xy;
    float z;
};
__device__ __forceinline__ DiffXY diff_xy(float4 p, float2 nxy, float nz)
{
    return DiffXY{add2(make_float2(p.x, p.y), nxy), p.z + nz};
}

__device__ __forceinline__ void tet_contrib_ec_xy_d(DiffXY d0, DiffXY d1, DiffXY d2, float4 x0, float4 x1, float4 x2,
                                                    const float* __restrict__ t, AccXY& A);

__device__ __forceinline__ void tet_contrib_ec_xy(float4 p0, float4 p1, float4 p2, float2 nxy, float nz,
                                                  float4 x0, float4 x1, float4 x2,
                                                  const float* __restrict__ t, AccXY& A)
{
    tet_contrib_ec_xy_d(diff_xy(p0, nxy, nz), diff_xy(p1, nxy, nz), diff_xy(p2, nxy, nz), x0, x1, x2, t, A);
}

__device__ __forceinline__ void tet_contrib_ec_xy_d(DiffXY d0, DiffXY d1, DiffXY d2, float4 x0, float4 x1, float4 x2,
                                                    const float* __restrict__ t, AccXY& A)
{
    // edges e_k = E_k + (u_k - u_i): rest edge x0..x2 plus the displacement difference (the
    // fp32 displacement state, edge3 / rest_edges_from_rows)
    const float2 e0 = add2(make_float2(x0.x, x0.y), d0.xy), e1 = add2(make_float2(x1.x, x1.y), d1.xy),
                 e2 = add2(make_float2(x2.x, x2.y), d2.xy);
    const float e0z = x0.z + d0.z, e1z = x1.z + d1.z, e2z = x2.z + d2.z;
    // u = t3 e1 - t4 e0
    const float2 u = fma2(bc2(t[3]), e1, mul2(bc2(-t[4]), e0));
    const float uz = __fmaf_rn(t[3], e1z, -__fmul_rn(t[4], e0z));
    // c = e0 x e1, k = u x e2 (scalar, as cross3)
    const float c0 = __fmaf_rn(e0.y, e1z, -__fmul_rn(e0z, e1.y));
    const float c1 = __fmaf_rn(e0z, e1.x, -__fmul_rn(e0.x, e1z));
    const float c2 = __fmaf_rn(e0.x, e1.y, -__fmul_rn(e0.y, e1.x));
    const float k0 = __fmaf_rn(u.y, e2z, -__fmul_rn(uz, e2.y));
    const float k1 = __fmaf_rn(uz, e2.x, -__fmul_rn(u.x, e2z));
    const float k2 = __fmaf_rn(u.x, e2.y, -__fmul_rn(u.y, e2.x));
    // r C w
    const float2 cw = fma2(bc2(t[5]), make_float2(c0, c1), make_float2(k0, k1));
    const float cwz = __fmaf_rn(t[5], c2, k2);
    // r (J - gamma)
    const float vc = __fmaf_rn(t[6], __fmaf_rn(e2z, c2, __fmaf_rn(e2.y, c1, __fmul_rn(e2.x, c0))), -t[7]);
    A.f01 = fma2(bc2(-vc), cw, fma2(bc2(-t[2]), e2, fma2(bc2(-t[1]), e1, fma2(bc2(-t[0]), e0, A.f01))));
    A.f2 = __fmaf_rn(-vc, cwz, __fmaf_rn(-t[2], e2z, __fmaf_rn(-t[1], e1z, __fmaf_rn(-t[0], e0z, A.f2))));
    A.h03 = fma2(cw, cw, A.h03);
    A.h24 = fma2(cw, bc2(cwz), A.h24);
    A.h1 = __fmaf_rn(cw.x, cw.y, A.h1);
    A.h5 = __fmaf_rn(cwz, cwz, A.h5);
}
