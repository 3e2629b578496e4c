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
        // V = 1 / (6 |det W|): |det| of the three non-own slot-weight rows equals |det Dm^-1|
        float d = e.w[0] * (e.w[4] * e.w[8] - e.w[5] * e.w[7]) -
                  e.w[1] * (e.w[3] * e.w[8] - e.w[5] * e.w[6]) +
                  e.w[2] * (e.w[3] * e.w[7] - e.w[4] * e.w[6]);
        e.V = __fdividef(1.0f / 6.0f, fabsf(d));
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
// per-entry Stable Neo-Hookean force/Hessian + Rayleigh damping, the arithmetic of
// _native.pyx:283-317 (F, cofactor and J of _native.pyx:175-198) in edge-difference form.
//   f  -= V (mu F w + lam (J - gamma) C w) + dsc He (x_i - x_t,i)
//   H  += (1 + dsc) He,  He = V (lam (C w)(C w)^T + mu |w|^2 I)
// H is kept as 6 unique entries (xx, xy, xz, yy, yz, zz).
template <typename R, bool DAMP = true>
__device__ __forceinline__ void tet_contrib(const R* __restrict__ e0, const R* __restrict__ e1,
                                            const R* __restrict__ e2, const R* __restrict__ w,
                                            R V, const Material<R>& m, const R* __restrict__ dx,
                                            R* __restrict__ f, R* __restrict__ H)
{
    R F[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) F[a * 3 + b] = e0[a] * w[b] + e1[a] * w[3 + b] + e2[a] * w[6 + b];
    R wo[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) wo[b] = -((w[b] + w[3 + b]) + w[6 + b]);
    R C[9];
    C[0] = F[4] * F[8] - F[7] * F[5];
    C[3] = F[7] * F[2] - F[1] * F[8];
    C[6] = F[1] * F[5] - F[4] * F[2];
    C[1] = F[5] * F[6] - F[8] * F[3];
    C[4] = F[8] * F[0] - F[2] * F[6];
    C[7] = F[2] * F[3] - F[5] * F[0];
    C[2] = F[3] * F[7] - F[6] * F[4];
    C[5] = F[6] * F[1] - F[0] * F[7];
    C[8] = F[0] * F[4] - F[3] * F[1];
    R J = F[0] * C[0] + F[3] * C[3] + F[6] * C[6];
    R cw[3], Fw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        cw[a] = C[a * 3 + 0] * wo[0] + C[a * 3 + 1] * wo[1] + C[a * 3 + 2] * wo[2];
        Fw[a] = F[a * 3 + 0] * wo[0] + F[a * 3 + 1] * wo[1] + F[a * 3 + 2] * wo[2];
    }
    R wsq = wo[0] * wo[0] + wo[1] * wo[1] + wo[2] * wo[2];
    R coef = m.lam * (J - m.gamma);
    R vl = V * m.lam, vmw = V * m.mu * wsq;
    R he[6];
    he[0] = vl * cw[0] * cw[0] + vmw;
    he[1] = vl * cw[0] * cw[1];
    he[2] = vl * cw[0] * cw[2];
    he[3] = vl * cw[1] * cw[1] + vmw;
    he[4] = vl * cw[1] * cw[2];
    he[5] = vl * cw[2] * cw[2] + vmw;
    if (DAMP) {
        R hd0 = he[0] * dx[0] + he[1] * dx[1] + he[2] * dx[2];
        R hd1 = he[1] * dx[0] + he[3] * dx[1] + he[4] * dx[2];
        R hd2 = he[2] * dx[0] + he[4] * dx[1] + he[5] * dx[2];
        f[0] -= V * (m.mu * Fw[0] + coef * cw[0]) + m.dsc * hd0;
        f[1] -= V * (m.mu * Fw[1] + coef * cw[1]) + m.dsc * hd1;
        f[2] -= V * (m.mu * Fw[2] + coef * cw[2]) + m.dsc * hd2;
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] += m.opd * he[q];
    } else {
        // one material per vertex: sum the undamped blocks; the caller applies
        // f -= dsc * (sum He) dx and H = (1 + dsc) sum He once per vertex
        f[0] -= V * (m.mu * Fw[0] + coef * cw[0]);
        f[1] -= V * (m.mu * Fw[1] + coef * cw[1]);
        f[2] -= V * (m.mu * Fw[2] + coef * cw[2]);
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] += he[q];
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
    // full symmetric matrix [H0 H1 H2; H1 H3 H4; H2 H4 H5]
    R a0 = H[3] * H[5] - H[4] * H[4];
    R a1 = H[2] * H[4] - H[1] * H[5];
    R a2 = H[1] * H[4] - H[2] * H[3];
    R a4 = H[0] * H[5] - H[2] * H[2];
    R a5 = H[2] * H[1] - H[0] * H[4];
    R a8 = H[0] * H[3] - H[1] * H[1];
    R det = H[0] * a0 + H[1] * a1 + H[2] * a2;
    R tr = (H[0] + H[3] + H[5]) / R(3);
    if (fabs(det) > eps_det * tr * tr * tr) {
        d[0] = (a0 * f[0] + a1 * f[1] + a2 * f[2]) / det;
        d[1] = (a1 * f[0] + a4 * f[1] + a5 * f[2]) / det;
        d[2] = (a2 * f[0] + a5 * f[1] + a8 * f[2]) / det;
    }
}

__device__ __forceinline__ bool finite3(double a, double b, double c)
{
    return isfinite(a) && isfinite(b) && isfinite(c);
}
