// vbd_kernels.cuh -- the sm_100a kernels of the VBD time step.
//
//   K1 k1_color_pass   per-colour Gauss-Seidel vertex update (_native.pyx:412-494, 582-589)
//   K2 k2_step_init    inertia target + adaptive warm start + fixed clamp (solver.py:120-164)
//   K3 k3_chebyshev    Chebyshev blend + history copy + non-finite check (solver.py:221-232,
//                      282-288, 312-315)
//   K4 k4_commit       v = (x - x_t)/h, rotate v_prev, x_t = x (solver.py:319-323)
//   plus state transfer (original <-> colour-major order), aux-buffer scatter and halo
//   pack/unpack for slab-decomposed scenes.
#pragma once
#include <cooperative_groups.h>

#include "vbd_common.cuh"

template <typename R> struct K1Args {
    typedef typename Vec4<R>::T R4;
    typedef typename PlaneT<R>::T PL;
    const PL* ent;           // entry planes (explicit layout) or int4 entries (compact)
    long long E;             // plane stride (entries)
    const PL* kinds;         // compact layout: kind table (KindRec); nullptr = explicit
    const R* vsv;            // one material per vertex: sum of V mu |w|^2 over its entries
    // fp32 displacement state (positions are x - X_rest): compact layout, the rest
    // edges of each kind (3 float4, k_kind_edges); explicit layout (disp), from the rows per
    // entry.  nullptr / 0: absolute positions (fp64, or fp32 after contacts were enabled)
    const float4* kedge;
    int disp;
    int max_deg;             // (host) max entries of one vertex: bulk-staging smem bound
    const long long* off;    // entry offsets of free vertices (nfree + 1)
    R4* pos;                 // current iterate x (in place)
    const R4* xt;            // x_t (w unused)
    const R4* y;             // inertia target, w = m / h^2
    const Material<R>* mat;  // per-material constants for this h
    const int* group;        // aux mode: vertex list (colour-major ids); nullptr = range
    int vbeg, count;         // range [vbeg, vbeg + count) or group[0..count)
    int nsolve;              // vertices >= nsolve are never solved (ghost / fixed)
    R4* out;                 // aux mode: results per group slot; nullptr = in place
    R eps_det;
    int mode;                // 0 block Newton, 1 diagonal GD
    unsigned long long* flag;  // non-finite report (nullptr = no check)
    const int* perm;         // colour-major -> original id (for the report)
    const int* stepctr;
    int iter;
    int pf_dist;             // L2 prefetch distance in CTAs (one residency wave)
    const int* vmat;         // per-vertex material when every vertex has one material, else null
    int line_search;         // 17-trial local backtracking (mode 0 only)
    // non-tet terms (host-built systems only; nullptr = none), solved vertices, colour-major:
    // spring CSR (other end, {l0, k, k_d}), world box {lo.xyz, k} {hi.xyz}, subspace index into
    // sub (3 R4: {b00 b01 b10 b11} {b20 b21 ax ay} {az dim})
    const long long* soff;
    const int* sp_oth;
    const R4* sp_par;
    const R4* box;
    const int* sub_idx;
    const R4* sub;
    R h;
    // contacts (ContactArrays, _system.py:86-96; nullptr = none): per solved vertex CSR of
    // (contact, slot); per contact cidx = 4 colour-major ids and creal = 4 R4:
    // {gamma0..3} {n.xyz, k_c} {t00 t01 t10 t11} {t20 t21 refresh 0}
    const long long* coff;
    const int* ccid;
    const int* cslot;
    const int4* cidx;
    const R4* creal;
    R mu_c, eps_u;
    // fused slab halo push (multi-GPU, peer memory): the first nb[0] vertices of the colour
    // range face the left neighbour, the next nb[1] the right one; their new positions are
    // also stored into the neighbour's ghost block (peer_pos[s] + peer_off[s])
    R4* peer_pos[2];
    int peer_off[2];
    int nb[2];
};

// The per-vertex body of K1: group g (W lanes, this thread is lane `lane`) solves vertex
// v = vbeg + g (or group[g]).  UM: one material per vertex (damping hoisted out of the loop).
// Local energy G_i of vertex v at position p (_native.pyx:201-258, tet + inertia terms),
// summed over the W lanes of the group (identical in every lane).
// Voronoi-region closest point on triangle abc, barycentric (_native.pyx:79-131)
template <typename R>
__device__ void closest_bary(const R* p, const R* a, const R* b, const R* c, R* bary)
{
    R ab[3], ac[3], ap[3], bp[3], cp[3];
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
    }
    const R d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    const R d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    if (d1 <= R(0) && d2 <= R(0)) { bary[0] = R(1); bary[1] = R(0); bary[2] = R(0); return; }
    for (int k = 0; k < 3; ++k) bp[k] = p[k] - b[k];
    const R d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    const R d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    if (d3 >= R(0) && d4 <= d3) { bary[0] = R(0); bary[1] = R(1); bary[2] = R(0); return; }
    const R vc = d1 * d4 - d3 * d2;
    if (vc <= R(0) && d1 >= R(0) && d3 <= R(0)) {
        const R v = d1 / (d1 - d3);
        bary[0] = R(1) - v; bary[1] = v; bary[2] = R(0);
        return;
    }
    for (int k = 0; k < 3; ++k) cp[k] = p[k] - c[k];
    const R d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    const R d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    if (d6 >= R(0) && d5 <= d6) { bary[0] = R(0); bary[1] = R(0); bary[2] = R(1); return; }
    const R vb = d5 * d2 - d1 * d6;
    if (vb <= R(0) && d2 >= R(0) && d6 <= R(0)) {
        const R w = d2 / (d2 - d6);
        bary[0] = R(1) - w; bary[1] = R(0); bary[2] = w;
        return;
    }
    const R va = d3 * d6 - d5 * d4;
    if (va <= R(0) && (d4 - d3) >= R(0) && (d5 - d6) >= R(0)) {
        const R w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        bary[0] = R(0); bary[1] = R(1) - w; bary[2] = w;
        return;
    }
    const R denom = R(1) / (va + vb + vc);
    const R v = vb * denom, w = vc * denom;
    bary[0] = R(1) - v - w; bary[1] = v; bary[2] = w;
}

// signed contact weights; DCD vertex-triangle anchors track the current closest point
// (_native.pyx:134-172)
template <typename R>
__device__ void contact_gamma(const K1Args<R>& a, int cid, R* gam)
{
    typedef typename Vec4<R>::T R4;
    const R4 g = a.creal[4 * cid], t3 = a.creal[4 * cid + 3];
    gam[0] = g.x; gam[1] = g.y; gam[2] = g.z; gam[3] = g.w;
    if (t3.z == R(0)) return;
    const int4 id = a.cidx[cid];
    const R4 pv = a.pos[id.x], p0 = a.pos[id.y], p1 = a.pos[id.z], p2 = a.pos[id.w];
    const R e1[3] = {p1.x - p0.x, p1.y - p0.y, p1.z - p0.z};
    const R e2[3] = {p2.x - p0.x, p2.y - p0.y, p2.z - p0.z};
    const R l1 = e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2];
    const R l2 = e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2];
    const R nr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const R nn = sqrt(nr[0] * nr[0] + nr[1] * nr[1] + nr[2] * nr[2]);
    R scale = l1 > l2 ? sqrt(l1) : sqrt(l2);
    if (scale < R(1e-30)) scale = R(1e-30);
    if (nn < R(1e-12) * scale * scale) return;
    const R P[3] = {pv.x, pv.y, pv.z}, A[3] = {p0.x, p0.y, p0.z}, B[3] = {p1.x, p1.y, p1.z},
            C[3] = {p2.x, p2.y, p2.z};
    R bary[3];
    closest_bary<R>(P, A, B, C, bary);
    gam[0] = R(1);
    gam[1] = -bary[0];
    gam[2] = -bary[1];
    gam[3] = -bary[2];
}

// contact penalty of G_i with vertex v at p (_native.pyx:239-249)
template <typename R>
__device__ R contact_energy(const K1Args<R>& a, int v, const R* p)
{
    typedef typename Vec4<R>::T R4;
    R e = R(0);
    for (long long kk = a.coff[v]; kk < a.coff[v + 1]; ++kk) {
        const int cid = a.ccid[kk], slot = a.cslot[kk];
        R gam[4];
        contact_gamma<R>(a, cid, gam);
        const int4 id = a.cidx[cid];
        const int ids[4] = {id.x, id.y, id.z, id.w};
        const R4 nk = a.creal[4 * cid + 1];
        R d = R(0);
        for (int k = 0; k < 4; ++k) {
            const R4 q = a.pos[ids[k]];
            const bool me = ids[k] == v && k == slot;
            d -= gam[k] * (nk.x * (me ? p[0] : q.x) + nk.y * (me ? p[1] : q.y) + nk.z * (me ? p[2] : q.z));
        }
        if (d > R(0)) e += R(0.5) * nk.w * d * d;
    }
    return e;
}

// contact penalty + friction force / Hessian of vertex v (_native.pyx:351-399)
template <typename R>
__device__ void contact_terms(const K1Args<R>& a, int v, R* f, R* H)
{
    typedef typename Vec4<R>::T R4;
    for (long long kk = a.coff[v]; kk < a.coff[v + 1]; ++kk) {
        const int cid = a.ccid[kk], slot = a.cslot[kk];
        R gam[4];
        contact_gamma<R>(a, cid, gam);
        const int4 id = a.cidx[cid];
        const int ids[4] = {id.x, id.y, id.z, id.w};
        const R4 nk = a.creal[4 * cid + 1];
        R d = R(0);
        for (int k = 0; k < 4; ++k) {
            const R4 q = a.pos[ids[k]];
            d -= gam[k] * (nk.x * q.x + nk.y * q.y + nk.z * q.z);
        }
        if (d <= R(0)) continue;
        const R n[3] = {nk.x, nk.y, nk.z};
        const R gs = gam[slot];
        R coef = nk.w * d * gs;
        for (int c = 0; c < 3; ++c) f[c] += coef * n[c];
        coef = nk.w * gs * gs;
        H[0] += coef * n[0] * n[0]; H[1] += coef * n[0] * n[1]; H[2] += coef * n[0] * n[2];
        H[3] += coef * n[1] * n[1]; H[4] += coef * n[1] * n[2]; H[5] += coef * n[2] * n[2];
        if (a.mu_c > R(0)) {
            const R4 ta = a.creal[4 * cid + 2], tb = a.creal[4 * cid + 3];
            const R T[3][2] = {{ta.x, ta.y}, {ta.z, ta.w}, {tb.x, tb.y}};
            const R lamc = nk.w * d;
            R dv[3] = {R(0), R(0), R(0)};
            for (int k = 0; k < 4; ++k) {
                const R4 q = a.pos[ids[k]], qt = a.xt[ids[k]];
                dv[0] += gam[k] * (q.x - qt.x);
                dv[1] += gam[k] * (q.y - qt.y);
                dv[2] += gam[k] * (q.z - qt.z);
            }
            const R u0 = T[0][0] * dv[0] + T[1][0] * dv[1] + T[2][0] * dv[2];
            const R u1 = T[0][1] * dv[0] + T[1][1] * dv[1] + T[2][1] * dv[2];
            const R un = sqrt(u0 * u0 + u1 * u1);
            R ratio;
            if (un < R(1e-14)) {
                ratio = R(2) / a.eps_u;
            } else {
                const R r = un / a.eps_u;
                const R f1 = un >= a.eps_u ? R(1) : R(2) * r - r * r;
                ratio = f1 / un;
                const R cf = -a.mu_c * lamc * gs * ratio;
                for (int c = 0; c < 3; ++c) f[c] += cf * (T[c][0] * u0 + T[c][1] * u1);
            }
            const R ch = a.mu_c * lamc * gs * gs * ratio;
            H[0] += ch * (T[0][0] * T[0][0] + T[0][1] * T[0][1]);
            H[1] += ch * (T[0][0] * T[1][0] + T[0][1] * T[1][1]);
            H[2] += ch * (T[0][0] * T[2][0] + T[0][1] * T[2][1]);
            H[3] += ch * (T[1][0] * T[1][0] + T[1][1] * T[1][1]);
            H[4] += ch * (T[1][0] * T[2][0] + T[1][1] * T[2][1]);
            H[5] += ch * (T[2][0] * T[2][0] + T[2][1] * T[2][1]);
        }
    }
}

// spring and world-box terms of G_i (_native.pyx:226-237, 250-257), vertex at p
template <typename R>
__device__ R extras_energy(const K1Args<R>& a, int v, const R* p)
{
    R e = R(0);
    if (a.soff)
    for (long long k = a.soff[v]; k < a.soff[v + 1]; ++k) {
        const typename Vec4<R>::T q = a.pos[a.sp_oth[k]], sp = a.sp_par[k];
        const R d0 = p[0] - q.x, d1 = p[1] - q.y, d2 = p[2] - q.z;
        const R len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        if (len < R(1e-12) * sp.x) {
            e += R(0.5) * sp.y * sp.x * sp.x;
        } else {
            const R t = len - sp.x;
            e += R(0.5) * sp.y * t * t;
        }
    }
    if (a.coff) e += contact_energy<R>(a, v, p);
    if (a.box) {
        const typename Vec4<R>::T lo = a.box[2 * v], hi = a.box[2 * v + 1];
        if (lo.w > R(0)) {
            const R l[3] = {lo.x, lo.y, lo.z}, u[3] = {hi.x, hi.y, hi.z};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                R t = l[c] - p[c];
                if (t > R(0)) e += R(0.5) * lo.w * t * t;
                t = p[c] - u[c];
                if (t > R(0)) e += R(0.5) * lo.w * t * t;
            }
        }
    }
    return e;
}

// spring (_native.pyx:319-349, per-spring Rayleigh damping) and world-box (:401-409) terms
template <typename R>
__device__ void extras_terms(const K1Args<R>& a, int v, const R* xi, const R* dx, R* f, R* H)
{
    if (a.soff)
    for (long long k = a.soff[v]; k < a.soff[v + 1]; ++k) {
        const typename Vec4<R>::T q = a.pos[a.sp_oth[k]], sp = a.sp_par[k];
        R dv[3] = {xi[0] - q.x, xi[1] - q.y, xi[2] - q.z};
        const R len = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
        R he[6];
        if (len < R(1e-12) * sp.x) {
            he[0] = he[3] = he[5] = sp.y;
            he[1] = he[2] = he[4] = R(0);
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) dv[c] = dv[c] / len;
            const R coef = R(1) - sp.x / len;
            const R fs = sp.y * (len - sp.x);
#pragma unroll
            for (int c = 0; c < 3; ++c) f[c] -= fs * dv[c];
            he[0] = sp.y * (dv[0] * dv[0] + coef * (R(1) - dv[0] * dv[0]));
            he[1] = sp.y * (dv[0] * dv[1] - coef * dv[0] * dv[1]);
            he[2] = sp.y * (dv[0] * dv[2] - coef * dv[0] * dv[2]);
            he[3] = sp.y * (dv[1] * dv[1] + coef * (R(1) - dv[1] * dv[1]));
            he[4] = sp.y * (dv[1] * dv[2] - coef * dv[1] * dv[2]);
            he[5] = sp.y * (dv[2] * dv[2] + coef * (R(1) - dv[2] * dv[2]));
        }
        const R dsc = sp.z / a.h;
        f[0] -= dsc * (he[0] * dx[0] + he[1] * dx[1] + he[2] * dx[2]);
        f[1] -= dsc * (he[1] * dx[0] + he[3] * dx[1] + he[4] * dx[2]);
        f[2] -= dsc * (he[2] * dx[0] + he[4] * dx[1] + he[5] * dx[2]);
#pragma unroll
        for (int c = 0; c < 6; ++c) H[c] += (R(1) + dsc) * he[c];
    }
    if (a.coff) contact_terms<R>(a, v, f, H);
    if (a.box) {
        const typename Vec4<R>::T lo = a.box[2 * v], hi = a.box[2 * v + 1];
        if (lo.w > R(0)) {
            const R l[3] = {lo.x, lo.y, lo.z}, u[3] = {hi.x, hi.y, hi.z};
            const int dg[3] = {0, 3, 5};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (xi[c] < l[c]) {
                    f[c] -= lo.w * (xi[c] - l[c]);
                    H[dg[c]] += lo.w;
                } else if (xi[c] > u[c]) {
                    f[c] -= lo.w * (xi[c] - u[c]);
                    H[dg[c]] += lo.w;
                }
            }
        }
    }
}

// SubspaceConstraint solve (_native.pyx:435-463): delta = B (B^T H B)^-1 B^T f, 1- or 2-D,
// with the reference's relative determinant guards.  H is symmetric (6 unique entries).
template <typename R>
__device__ void subspace_solve(const typename Vec4<R>::T* sub3, const R* f, const R* H, R eps_det, R* d)
{
    const typename Vec4<R>::T s0 = sub3[0], s1 = sub3[1], s2 = sub3[2];
    const R B[3][2] = {{s0.x, s0.y}, {s0.z, s0.w}, {s1.x, s1.y}};
    const int dim = (int)s2.y;
    const R Hm[3][3] = {{H[0], H[1], H[2]}, {H[1], H[3], H[4]}, {H[2], H[4], H[5]}};
    R rhs[2], am[2][2];
    for (int p = 0; p < dim; ++p) {
        rhs[p] = B[0][p] * f[0] + B[1][p] * f[1] + B[2][p] * f[2];
        for (int q = 0; q < dim; ++q) {
            R acc = R(0);
#pragma unroll
            for (int k = 0; k < 3; ++k)
                acc += B[k][p] * (Hm[k][0] * B[0][q] + Hm[k][1] * B[1][q] + Hm[k][2] * B[2][q]);
            am[p][q] = acc;
        }
    }
    d[0] = d[1] = d[2] = R(0);
    if (dim == 1) {
        if (fabs(am[0][0]) > eps_det * fabs(am[0][0])) {
            const R q0 = rhs[0] / am[0][0];
#pragma unroll
            for (int c = 0; c < 3; ++c) d[c] = B[c][0] * q0;
        }
    } else {
        const R det = am[0][0] * am[1][1] - am[0][1] * am[1][0];
        const R tr = R(0.5) * (am[0][0] + am[1][1]);
        if (fabs(det) > eps_det * tr * tr) {
            const R q0 = (am[1][1] * rhs[0] - am[0][1] * rhs[1]) / det;
            const R q1 = (am[0][0] * rhs[1] - am[1][0] * rhs[0]) / det;
#pragma unroll
            for (int c = 0; c < 3; ++c) d[c] = B[c][0] * q0 + B[c][1] * q1;
        }
    }
}

// rest edges of an entry in the fp32 displacement state (kind table, or from the rows of an
// explicit entry); false = absolute positions
template <typename R>
__device__ __forceinline__ bool rest_edges_of(const K1Args<R>& a, int kind, const R* w, float4* ex)
{
    if constexpr (sizeof(R) == 4) {
        if (a.kedge && kind >= 0) {
            const float4* p = a.kedge + 3LL * kind;
            ex[0] = __ldg(p);
            ex[1] = __ldg(p + 1);
            ex[2] = __ldg(p + 2);
            return true;
        }
        if (a.disp && kind < 0) {
            rest_edges_from_rows(reinterpret_cast<const float*>(w), ex);
            return true;
        }
    }
    (void)a; (void)kind; (void)w; (void)ex;
    return false;
}

template <typename R, int W>
__device__ R local_energy(const K1Args<R>& a, long long beg, long long end, int lane, unsigned gmask,
                          const R* p, const typename Vec4<R>::T& y4, int v)
{
    typedef typename Vec4<R>::T R4;
    R e = R(0);
    for (long long k = beg + lane; k < end; k += W) {
        Entry<R> en;
        R mu, lam, gamma;
        int ek_kind = -1;
        if (a.kinds) {
            const EntryK ek = EntryK::load(reinterpret_cast<const int4*>(a.ent), k);
            ek_kind = ek.kind;
            R r[KindRec<R>::NR];
            load_kind<R, KindRec<R>::Q>(a.kinds, ek.kind, r);
#pragma unroll
            for (int j = 0; j < 3; ++j) en.n[j] = ek.n[j];
#pragma unroll
            for (int j = 0; j < 9; ++j) en.w[j] = r[12 + j];
            en.V = r[21];
            mu = r[22]; lam = r[23]; gamma = r[11];
        } else {
            en = Entry<R>::load(a.ent, a.E, k);
            const Material<R> m = a.mat[en.mat];
            mu = m.mu; lam = m.lam; gamma = m.gamma;
        }
        const R4 q0 = a.pos[en.n[0]], q1 = a.pos[en.n[1]], q2 = a.pos[en.n[2]];
        float4 ex[3];
        const bool has = rest_edges_of<R>(a, ek_kind, en.w, ex);
        R e0[3], e1[3], e2[3];
        edge3<R>(q0, p, ex[0], has, e0);
        edge3<R>(q1, p, ex[1], has, e1);
        edge3<R>(q2, p, ex[2], has, e2);
        R F[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                F[r * 3 + c] = e0[r] * en.w[c] + e1[r] * en.w[3 + c] + e2[r] * en.w[6 + c];
        R ic = R(0);
#pragma unroll
        for (int q = 0; q < 9; ++q) ic += F[q] * F[q];
        const R J = F[0] * (F[4] * F[8] - F[7] * F[5]) + F[3] * (F[7] * F[2] - F[1] * F[8]) +
                    F[6] * (F[1] * F[5] - F[4] * F[2]);
        const R psi = (R(0.5) * mu) * (ic - R(3)) + (R(0.5) * lam) * (J - gamma) * (J - gamma);
        e += en.V * psi;
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) e += __shfl_xor_sync(gmask, e, o, W);
    if (a.soff || a.coff || a.box) e += extras_energy<R>(a, v, p);
    R ein = R(0);
    const R d0 = p[0] - y4.x, d1 = p[1] - y4.y, d2 = p[2] - y4.z;
    ein = ein + ((R(0.5) * y4.w) * d0) * d0;
    ein = ein + ((R(0.5) * y4.w) * d1) * d1;
    ein = ein + ((R(0.5) * y4.w) * d2) * d2;
    return ein + e;
}

// explicit layout: U entries per lane per iteration; all their loads (entry planes, then the
// 3U neighbour gathers) are issued before any math, for memory-level parallelism.  The
// per-entry constants are derived from the rows on the fly (ec_terms).
template <typename R, int W, int U, bool UM>
__device__ __forceinline__ void k1_accumulate_explicit(const K1Args<R>& a, long long beg, long long end,
                                                       int lane, const R* xi, const R* dx,
                                                       const Material<R>& mv, R* f, R* H)
{
    typedef typename Vec4<R>::T R4;
    R sv = R(0);
    for (long long k0 = beg + lane; k0 < end; k0 += (long long)W * U) {
        Entry<R> e[U];
        R4 p[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) e[u] = Entry<R>::load(a.ent, a.E, k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) {
                p[u][0] = a.pos[e[u].n[0]];
                p[u][1] = a.pos[e[u].n[1]];
                p[u][2] = a.pos[e[u].n[2]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) {
                float4 ex[3];
                const bool has = rest_edges_of<R>(a, -1, e[u].w, ex);
                R e0[3], e1[3], e2[3];
                edge3<R>(p[u][0], xi, ex[0], has, e0);
                edge3<R>(p[u][1], xi, ex[1], has, e1);
                edge3<R>(p[u][2], xi, ex[2], has, e2);
                const Material<R> m = UM ? mv : a.mat[e[u].mat];
                R t[9];
                ec_terms<R>(e[u].w, e[u].V, m.mu, m.lam, m.gamma, t);
                tet_contrib_ec<R, !UM>(e0, e1, e2, t, m.dsc, m.opd, dx, f, H, sv);
            }
        }
    }
}

// compact layout: one 16-byte entry per (vertex, tet); the per-kind constants come from the
// kind table (L1-resident).  UM: one material per vertex, damping hoisted -- its dsc / opd
// are returned from the records.  SENT: the CTA's entries were staged in shared memory by a
// bulk copy (k1_color_pass_bulk), entry k at sent[k - ebase].
template <typename R, int W, int U, bool UM, bool SENT>
__device__ __forceinline__ void k1_accumulate_compact(const K1Args<R>& a, long long beg, long long end,
                                                      int lane, const R* xi, const R* dx, R* f, R* H,
                                                      R& dsc, R& opd, const int4* sent, long long ebase)
{
    typedef typename Vec4<R>::T R4;
    const int4* __restrict__ ent = reinterpret_cast<const int4*>(a.ent);
    R sv = R(0);
    for (long long k0 = beg + lane; k0 < end; k0 += (long long)W * U) {
        EntryK e[U];
        R4 p[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) {
                if constexpr (SENT) {
                    const int4 v = sent[k - ebase];
                    e[u].n[0] = v.x; e[u].n[1] = v.y; e[u].n[2] = v.z; e[u].kind = v.w;
                } else {
                    e[u] = EntryK::load(ent, k);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) {
                p[u][0] = a.pos[e[u].n[0]];
                p[u][1] = a.pos[e[u].n[1]];
                p[u][2] = a.pos[e[u].n[2]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = k0 + (long long)u * W;
            if (u == 0 || k < end) {
                R r[KindRec<R>::HOT];
                load_kind<R, KindRec<R>::QH>(a.kinds, e[u].kind, r);
                float4 ex[3];
                const bool has = rest_edges_of<R>(a, e[u].kind, r, ex);
                R e0[3], e1[3], e2[3];
                edge3<R>(p[u][0], xi, ex[0], has, e0);
                edge3<R>(p[u][1], xi, ex[1], has, e1);
                edge3<R>(p[u][2], xi, ex[2], has, e2);
                tet_contrib_ec<R, !UM>(e0, e1, e2, r, r[9], r[10], dx, f, H, sv);
                if (UM) {
                    dsc = r[9];
                    opd = r[10];
                }
            }
        }
    }
}

template <typename R, int W, int U, bool UM, bool LS = false, bool KC = false, bool SENT = false>
__device__ __forceinline__ void k1_vertex_impl(const K1Args<R>& a, int g, int lane,
                                               const int4* sent = nullptr, long long ebase = 0,
                                               unsigned bar = 0)
{
    typedef typename Vec4<R>::T R4;
    const unsigned gmask =
        (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
    const int v = a.group ? a.group[g] : a.vbeg + g;
    const R4 xi4 = a.pos[v];
    if (v >= a.nsolve) {  // fixed / ghost: keep x (_native.pyx:424-426)
        if (lane == 0 && a.out) a.out[g] = xi4;
        return;
    }
    const R xi[3] = {xi4.x, xi4.y, xi4.z};
    const R4 xt4 = a.xt[v];
    const R dx[3] = {xi[0] - xt4.x, xi[1] - xt4.y, xi[2] - xt4.z};
    R f[3] = {R(0), R(0), R(0)};
    R H[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
    const long long beg = a.off[v], end = a.off[v + 1];
    const R4 y4 = a.y[v];  // inertia target, w = m / h^2 (issued early: used after the sweep)
    if constexpr (SENT) mbar_wait_parity(bar, 0);  // the CTA's entries have landed in smem
    Material<R> mv;
    if constexpr (KC) {
        mv.dsc = R(0);
        mv.opd = R(1);
        k1_accumulate_compact<R, W, U, UM, SENT>(a, beg, end, lane, xi, dx, f, H, mv.dsc, mv.opd, sent, ebase);
        if (UM) {  // lane 0 holds the vertex's first entry: its material is the vertex's
            mv.dsc = __shfl_sync(gmask, mv.dsc, 0, W);
            mv.opd = __shfl_sync(gmask, mv.opd, 0, W);
        }
    } else {
        if (UM) mv = a.mat[a.vmat[v]];
        k1_accumulate_explicit<R, W, U, UM>(a, beg, end, lane, xi, dx, mv, f, H);
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int q = 0; q < 3; ++q) f[q] += __shfl_xor_sync(gmask, f[q], o, W);
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] += __shfl_xor_sync(gmask, H[q], o, W);
    }
    if (UM) {  // sum over the vertex's entries of V mu |w|^2, precomputed in entry order
        const R s = a.vsv[v];
        H[0] = H[0] + s;
        H[3] = H[3] + s;
        H[5] = H[5] + s;
    }
    if (!LS && lane != 0) return;
    vertex_terms<R>(f, H, dx, xi, y4.x, y4.y, y4.z, y4.w, UM && end > beg, mv.dsc, mv.opd);
    R d[3];
    if (a.soff || a.coff || a.box) {
        extras_terms<R>(a, v, xi, dx, f, H);
        const int si = a.sub_idx ? a.sub_idx[v] : -1;
        if (si >= 0 && a.mode == 0) subspace_solve<R>(a.sub + 3 * si, f, H, a.eps_det, d);
        else block_solve<R>(f, H, a.eps_det, a.mode, d);
    } else {
        block_solve<R>(f, H, a.eps_det, a.mode, d);
    }
    R4 nx = xi4;
    if (LS && a.mode == 0) {
        // 17-trial backtracking on G_i (_native.pyx:481-492); every lane of the group runs
        // the same trials on the same reduced energies
        const R e0 = local_energy<R, W>(a, beg, end, lane, gmask, xi, y4, v);
        R alpha = R(1);
        for (int trial = 0; trial < 17; ++trial) {
            const R cand[3] = {xi[0] + alpha * d[0], xi[1] + alpha * d[1], xi[2] + alpha * d[2]};
            if (local_energy<R, W>(a, beg, end, lane, gmask, cand, y4, v) <= e0) {
                nx.x = cand[0];
                nx.y = cand[1];
                nx.z = cand[2];
                break;
            }
            alpha *= R(0.5);
        }
        if (lane != 0) return;
    } else {
        nx.x = xi[0] + d[0];
        nx.y = xi[1] + d[1];
        nx.z = xi[2] + d[2];
    }
    if (a.out) {
        a.out[g] = nx;
    } else {
        a.pos[v] = nx;
        if (a.peer_pos[0] || a.peer_pos[1]) {
            const int j = v - a.vbeg;
            if (j < a.nb[0]) {
                a.peer_pos[0][a.peer_off[0] + j] = nx;  // NVLink store into the left ghost
            } else if (j < a.nb[0] + a.nb[1]) {
                a.peer_pos[1][a.peer_off[1] + (j - a.nb[0])] = nx;
            }
        }
    }
    if (a.flag && !finite3(nx.x, nx.y, nx.z))
        atomicMin(a.flag, StepFlag::key((unsigned)*a.stepctr, (unsigned)a.iter, (unsigned)a.perm[v]));
}

template <typename R, int W, int U>
__device__ __forceinline__ void k1_vertex(const K1Args<R>& a, int g, int lane)
{
    if (a.kinds) {
        if (a.vmat) k1_vertex_impl<R, W, U, true, false, true>(a, g, lane);
        else k1_vertex_impl<R, W, U, false, false, true>(a, g, lane);
    } else {
        if (a.vmat) k1_vertex_impl<R, W, U, true>(a, g, lane);
        else k1_vertex_impl<R, W, U, false>(a, g, lane);
    }
}

// K1 with the local line search (protocol path, line_search=True)
template <typename R>
__global__ void __launch_bounds__(256) k1_color_pass_ls(const K1Args<R> a)
{
    const int g = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) / 4);
    if (g >= a.count) return;
    if (a.kinds) k1_vertex_impl<R, 4, 1, false, true, true>(a, g, threadIdx.x & 3);
    else k1_vertex_impl<R, 4, 1, false, true>(a, g, threadIdx.x & 3);
}

// One group of W lanes per vertex; lane j handles entries j, j+W, ... of its vertex and the
// group reduces f (3) and H (6) with a fixed xor-butterfly (bitwise deterministic).
template <typename R, int W, int U, int MINB, bool PF, bool UM, bool KC = false>
__global__ void __launch_bounds__(256, MINB) k1_color_pass(const K1Args<R> a)
{
    typedef typename Vec4<R>::T R4;
    const int g = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) / W);
    const int lane = threadIdx.x & (W - 1);
    if (PF && threadIdx.x == 0 && !a.group) {
        // A CTA's entries are one contiguous range per plane.  The TMA unit streams into L2
        // (cp.async.bulk.prefetch.L2) the range of the CTA one residency wave ahead
        // (pf_dist CTAs later; the first wave also fetches its own), so the per-lane loads
        // of later waves hit L2 and DRAM sees a deep queue without registers or smem.
        const int per = (int)(blockDim.x / W);
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const long long b = w == 0 ? (long long)blockIdx.x + a.pf_dist : (long long)blockIdx.x;
            if (w == 1 && blockIdx.x >= (unsigned)a.pf_dist) break;
            const long long g0 = b * per;
            const long long g1 = min((long long)a.count, g0 + per);
            if (g0 >= g1) continue;
            const long long e0 = a.off[a.vbeg + g0], e1 = a.off[a.vbeg + g1];
            const unsigned bytes = (unsigned)((e1 - e0) * 16);
            if (bytes)
#pragma unroll
                for (int pl = 0; pl < (KC ? 1 : EntryPlanes<R>::P); ++pl) {
                    const void* src = reinterpret_cast<const char*>(a.ent) + 16 * (pl * a.E + e0);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes)
                                 : "memory");
                }
        }
    }
    pdl_wait();  // entries are step constants (prefetched above); positions are not
    pdl_launch_dependents();
    if (g < a.count) k1_vertex_impl<R, W, U, UM, false, KC>(a, g, lane);
}

// ---------------------------------------------------------------------------------------
// K1, compact layout, range mode, entries staged by the bulk-copy engine: a CTA's vertices
// are consecutive, so their entries are one contiguous range [e0, e1) of 16-byte records.
// One thread arms an mbarrier and issues a single cp.async.bulk (TMA, SASS UBLKCP) of the
// range into shared memory; meanwhile every thread loads its vertex's x / x_t / y / CSR
// offsets; then the entry reads are LDS and the only long-latency loads left in the sweep
// are the neighbour gathers.  Dynamic smem = VPB x max degree x 16 B (host-checked).

template <typename R, int W, int U, int MINB, bool UM>
__global__ void __launch_bounds__(256, MINB) k1_color_pass_bulk(const K1Args<R> a)
{
    extern __shared__ __align__(16) int4 sent[];
    __shared__ __align__(8) unsigned long long mbar;
    constexpr int VPB = 256 / W;
    const long long g0 = (long long)blockIdx.x * VPB;
    const long long g1 = min((long long)a.count, g0 + VPB);
    const long long e0 = a.off[a.vbeg + g0];
    const unsigned bar = smem_u32(&mbar);
    if (threadIdx.x == 0) {
        const long long e1 = a.off[a.vbeg + g1];
        const unsigned bytes = (unsigned)((e1 - e0) * 16);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        if (bytes)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sent)),
                "l"(reinterpret_cast<const int4*>(a.ent) + e0), "r"(bytes), "r"(bar)
                : "memory");
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    pdl_wait();       // the entry copy above reads step constants only
    pdl_launch_dependents();
    const int g = (int)(g0 + threadIdx.x / W);
    const int lane = threadIdx.x & (W - 1);
    if (g < a.count) k1_vertex_impl<R, W, U, UM, false, true, true>(a, g, lane, sent, e0, bar);
}

// ---------------------------------------------------------------------------------------
// Incremental potential G(x) = 1/(2h^2)|x - y|_M^2 + E(x) (_assembly.py:29-82, no contacts):
// the metrics path of harness.run_simulation (harness.py:664-678) on the device.  Each tet is
// counted once, from the entry of its smallest solved colour-major vertex; each spring from
// its smaller solved end.  Per-block sums in double, summed in order on the host.
template <typename R, int W>
__global__ void __launch_bounds__(256) k_energy_elastic(const K1Args<R> a, int nsolve, double* partial)
{
    typedef typename Vec4<R>::T R4;
    __shared__ double red[256];
    const int g = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) / W);
    const int lane = threadIdx.x & (W - 1);
    double e = 0.0;
    if (g < nsolve) {
        const int v = g;
        const R4 xi4 = a.pos[v];
        for (long long k = a.off[v] + lane; k < a.off[v + 1]; k += W) {
            int n[3], kind = -1;
            R w[9], V, mu, lam, gamma;
            if (a.kinds) {
                const EntryK ek = EntryK::load(reinterpret_cast<const int4*>(a.ent), k);
                kind = ek.kind;
                R r[KindRec<R>::NR];
                load_kind<R, KindRec<R>::Q>(a.kinds, ek.kind, r);
                for (int j = 0; j < 3; ++j) n[j] = ek.n[j];
                for (int j = 0; j < 9; ++j) w[j] = r[12 + j];
                V = r[21]; mu = r[22]; lam = r[23]; gamma = r[11];
            } else {
                const Entry<R> en = Entry<R>::load(a.ent, a.E, k);
                for (int j = 0; j < 3; ++j) n[j] = en.n[j];
                for (int j = 0; j < 9; ++j) w[j] = en.w[j];
                V = en.V;
                const Material<R> m = a.mat[en.mat];
                mu = m.mu; lam = m.lam; gamma = m.gamma;
            }
            bool own = true;
            for (int j = 0; j < 3; ++j) own = own && (n[j] > v || n[j] >= nsolve);
            if (!own) continue;
            R ed[3][3];
            float4 ex[3];
            const bool has = rest_edges_of<R>(a, kind, w, ex);
            const R xi[3] = {xi4.x, xi4.y, xi4.z};
            for (int j = 0; j < 3; ++j) edge3<R>(a.pos[n[j]], xi, ex[j], has, ed[j]);
            R F[9];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    F[r * 3 + c] = ed[0][r] * w[c] + ed[1][r] * w[3 + c] + ed[2][r] * w[6 + c];
            R ic = R(0);
            for (int q = 0; q < 9; ++q) ic += F[q] * F[q];
            const R J = F[0] * (F[4] * F[8] - F[7] * F[5]) + F[3] * (F[7] * F[2] - F[1] * F[8]) +
                        F[6] * (F[1] * F[5] - F[4] * F[2]);
            e += (double)V * (0.5 * (double)mu * ((double)ic - 3.0) +
                              0.5 * (double)lam * ((double)J - (double)gamma) * ((double)J - (double)gamma));
        }
        if (lane == 0 && a.soff) {
            for (long long k = a.soff[v]; k < a.soff[v + 1]; ++k) {
                const int o = a.sp_oth[k];
                if (o < v && o < nsolve) continue;  // counted from the other end
                const R4 q = a.pos[o], sp = a.sp_par[k];
                const double d0 = (double)xi4.x - q.x, d1 = (double)xi4.y - q.y, d2 = (double)xi4.z - q.z;
                const double t = sqrt(d0 * d0 + d1 * d1 + d2 * d2) - (double)sp.x;
                e += 0.5 * (double)sp.y * t * t;
            }
        }
    }
    red[threadIdx.x] = e;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// inertia of every vertex and the world-box penalty
template <typename R>
__global__ void __launch_bounds__(256) k_energy_vertex(const K1Args<R> a, const R* __restrict__ mass, int n,
                                                       double inv_h2, double* partial)
{
    typedef typename Vec4<R>::T R4;
    __shared__ double red[256];
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (v < n) {
        const R4 x = a.pos[v], y = a.y[v];
        const double d0 = (double)x.x - y.x, d1 = (double)x.y - y.y, d2 = (double)x.z - y.z;
        e = 0.5 * inv_h2 * (double)mass[v] * (d0 * d0 + d1 * d1 + d2 * d2);
        if (a.box) {
            const R4 lo = a.box[2 * v], hi = a.box[2 * v + 1];
            if (lo.w > R(0)) {
                const double xv[3] = {x.x, x.y, x.z}, l[3] = {lo.x, lo.y, lo.z}, u[3] = {hi.x, hi.y, hi.z};
                for (int c = 0; c < 3; ++c) {
                    const double b = fmax(l[c] - xv[c], 0.0), t = fmax(xv[c] - u[c], 0.0);
                    e += 0.5 * (double)lo.w * (b * b + t * t);
                }
            }
        }
    }
    red[threadIdx.x] = e;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

template <typename R>
__global__ void k_scatter_group(const typename Vec4<R>::T* __restrict__ out, const int* __restrict__ group,
                                int ng, typename Vec4<R>::T* pos)
{
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < ng) pos[group[g]] = out[g];
}

// ---------------------------------------------------------------------------------------
// K2: y = x_t + h v_t + h^2 a (solver.py:120-122), warm start (solver.py:125-164), fixed
// clamp, y.w = m / h^2, history seed.
template <typename R> struct StepArgs {
    typedef typename Vec4<R>::T R4;
    int n;          // all vertices
    int nsolve;     // free (solved) vertices; [nsolve, nfree_all) are ghosts
    int nfree_all;  // vertices >= nfree_all are fixed
    R4 *pos, *xt, *vt, *vprev, *y, *ha, *hb;
    const R* mass;
    double h, hh;   // h and h*h (host-computed)
    double a[3];    // a_ext
    double an[3];   // a_ext / |a_ext|
    double anorm;   // |a_ext|
    int init_mode;  // 0 prev_pos, 1 inertia, 2 inertia_accel, 3 adaptive
    int hist;       // Chebyshev history needed
    unsigned long long* flag;
    const int* perm;
    int* stepctr;
    const int* sub_idx;  // SubspaceConstraint projection of the warm start (nullptr = none)
    const R4* sub;
};

template <typename R>
__device__ __forceinline__ void k2_vertex(const StepArgs<R>& s, int i)
{
    typedef typename Vec4<R>::T R4;
    const R4 xt = s.xt[i], vt = s.vt[i];
    const R h = (R)s.h, hh = (R)s.hh;
    const R ax = (R)s.a[0], ay = (R)s.a[1], az = (R)s.a[2];
    // every operation rounded separately, in the reference's NumPy order (solver.py:120-164):
    // no FMA contraction, so K2 gives the same bits wherever it is inlined (k2_step_init, the
    // persistent and resident step kernels)
    R4 y;
    const R xh[3] = {add_rn(xt.x, mul_rn(h, vt.x)), add_rn(xt.y, mul_rn(h, vt.y)), add_rn(xt.z, mul_rn(h, vt.z))};
    y.x = add_rn(xh[0], mul_rn(hh, ax));
    y.y = add_rn(xh[1], mul_rn(hh, ay));
    y.z = add_rn(xh[2], mul_rn(hh, az));
    y.w = s.mass[i] / hh;
    R4 x = xt;
    x.w = R(0);
    if (i < s.nfree_all) {
        if (s.init_mode == 1 || (s.init_mode == 3 && s.anorm == 0.0)) {
            x.x = xh[0];
            x.y = xh[1];
            x.z = xh[2];
        } else if (s.init_mode == 2) {
            x.x = y.x; x.y = y.y; x.z = y.z;
        } else if (s.init_mode == 3) {
            const R4 vp = s.vprev[i];
            R atx = (vt.x - vp.x) / h, aty = (vt.y - vp.y) / h, atz = (vt.z - vp.z) / h;
            R comp = add_rn(add_rn(mul_rn(atx, (R)s.an[0]), mul_rn(aty, (R)s.an[1])), mul_rn(atz, (R)s.an[2]));
            R at = comp / (R)s.anorm;
            at = at < R(0) ? R(0) : (at > R(1) ? R(1) : at);
            R sc = mul_rn(hh, at);
            x.x = add_rn(xh[0], mul_rn(sc, ax));
            x.y = add_rn(xh[1], mul_rn(sc, ay));
            x.z = add_rn(xh[2], mul_rn(sc, az));
        }
    } else if (s.flag && !finite3(x.x, x.y, x.z)) {  // fixed vertices never pass through K1
        atomicMin(s.flag, StepFlag::key((unsigned)*s.stepctr, 1u, (unsigned)s.perm[i]));
    }
    if (s.sub_idx && i < s.nsolve && s.sub_idx[i] >= 0) {  // solver.py:158-162
        const R4* b = s.sub + 3 * s.sub_idx[i];
        const R4 s0 = b[0], s1 = b[1], s2 = b[2];
        const R B[3][2] = {{s0.x, s0.y}, {s0.z, s0.w}, {s1.x, s1.y}};
        const R an[3] = {s1.z, s1.w, s2.x};
        const R r[3] = {x.x - an[0], x.y - an[1], x.z - an[2]};
        R c[2] = {R(0), R(0)};
        const int dim = (int)s2.y;
        for (int q = 0; q < dim; ++q) c[q] = B[0][q] * r[0] + B[1][q] * r[1] + B[2][q] * r[2];
        x.x = an[0] + B[0][0] * c[0] + B[0][1] * c[1];
        x.y = an[1] + B[1][0] * c[0] + B[1][1] * c[1];
        x.z = an[2] + B[2][0] * c[0] + B[2][1] * c[1];
    }
    s.y[i] = y;
    s.pos[i] = x;
    if (s.hist) s.ha[i] = x;
}

template <typename R>
__global__ void k2_step_init(const StepArgs<R> s)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s.n) k2_vertex<R>(s, i);
}

// x <- omega (x - x_pp) + x_pp (solver.py:221-232); shared by K3 and the resident step kernel
template <typename R>
__device__ __forceinline__ typename Vec4<R>::T k3_blend(typename Vec4<R>::T x, typename Vec4<R>::T pp, double omega)
{
    const R w = (R)omega;  // omega (x - x_pp) + x_pp, rounded per operation (no contraction)
    x.x = add_rn(mul_rn(w, x.x - pp.x), pp.x);
    x.y = add_rn(mul_rn(w, x.y - pp.y), pp.y);
    x.z = add_rn(mul_rn(w, x.z - pp.z), pp.z);
    return x;
}

// v = (x - x_t) / h (solver.py:319-323); shared by K4 and the resident step kernel
template <typename R>
__device__ __forceinline__ typename Vec4<R>::T k4_velocity(typename Vec4<R>::T x, typename Vec4<R>::T x0, double h)
{
    const R hr = (R)h;
    typename Vec4<R>::T v;
    v.x = (x.x - x0.x) / hr;
    v.y = (x.y - x0.y) / hr;
    v.z = (x.z - x0.z) / hr;
    v.w = R(0);
    return v;
}

// K3: Chebyshev semi-iterative blend against the iterate two sweeps back, then copy the
// blended iterate into the history buffer that becomes x_prev1 (solver.py:221-232, 312-315),
// then the non-finite check of solver.py:282-288.
template <typename R>
__device__ __forceinline__ void k3_vertex(typename Vec4<R>::T* pos, typename Vec4<R>::T* hist,
                                          double omega, int blend, unsigned long long* flag,
                                          const int* perm, const int* stepctr, int iter, int i,
                                          const unsigned char* coll = nullptr)
{
    typedef typename Vec4<R>::T R4;
    R4 x = pos[i];
    if (blend && !(coll && coll[i])) {  // colliding vertices keep x (solver.py:229-230)
        x = k3_blend<R>(x, hist[i], omega);
        pos[i] = x;
    }
    hist[i] = x;
    if (flag && !finite3(x.x, x.y, x.z))
        atomicMin(flag, StepFlag::key((unsigned)*stepctr, (unsigned)iter, (unsigned)perm[i]));
}

template <typename R>
__global__ void k3_chebyshev(typename Vec4<R>::T* pos, typename Vec4<R>::T* hist, int n,
                             double omega, int blend, unsigned long long* flag,
                             const int* perm, const int* stepctr, int iter,
                             const unsigned char* coll = nullptr)
{
    pdl_wait();
    pdl_launch_dependents();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) k3_vertex<R>(pos, hist, omega, blend, flag, perm, stepctr, iter, i, coll);
}

// K4: velocity commit (solver.py:319-323); skipped when the step reported a non-finite state.
template <typename R>
__device__ __forceinline__ void k4_vertex(typename Vec4<R>::T* pos, typename Vec4<R>::T* xt,
                                          typename Vec4<R>::T* vt, typename Vec4<R>::T* vprev,
                                          double h, int i)
{
    typedef typename Vec4<R>::T R4;
    const R4 x = pos[i], x0 = xt[i], v0 = vt[i];
    const R4 v = k4_velocity<R>(x, x0, h);
    vprev[i] = v0;
    vt[i] = v;
    xt[i] = x;
}

template <typename R>
__global__ void k4_commit(typename Vec4<R>::T* pos, typename Vec4<R>::T* xt, typename Vec4<R>::T* vt,
                          typename Vec4<R>::T* vprev, int n, double h,
                          const unsigned long long* flag, int* stepctr)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) atomicAdd(stepctr, 1);
    if (i >= n || *flag != StepFlag::NONE) return;
    k4_vertex<R>(pos, xt, vt, vprev, h, i);
}

// ---------------------------------------------------------------------------------------
// Whole step in one persistent cooperative launch (small scenes: the per-colour passes of
// C1-C3 are a few microseconds of work, so graph-node launch latency would dominate).
// The same K1..K4 bodies run grid-stride, separated by grid-wide barriers.

#define VBD_PERSIST_MAX_COLORS 64

template <typename R> struct PersistArgs {
    K1Args<R> k1;
    StepArgs<R> s;
    int ncolors;
    int cbeg[VBD_PERSIST_MAX_COLORS];
    int ccnt[VBD_PERSIST_MAX_COLORS];
    int n_max;
    int chebyshev;          // rho != 0
    const double* omegas;   // [n_max + 1]
};

template <typename R, int W, int U>
__global__ void __launch_bounds__(256, 3) k_step_persistent(const PersistArgs<R> p)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    const int n = p.s.n;
    for (int i = tid; i < n; i += nth) k2_vertex<R>(p.s, i);
    grid.sync();
    const int lane = threadIdx.x & (W - 1);
    for (int it = 1; it <= p.n_max; ++it) {
        for (int c = 0; c < p.ncolors; ++c) {
            K1Args<R> a = p.k1;
            a.vbeg = p.cbeg[c];
            a.count = p.ccnt[c];
            a.iter = it;
            for (int g = tid / W; g < a.count; g += nth / W) k1_vertex<R, W, U>(a, g, lane);
            grid.sync();
        }
        if (p.chebyshev) {
            typename Vec4<R>::T* hist = (it % 2 == 1) ? p.s.hb : p.s.ha;
            const double w = p.omegas[it];
            const int blend = (it >= 2 && w != 1.0) ? 1 : 0;
            for (int i = tid; i < n; i += nth)
                k3_vertex<R>(p.s.pos, hist, w, blend, p.s.flag, p.s.perm, p.s.stepctr, it, i);
            grid.sync();
        }
    }
    if (*p.s.flag == StepFlag::NONE)
        for (int i = tid; i < n; i += nth) k4_vertex<R>(p.s.pos, p.s.xt, p.s.vt, p.s.vprev, p.s.h, i);
    if (tid == 0) atomicAdd(p.s.stepctr, 1);
}

// ---------------------------------------------------------------------------------------
// state transfer: original-order (N,3) float64 <-> colour-major R4

// rest: colour-major rest positions (fp32 displacement state: position-like vectors are
// stored as x - X); nullptr for velocities and absolute states
template <typename R>
__global__ void k_load_vec(const double* __restrict__ src, typename Vec4<R>::T* dst,
                           const int* __restrict__ perm, int n, const double4* __restrict__ rest = nullptr)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long o = perm[i];
    double x = src[3 * o], y = src[3 * o + 1], z = src[3 * o + 2];
    if (rest) {
        const double4 r = rest[i];
        x -= r.x;
        y -= r.y;
        z -= r.z;
    }
    typename Vec4<R>::T v;
    v.x = (R)x;
    v.y = (R)y;
    v.z = (R)z;
    v.w = R(0);
    dst[i] = v;
}

template <typename R>
__global__ void k_store_vec(const typename Vec4<R>::T* __restrict__ src, double* dst,
                            const int* __restrict__ inv, int n, const double4* __restrict__ rest = nullptr)
{
    int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int i = inv[o];
    typename Vec4<R>::T v = src[i];
    double x = (double)v.x, y = (double)v.y, z = (double)v.z;
    if (rest) {
        const double4 r = rest[i];
        x += r.x;
        y += r.y;
        z += r.z;
    }
    dst[3LL * o] = x;
    dst[3LL * o + 1] = y;
    dst[3LL * o + 2] = z;
}

template <typename R>
__global__ void k_set_targets(const int* __restrict__ ids, const double* __restrict__ xyz, int n,
                              typename Vec4<R>::T* xt, typename Vec4<R>::T* pos,
                              const double4* __restrict__ rest = nullptr)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double x = xyz[3 * k], y = xyz[3 * k + 1], z = xyz[3 * k + 2];
    if (rest) {
        const double4 r = rest[ids[k]];
        x -= r.x;
        y -= r.y;
        z -= r.z;
    }
    typename Vec4<R>::T v;
    v.x = (R)x;
    v.y = (R)y;
    v.z = (R)z;
    v.w = R(0);
    xt[ids[k]] = v;
    pos[ids[k]] = v;
}

// aux-buffer results of a group pass in double, absolute (+ rest in the displacement state)
template <typename R>
__global__ void k_group_abs(const typename Vec4<R>::T* __restrict__ out, const int* __restrict__ g,
                            const double4* __restrict__ rest, int ng, double* __restrict__ dst)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const typename Vec4<R>::T v = out[k];
    double x = (double)v.x, y = (double)v.y, z = (double)v.z;
    if (rest) {
        const double4 r = rest[g[k]];
        x += r.x;
        y += r.y;
        z += r.z;
    }
    dst[3LL * k] = x;
    dst[3LL * k + 1] = y;
    dst[3LL * k + 2] = z;
}

// colour-major rest positions (double4) from original-order (N, 3)
__global__ void k_rest_positions(const double* __restrict__ src, const int* __restrict__ perm, int n,
                                 double4* __restrict__ rest)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long o = perm[i];
    rest[i] = make_double4(src[3 * o], src[3 * o + 1], src[3 * o + 2], 0.0);
}

// fp32 displacement state -> absolute (contacts need absolute positions): x = fl32(X + u)
__global__ void k_disp_to_abs(float4* v, const double4* __restrict__ rest, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 u = v[i];
    const double4 r = rest[i];
    v[i] = make_float4((float)(r.x + (double)u.x), (float)(r.y + (double)u.y), (float)(r.z + (double)u.z), u.w);
}

template <typename R>
__global__ void k_fill_mih2(typename Vec4<R>::T* y, const R* mass, int n, double hh)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i].w = mass[i] / (R)hh;
}

// Global backtracking trial of baselines._global_line_search (baselines.py:139-149):
// x = checkpoint + alpha * (x_new - checkpoint), each operation rounded on its own as NumPy
// evaluates it (no contraction into an FMA).
__device__ __forceinline__ double ls_axpy(double c, double xn, double alpha)
{
    return __dadd_rn(c, __dmul_rn(alpha, __dsub_rn(xn, c)));
}
__device__ __forceinline__ float ls_axpy(float c, float xn, double alpha)
{
    return __fadd_rn(c, __fmul_rn((float)alpha, __fsub_rn(xn, c)));
}

template <typename R>
__global__ void k_ls_blend(typename Vec4<R>::T* pos, const typename Vec4<R>::T* ckpt,
                           const typename Vec4<R>::T* xn, double alpha, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    typename Vec4<R>::T x = xn[i];
    const typename Vec4<R>::T c = ckpt[i];
    x.x = ls_axpy(c.x, x.x, alpha);
    x.y = ls_axpy(c.y, x.y, alpha);
    x.z = ls_axpy(c.z, x.z, alpha);
    pos[i] = x;
}

// halo exchange for slab-decomposed scenes: gather/scatter the positions of a vertex list
// Neighbour phase barrier over peer memory (slab P2P halo).  flags[0] of a context is
// written by its left neighbour, flags[1] by its right one; values are monotonically
// increasing phase stamps base + phase, base = phases of all previous steps (identical on
// every rank because every rank runs the same phase sequence).
// The release of a phase.  The colour pass before it stored its slab-boundary vertices
// straight into the neighbours' ghost slots (plain st.global through the cudaIpc mapping, no
// per-store fence).  This kernel is stream-ordered after that grid has completed, so those
// stores happen-before this thread; the system-scope fence + st.release.sys below publishes
// all of them with one release per phase, and the neighbour's k_phase_wait (ld.acquire.sys)
// synchronises with it before its next phase reads a ghost.
__global__ void k_phase_signal(unsigned long long* left_slot, unsigned long long* right_slot,
                               const unsigned long long* epoch, unsigned long long pps, int phase)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long v = *epoch + (unsigned long long)phase;
    __threadfence_system();
    if (left_slot) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(left_slot), "l"(v) : "memory");
    if (right_slot) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(right_slot), "l"(v) : "memory");
}

__global__ void k_phase_wait(const unsigned long long* flags, int need_left, int need_right,
                             const unsigned long long* epoch, unsigned long long pps, int phase,
                             int* err)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // neighbours must have completed the previous phase (phase - 1)
    const unsigned long long target = *epoch + (unsigned long long)(phase - 1);
    for (int side = 0; side < 2; ++side) {
        if (!(side == 0 ? need_left : need_right)) continue;
        unsigned long long v = 0;
        long long spins = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + side) : "memory");
            if (v >= target) break;
            if (++spins > (1ll << 26)) {  // ~seconds: report instead of hanging the GPU
                atomicExch(err, 1);
                break;
            }
            __nanosleep(64);
        }
    }
    __threadfence_system();
}

__global__ void k_epoch_advance(unsigned long long* epoch, unsigned long long pps)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) *epoch += pps;
}

template <typename R>
__global__ void k_halo_pack(const typename Vec4<R>::T* __restrict__ pos, const int* __restrict__ ids,
                            int n, typename Vec4<R>::T* __restrict__ buf)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] = pos[ids[i]];
}

template <typename R>
__global__ void k_halo_unpack(typename Vec4<R>::T* pos, const int* __restrict__ ids, int n,
                              const typename Vec4<R>::T* __restrict__ buf)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pos[ids[i]] = buf[i];
}


// Per-vertex sum over its entries (CSR order) of V mu |w|^2 -- the constant diagonal Hessian
// term of every entry (ec_terms t[8]) -- for one material per vertex (UM).  Summed here once in
// entry order and added after the lane reduction by every K1 variant, so all of them stay
// bitwise equal; the sweep no longer loads or adds it per entry.
template <typename R>
__global__ void k_vertex_sv(const K1Args<R> a, int nsolve, R* __restrict__ out)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nsolve) return;
    R s = R(0);
    const long long beg = a.off[v], end = a.off[v + 1];
    if (a.kinds) {
        for (long long k = beg; k < end; ++k) {
            const int kind = reinterpret_cast<const int4*>(a.ent)[k].w;
            R r[KindRec<R>::HOT];
            load_kind<R, KindRec<R>::QH>(a.kinds, kind, r);
            s = s + r[8];
        }
    } else {
        const Material<R> m = a.mat[a.vmat[v]];
        for (long long k = beg; k < end; ++k) {
            const Entry<R> e = Entry<R>::load(a.ent, a.E, k);
            R t[9];
            ec_terms<R>(e.w, e.V, m.mu, m.lam, m.gamma, t);
            s = s + t[8];
        }
    }
    out[v] = s;
}
