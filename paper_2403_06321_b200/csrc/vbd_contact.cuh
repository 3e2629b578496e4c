// vbd_contact.cuh -- contact detection on the device (contact.py restated):
//   * broad phase (contact.py:277-343): padded, swept AABBs of surface vertices, triangles
//     and edges hashed into a uniform grid (cell = 1.5 x the median rest surface edge);
//     candidates are joined per cell, deduplicated as packed ascending codes (the
//     reference's sorted (vertex, triangle) / (edge, edge) order) and filtered exactly:
//     no shared vertex, AABBs overlap, at least one non-fixed vertex.  The filtered pair set
//     is the set of overlapping padded boxes, independent of the hash, as in the reference.
//   * DCD vertex-triangle narrow phase (contact.py:346-439) at x_t;
//   * CCD vertex-triangle / edge-edge (contact.py:442-737): coplanarity cubic on linear
//     trajectories x_t -> x, real roots in [0,1] (max-normalised coefficients, degree drop at
//     1e-14, |imag| < 1e-8), 20-step bracketed bisection, containment, side orientation.
//   * contact records in the K1 format (colour-major ids, {gamma}{n, k_c}{tangent}{refresh})
//     and the sticky colliding flags of ContactSet.mark_flags (contact.py:111-118).
// All detection arithmetic is fp64, in the reference's operation order.
#pragma once
#include "vbd_common.cuh"

#define VBD_CELL_BITS 21
#define VBD_CELL_MASK ((1ll << VBD_CELL_BITS) - 1)

struct D3 {
    double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return d3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 cross(D3 a, D3 b)
{
    return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double norm(D3 a) { return sqrt(dot(a, a)); }

template <typename R> __device__ __forceinline__ D3 ld3(const typename Vec4<R>::T* p, int i)
{
    const typename Vec4<R>::T v = p[i];
    return d3((double)v.x, (double)v.y, (double)v.z);
}

// the geometry a detection pass reads: surface primitives in original order (ids mapped to
// the colour-major position arrays) and the start / end positions
template <typename R> struct CollArgs {
    typedef typename Vec4<R>::T R4;
    const int* sv;      // surface vertices (colour-major), ascending original id
    const int4* tri;    // surface triangles (colour-major), original order
    const int2* edge;   // surface edges (colour-major), original order
    int nsv, ntri, nedge;
    const unsigned char* active;  // per colour-major vertex: not fixed
    const R4* xs;       // start positions
    const R4* xe;       // end positions
    double cell, pad;
};

// Graph mode (one CUDA graph per contact step, vbd_capi.cu step_contacts_graph): every array
// runs at a fixed capacity and its unused tail holds a SENTINEL (key / code ~0, record idx.x
// < 0) instead of a host-read count; the kernels below skip sentinels, so the same kernels
// serve the host-synchronised path (no sentinels) and the captured one.
#define VBD_SENT 0xffffffffffffffffull

// ---------------------------------------------------------------------------------------
// broad phase

__device__ __forceinline__ long long cell_of(double v, double cell) { return (long long)floor(v / cell); }

__device__ __forceinline__ unsigned long long cell_key(long long ix, long long iy, long long iz)
{
    return (unsigned long long)(((ix & VBD_CELL_MASK) << (2 * VBD_CELL_BITS)) | ((iy & VBD_CELL_MASK) << VBD_CELL_BITS) |
                                (iz & VBD_CELL_MASK));
}

// AABB of primitive p of `what` (0 vertex, 1 triangle, 2 edge), padded
template <typename R>
__device__ void prim_box(const CollArgs<R>& c, int what, int p, double* lo, double* hi)
{
    int ids[3];
    int n = 1;
    if (what == 0) {
        ids[0] = c.sv[p];
    } else if (what == 1) {
        const int4 t = c.tri[p];
        ids[0] = t.x; ids[1] = t.y; ids[2] = t.z;
        n = 3;
    } else {
        const int2 e = c.edge[p];
        ids[0] = e.x; ids[1] = e.y;
        n = 2;
    }
    double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
    double ls[3] = {INFINITY, INFINITY, INFINITY}, hs[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < n; ++k) {
        const D3 a = ld3<R>(c.xs, ids[k]), b = ld3<R>(c.xe, ids[k]);
        const double av[3] = {a.x, a.y, a.z}, bv[3] = {b.x, b.y, b.z};
        for (int q = 0; q < 3; ++q) {
            ls[q] = fmin(ls[q], av[q]);
            hs[q] = fmax(hs[q], av[q]);
            l[q] = fmin(l[q], bv[q]);
            h[q] = fmax(h[q], bv[q]);
        }
    }
    for (int q = 0; q < 3; ++q) {  // min(xs.min, xe.min) - pad, max(xs.max, xe.max) + pad
        lo[q] = fmin(ls[q], l[q]) - c.pad;
        hi[q] = fmax(hs[q], h[q]) + c.pad;
    }
}

template <typename R>
__global__ void k_cell_count(const CollArgs<R> c, int what, int n, long long* cnt)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double lo[3], hi[3];
    prim_box<R>(c, what, p, lo, hi);
    long long m = 1;
    for (int q = 0; q < 3; ++q) m *= cell_of(hi[q], c.cell) - cell_of(lo[q], c.cell) + 1;
    cnt[p] = m;
}

template <typename R>
__global__ void k_cell_emit(const CollArgs<R> c, int what, int n, const long long* __restrict__ off,
                            unsigned long long* __restrict__ key, int* __restrict__ own, long long cap = 0)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double lo[3], hi[3];
    prim_box<R>(c, what, p, lo, hi);
    long long l[3], h[3];
    for (int q = 0; q < 3; ++q) {
        l[q] = cell_of(lo[q], c.cell);
        h[q] = cell_of(hi[q], c.cell);
    }
    long long w = off[p];
    for (long long ix = l[0]; ix <= h[0]; ++ix)
        for (long long iy = l[1]; iy <= h[1]; ++iy)
            for (long long iz = l[2]; iz <= h[2]; ++iz, ++w) {
                if (cap && w >= cap) return;  // graph mode: overflow (flagged by k_sent_tail)
                key[w] = cell_key(ix, iy, iz);
                own[w] = p;
            }
}

// lower bound of k in the sorted keys
__device__ __forceinline__ long long lower_key(const unsigned long long* keys, long long n, unsigned long long k)
{
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// query cells against the sorted target cells: count (FILL = false) or write the packed codes
// q * width + t (vertex-triangle) / min * width + max (edge-edge, SELF: only q < t)
template <bool FILL, bool SELF>
__global__ void k_cell_join(const unsigned long long* __restrict__ qkey, const int* __restrict__ qown,
                            long long nq, const unsigned long long* __restrict__ tkey,
                            const int* __restrict__ town, long long nt, long long width,
                            long long* __restrict__ cnt, const long long* __restrict__ off,
                            unsigned long long* __restrict__ codes, long long cap = 0)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const unsigned long long k = qkey[i];
    if (k == VBD_SENT) {  // padding (graph mode)
        if (!FILL) cnt[i] = 0;
        return;
    }
    long long j = lower_key(tkey, nt, k);
    long long c = 0, w = FILL ? off[i] : 0;
    const long long q = qown[i];
    for (; j < nt && tkey[j] == k; ++j) {
        const long long t = town[j];
        if (SELF && !(q < t)) continue;
        if (FILL && (!cap || w < cap)) codes[w] = (unsigned long long)(q * width + t);
        if (FILL) ++w;
        ++c;
    }
    if (!FILL) cnt[i] = c;
}

// graph mode: the tail [total, cap) of a key array gets the sentinel (and own = -1); a total
// over the capacity raises the overflow flag (the step is redone on the host path)
__global__ void k_sent_tail(unsigned long long* __restrict__ key, int* __restrict__ own,
                            const long long* __restrict__ total, long long cap, int* __restrict__ overflow)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long t = *total;
    if (i == 0 && t > cap) atomicExch(overflow, 1);
    if (i >= cap || i < t) return;
    key[i] = VBD_SENT;
    if (own) own[i] = -1;
}

// ---------------------------------------------------------------------------------------
// narrow phases

// tangent_basis (contact.py:129-142): cross with the axis of the smallest |n| component
__device__ void tangent_basis(D3 n, D3& t1, D3& t2)
{
    const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
    int k = 0;
    if (an[1] < an[k]) k = 1;
    if (an[2] < an[k]) k = 2;
    const D3 ax = d3(k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0);
    t1 = cross(n, ax);
    const double l1 = norm(t1);
    t1 = d3(t1.x / l1, t1.y / l1, t1.z / l1);
    t2 = cross(n, t1);
    const double l2 = norm(t2);
    t2 = d3(t2.x / l2, t2.y / l2, t2.z / l2);
}

// closest point on triangle abc (contact.py:145-177, batch: contact.py:346-385)
__device__ void closest_point_tri(D3 p, D3 a, D3 b, D3 c, D3& q, double* bary)
{
    const D3 ab = b - a, ac = c - a, ap = p - a;
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) { q = a; bary[0] = 1.0; bary[1] = 0.0; bary[2] = 0.0; return; }
    const D3 bp = p - b;
    const double d3v = dot(ab, bp), d4 = dot(ac, bp);
    if (d3v >= 0.0 && d4 <= d3v) { q = b; bary[0] = 0.0; bary[1] = 1.0; bary[2] = 0.0; return; }
    const double vc = d1 * d4 - d3v * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3v <= 0.0) {
        const double v = d1 / (d1 - d3v);
        q = a + v * ab;
        bary[0] = 1.0 - v; bary[1] = v; bary[2] = 0.0;
        return;
    }
    const D3 cp = p - c;
    const double d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) { q = c; bary[0] = 0.0; bary[1] = 0.0; bary[2] = 1.0; return; }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = d2 / (d2 - d6);
        q = a + w * ac;
        bary[0] = 1.0 - w; bary[1] = 0.0; bary[2] = w;
        return;
    }
    const double va = d3v * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3v) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3v) / ((d4 - d3v) + (d5 - d6));
        q = b + w * (c - b);
        bary[0] = 0.0; bary[1] = 1.0 - w; bary[2] = w;
        return;
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    q = (a + v * ab) + w * ac;
    bary[0] = 1.0 - v - w; bary[1] = v; bary[2] = w;
}

// one contact in the K1 record format (colour-major ids) + its kind / key for dedupe
struct ContactRec {
    int4 idx;
    double g[4];
    double n[3];
    double t[6];  // tangent (3,2) row-major: t[a*2+k]
    double kc;
    int refresh;  // DCD vertex-triangle
    int ccd;
};

__device__ void make_rec(ContactRec& r, int4 idx, const double* gam, D3 n, double kc, int refresh, int ccd)
{
    r.idx = idx;
    for (int k = 0; k < 4; ++k) r.g[k] = gam[k];
    r.n[0] = n.x; r.n[1] = n.y; r.n[2] = n.z;
    D3 t1, t2;
    tangent_basis(n, t1, t2);
    r.t[0] = t1.x; r.t[1] = t2.x; r.t[2] = t1.y; r.t[3] = t2.y; r.t[4] = t1.z; r.t[5] = t2.z;
    r.kc = kc;
    r.refresh = refresh;
    r.ccd = ccd;
}

// DCD vertex-triangle (contact.py:388-439) on the filtered candidate `code` (k * ntri + t)
template <typename R>
__global__ void k_dcd_vt(const CollArgs<R> c, const unsigned long long* __restrict__ codes, long long n,
                         double radius, double kc, int has_max_depth, double max_depth,
                         ContactRec* __restrict__ out, int* __restrict__ acc)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (codes[i] == VBD_SENT) {  // padding (graph mode)
        acc[i] = 0;
        return;
    }
    const long long k = (long long)(codes[i] / (unsigned long long)c.ntri);
    const int t = (int)(codes[i] % (unsigned long long)c.ntri);
    acc[i] = 0;
    const int v = c.sv[k];
    const int4 tr = c.tri[t];
    double vl[3], vh[3], tl[3], th[3];
    prim_box<R>(c, 0, (int)k, vl, vh);
    prim_box<R>(c, 1, t, tl, th);
    bool keep = tr.x != v && tr.y != v && tr.z != v;
    for (int q = 0; q < 3; ++q) keep = keep && tl[q] <= vh[q] && vl[q] <= th[q];
    keep = keep && (c.active[v] || c.active[tr.x] || c.active[tr.y] || c.active[tr.z]);
    if (!keep) return;
    const D3 a = ld3<R>(c.xs, tr.x), b = ld3<R>(c.xs, tr.y), cc = ld3<R>(c.xs, tr.z), p = ld3<R>(c.xs, v);
    D3 nrm = cross(b - a, cc - a);
    const double nn = norm(nrm);
    const double scale = fmax(fmax(norm(b - a), norm(cc - a)), 1e-30);
    if (!(nn >= 1e-12 * scale * scale)) return;
    nrm = d3(nrm.x / nn, nrm.y / nn, nrm.z / nn);
    D3 q;
    double bary[3];
    closest_point_tri(p, a, b, cc, q, bary);
    const double dist = norm(p - q);
    const double sgn = dot(p - a, nrm);
    const bool behind = sgn < 0.0 && dist <= fabs(sgn) * (1.0 + 1e-9) + 1e-15;
    bool accept = dist <= radius || behind;
    if (has_max_depth) accept = accept && !(behind && -sgn > max_depth);
    if (!accept) return;
    const double gam[4] = {1.0, -bary[0], -bary[1], -bary[2]};
    make_rec(out[i], make_int4(v, tr.x, tr.y, tr.z), gam, nrm, kc, 1, 0);
    acc[i] = 1;
}

// real roots of c3 t^3 + c2 t^2 + c1 t + c0 in [0, 1] (contact.py:509-546): coefficients
// max-normalised, leading terms below 1e-14 drop the degree, roots with |imag| < 1e-8 count
// as real, kept within 1e-10 of [0,1] and clipped; ascending, nr <= 3
__device__ int roots_unit(double c0, double c1, double c2, double c3, double* out)
{
    double co[4] = {c3, c2, c1, c0};
    const double lead = fmax(fmax(fabs(co[0]), fabs(co[1])), fmax(fabs(co[2]), fabs(co[3])));
    if (!(lead > 0.0)) return 0;
    for (int k = 0; k < 4; ++k) co[k] /= lead;
    int nz = 0;
    while (nz < 4 && !(fabs(co[nz]) > 1e-14)) ++nz;
    double re[3], im[3];
    int nr = 0;
    if (nz == 0) {  // monic cubic t^3 + a t^2 + b t + c
        const double a = co[1] / co[0], b = co[2] / co[0], cc = co[3] / co[0];
        const double Q = (a * a - 3.0 * b) / 9.0, Rr = (2.0 * a * a * a - 9.0 * a * b + 27.0 * cc) / 54.0;
        const double Q3 = Q * Q * Q;
        if (Rr * Rr < Q3) {  // three real roots (trigonometric)
            const double th = acos(fmax(-1.0, fmin(1.0, Rr / sqrt(Q3))));
            const double sq = -2.0 * sqrt(Q);
            re[0] = sq * cos(th / 3.0) - a / 3.0;
            re[1] = sq * cos((th + 2.0 * M_PI) / 3.0) - a / 3.0;
            re[2] = sq * cos((th - 2.0 * M_PI) / 3.0) - a / 3.0;
            im[0] = im[1] = im[2] = 0.0;
        } else {  // one real root and a complex pair
            const double A = -copysign(cbrt(fabs(Rr) + sqrt(Rr * Rr - Q3)), Rr);
            const double B = A != 0.0 ? Q / A : 0.0;
            re[0] = (A + B) - a / 3.0;
            re[1] = re[2] = -0.5 * (A + B) - a / 3.0;
            im[0] = 0.0;
            im[1] = im[2] = 0.5 * sqrt(3.0) * fabs(A - B);
        }
        // Newton polish of the real candidates on the normalised cubic
        for (int k = 0; k < 3; ++k) {
            if (im[k] != 0.0 && fabs(im[k]) >= 1e-8) continue;
            double x = re[k];
            for (int it = 0; it < 3; ++it) {
                const double f = ((co[0] * x + co[1]) * x + co[2]) * x + co[3];
                const double df = (3.0 * co[0] * x + 2.0 * co[1]) * x + co[2];
                if (df == 0.0) break;
                const double xn = x - f / df;
                if (!(fabs(xn - x) < 1e-3)) break;
                x = xn;
            }
            re[k] = x;
        }
        nr = 3;
    } else if (nz == 1) {  // quadratic co1 t^2 + co2 t + co3
        const double a = co[1], b = co[2], cc = co[3];
        const double disc = b * b - 4.0 * a * cc;
        if (disc >= 0.0) {
            const double s = sqrt(disc);
            const double qq = -0.5 * (b + copysign(s, b));
            re[0] = qq / a;
            re[1] = qq != 0.0 ? cc / qq : -b / (2.0 * a);
            im[0] = im[1] = 0.0;
        } else {
            re[0] = re[1] = -b / (2.0 * a);
            im[0] = im[1] = sqrt(-disc) / (2.0 * fabs(a));
        }
        nr = 2;
    } else if (nz == 2) {
        re[0] = -co[3] / co[2];
        im[0] = 0.0;
        nr = 1;
    } else {
        return 0;
    }
    int m = 0;
    for (int k = 0; k < nr; ++k) {
        if (!(fabs(im[k]) < 1e-8)) continue;
        const double r = re[k];
        if (r > -1e-10 && r < 1.0 + 1e-10) out[m++] = fmin(fmax(r, 0.0), 1.0);
    }
    for (int i = 1; i < m; ++i)  // ascending
        for (int j = i; j > 0 && out[j] < out[j - 1]; --j) {
            const double tmp = out[j];
            out[j] = out[j - 1];
            out[j - 1] = tmp;
        }
    return m;
}

// coplanarity (u0 + t u1) x (v0 + t v1) . (w0 + t w1) (contact.py:500-506)
__device__ __forceinline__ double coplanar(D3 u0, D3 u1, D3 v0, D3 v1, D3 w0, D3 w1, double t)
{
    const D3 ut = u0 + t * u1, vt = v0 + t * v1, wt = w0 + t * w1;
    return dot(cross(ut, vt), wt);
}

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// _bisect_batch for one root (contact.py:549-571)
__device__ double bisect(D3 u0, D3 u1, D3 v0, D3 v1, D3 w0, D3 w1, double t)
{
    double lo = fmax(0.0, t - 1e-3), hi = fmin(1.0, t + 1e-3);
    const double flo = coplanar(u0, u1, v0, v1, w0, w1, lo), fhi = coplanar(u0, u1, v0, v1, w0, w1, hi);
    if (flo == 0.0) return lo;
    if (!(fhi != 0.0 && sgn(flo) != sgn(fhi))) return t;
    const double slo = sgn(flo);
    for (int it = 0; it < 20; ++it) {
        const double mid = 0.5 * (lo + hi);
        const double fm = coplanar(u0, u1, v0, v1, w0, w1, mid);
        if (fm == 0.0) return mid;
        if (sgn(fm) == slo) lo = mid;
        else hi = mid;
    }
    return 0.5 * (lo + hi);
}

__device__ __forceinline__ void cubic_coeffs(D3 u0, D3 u1, D3 v0, D3 v1, D3 w0, D3 w1, double* c)
{
    const D3 q0 = cross(u0, v0);
    const D3 q1 = cross(u0, v1) + cross(u1, v0);
    const D3 q2 = cross(u1, v1);
    c[0] = dot(q0, w0);
    c[1] = dot(q0, w1) + dot(q1, w0);
    c[2] = dot(q1, w1) + dot(q2, w0);
    c[3] = dot(q2, w1);
}

// CCD vertex-triangle (contact.py:574-651)
template <typename R>
__global__ void k_ccd_vt(const CollArgs<R> c, const unsigned long long* __restrict__ codes, long long n, double kc,
                         ContactRec* __restrict__ out, int* __restrict__ acc)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (codes[i] == VBD_SENT) {  // padding (graph mode)
        acc[i] = 0;
        return;
    }
    acc[i] = 0;
    const long long k = (long long)(codes[i] / (unsigned long long)c.ntri);
    const int t = (int)(codes[i] % (unsigned long long)c.ntri);
    const int v = c.sv[k];
    const int4 tr = c.tri[t];
    double vl[3], vh[3], tl[3], th[3];
    prim_box<R>(c, 0, (int)k, vl, vh);
    prim_box<R>(c, 1, t, tl, th);
    bool keep = tr.x != v && tr.y != v && tr.z != v;
    for (int q = 0; q < 3; ++q) keep = keep && tl[q] <= vh[q] && vl[q] <= th[q];
    keep = keep && (c.active[v] || c.active[tr.x] || c.active[tr.y] || c.active[tr.z]);
    if (!keep) return;
    const D3 s0 = ld3<R>(c.xs, tr.x), s1 = ld3<R>(c.xs, tr.y), s2 = ld3<R>(c.xs, tr.z), sv = ld3<R>(c.xs, v);
    const D3 e0 = ld3<R>(c.xe, tr.x), e1 = ld3<R>(c.xe, tr.y), e2 = ld3<R>(c.xe, tr.z), ev = ld3<R>(c.xe, v);
    const D3 u0 = s1 - s0, u1 = (e1 - e0) - u0, v0 = s2 - s0, v1 = (e2 - e0) - v0;
    const D3 w0 = sv - s0, w1 = (ev - e0) - w0;
    double co[4], rt[3];
    cubic_coeffs(u0, u1, v0, v1, w0, w1, co);
    const int nr = roots_unit(co[0], co[1], co[2], co[3], rt);
    for (int r = 0; r < nr; ++r) {
        const double toi = bisect(u0, u1, v0, v1, w0, w1, rt[r]);
        const D3 a = s0 + toi * (e0 - s0), b = s1 + toi * (e1 - s1), cc = s2 + toi * (e2 - s2), p = sv + toi * (ev - sv);
        const D3 nrm = cross(b - a, cc - a);
        const double nn = norm(nrm);
        if (!(nn >= 1e-30)) continue;
        const D3 f1 = b - a, f2 = cc - a;
        const double m00 = dot(f1, f1), m01 = dot(f1, f2), m11 = dot(f2, f2);
        const double det = m00 * m11 - m01 * m01;
        if (!(det > 0.0)) continue;
        const double r0 = dot(f1, p - a), r1 = dot(f2, p - a);
        const double wb = (m11 * r0 - m01 * r1) / det, wc = (m00 * r1 - m01 * r0) / det;
        const double wa = 1.0 - wb - wc;
        if (!(fmin(fmin(wa, wb), wc) >= -1e-8)) continue;
        D3 ni = d3(nrm.x / nn, nrm.y / nn, nrm.z / nn);
        double side = dot(sv - s0, ni);
        if (side == 0.0) side = -dot((ev - sv) - (e0 - s0), ni);
        if (side < 0.0) ni = d3(-ni.x, -ni.y, -ni.z);
        const double gam[4] = {1.0, -fmin(fmax(wa, 0.0), 1.0), -fmin(fmax(wb, 0.0), 1.0), -fmin(fmax(wc, 0.0), 1.0)};
        make_rec(out[i], make_int4(v, tr.x, tr.y, tr.z), gam, ni, kc, 0, 1);
        acc[i] = 1;
        return;
    }
}

// CCD edge-edge (contact.py:654-737); code = e * nedge + o, e < o
template <typename R>
__global__ void k_ccd_ee(const CollArgs<R> c, const unsigned long long* __restrict__ codes, long long n, double kc,
                         ContactRec* __restrict__ out, int* __restrict__ acc)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (codes[i] == VBD_SENT) {  // padding (graph mode)
        acc[i] = 0;
        return;
    }
    acc[i] = 0;
    const int e = (int)(codes[i] / (unsigned long long)c.nedge);
    const int o = (int)(codes[i] % (unsigned long long)c.nedge);
    const int2 ea = c.edge[e], eb = c.edge[o];
    double al[3], ah[3], bl[3], bh[3];
    prim_box<R>(c, 2, e, al, ah);
    prim_box<R>(c, 2, o, bl, bh);
    bool keep = ea.x != eb.x && ea.x != eb.y && ea.y != eb.x && ea.y != eb.y;
    for (int q = 0; q < 3; ++q) keep = keep && bl[q] <= ah[q] && al[q] <= bh[q];
    keep = keep && (c.active[ea.x] || c.active[ea.y] || c.active[eb.x] || c.active[eb.y]);
    if (!keep) return;
    const D3 sa0 = ld3<R>(c.xs, ea.x), sa1 = ld3<R>(c.xs, ea.y), sb0 = ld3<R>(c.xs, eb.x), sb1 = ld3<R>(c.xs, eb.y);
    const D3 xa0 = ld3<R>(c.xe, ea.x), xa1 = ld3<R>(c.xe, ea.y), xb0 = ld3<R>(c.xe, eb.x), xb1 = ld3<R>(c.xe, eb.y);
    const D3 u0 = sa1 - sa0, u1 = (xa1 - xa0) - u0, v0 = sb1 - sb0, v1 = (xb1 - xb0) - v0;
    const D3 w0 = sb0 - sa0, w1 = (xb0 - xa0) - w0;
    double co[4], rt[3];
    cubic_coeffs(u0, u1, v0, v1, w0, w1, co);
    const int nr = roots_unit(co[0], co[1], co[2], co[3], rt);
    for (int r = 0; r < nr; ++r) {
        const double toi = bisect(u0, u1, v0, v1, w0, w1, rt[r]);
        const D3 pa0 = sa0 + toi * (xa0 - sa0), pa1 = sa1 + toi * (xa1 - sa1);
        const D3 pb0 = sb0 + toi * (xb0 - sb0), pb1 = sb1 + toi * (xb1 - sb1);
        const D3 da = pa1 - pa0, db = pb1 - pb0;
        const double la = norm(da), lb = norm(db);
        if (!(la >= 1e-30 && lb >= 1e-30)) continue;
        const D3 cr = cross(d3(da.x / la, da.y / la, da.z / la), d3(db.x / lb, db.y / lb, db.z / lb));
        const double cn = norm(cr);
        if (!(cn >= 1e-9)) continue;
        const D3 rr = pb0 - pa0;
        const double aa = dot(da, da), ee = dot(db, db), bb = dot(da, db);
        const double denom = aa * ee - bb * bb;
        if (!(denom > 1e-30)) continue;
        const double dbr = dot(db, rr), dar = dot(da, rr);
        const double s = (bb * (-dbr) + ee * dar) / denom;
        const double tt = (bb * s - dbr) / ee;
        if (!(fmin(fmin(s, 1.0 - s), fmin(tt, 1.0 - tt)) >= -1e-8)) continue;
        const double si = fmin(fmax(s, 0.0), 1.0), ti = fmin(fmax(tt, 0.0), 1.0);
        D3 nv = d3(cr.x / cn, cr.y / cn, cr.z / cn);
        double side = dot(((1 - ti) * sb0 + ti * sb1) - ((1 - si) * sa0 + si * sa1), nv);
        if (side == 0.0) side = dot(sb0 - sa0, nv);
        if (side > 0.0) nv = d3(-nv.x, -nv.y, -nv.z);
        const double gam[4] = {1.0 - si, si, -(1.0 - ti), -ti};
        make_rec(out[i], make_int4(ea.x, ea.y, eb.x, eb.y), gam, nv, kc, 0, 1);
        acc[i] = 1;
        return;
    }
}

// gap d = -sum_k gamma_k n . x_k > 0 at the given positions, flag the contact's vertices
// (ContactSet.mark_flags, contact.py:111-118: DCD by gap, CCD always)
template <typename R>
__global__ void k_mark_flags(const ContactRec* __restrict__ recs, int n, const typename Vec4<R>::T* __restrict__ x,
                             unsigned char* __restrict__ flag)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ContactRec& r = recs[i];
    if (r.idx.x < 0) return;  // padding (graph mode)
    const int ids[4] = {r.idx.x, r.idx.y, r.idx.z, r.idx.w};
    bool on = r.ccd != 0;
    if (!on) {  // Contact.gap: sep = -(sum_k gamma_k x_k), d = sep . n (contact.py:70-74)
        D3 acc = r.g[0] * ld3<R>(x, ids[0]);
        for (int k = 1; k < 4; ++k) acc = acc + r.g[k] * ld3<R>(x, ids[k]);
        const D3 sep = d3(-acc.x, -acc.y, -acc.z);
        on = (sep.x * r.n[0] + sep.y * r.n[1] + sep.z * r.n[2]) > 0.0;
    }
    if (on)
        for (int k = 0; k < 4; ++k) flag[ids[k]] = 1;
}

// K1 records (cidx, creal) and the (vertex << 32 | cid) incidence keys of each contact
template <typename R>
__global__ void k_pack_contacts(const ContactRec* __restrict__ recs, int n, int4* __restrict__ cidx,
                                typename Vec4<R>::T* __restrict__ creal, unsigned long long* __restrict__ inc)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const ContactRec& r = recs[i];
    if (r.idx.x < 0) {  // padding (graph mode): sorts after every real key
        for (int k = 0; k < 4; ++k) inc[4 * i + k] = VBD_SENT;
        return;
    }
    cidx[i] = r.idx;
    typename Vec4<R>::T* o = creal + 4 * i;
    o[0].x = (R)r.g[0]; o[0].y = (R)r.g[1]; o[0].z = (R)r.g[2]; o[0].w = (R)r.g[3];
    o[1].x = (R)r.n[0]; o[1].y = (R)r.n[1]; o[1].z = (R)r.n[2]; o[1].w = (R)r.kc;
    o[2].x = (R)r.t[0]; o[2].y = (R)r.t[1]; o[2].z = (R)r.t[2]; o[2].w = (R)r.t[3];
    o[3].x = (R)r.t[4]; o[3].y = (R)r.t[5]; o[3].z = (R)r.refresh; o[3].w = R(0);
    const int ids[4] = {r.idx.x, r.idx.y, r.idx.z, r.idx.w};
    for (int k = 0; k < 4; ++k)
        inc[4 * i + k] = ((unsigned long long)(unsigned)ids[k] << 32) | ((unsigned long long)i << 2) | (unsigned)k;
}

// per solved vertex CSR from the sorted incidence keys (cid << 2 | slot in the low word)
__global__ void k_contact_csr(const unsigned long long* __restrict__ keys, long long m, long long nsolve,
                              long long* __restrict__ off, int* __restrict__ cid, int* __restrict__ slot)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const bool pad = keys[i] == VBD_SENT;  // graph mode: keys of padding records sort last
    const long long v = pad ? nsolve + 1 : (long long)(keys[i] >> 32);
    const unsigned lo = (unsigned)(keys[i] & 0xffffffffu);
    if (!pad) {
        cid[i] = (int)(lo >> 2);
        slot[i] = (int)(lo & 3u);
    }
    if (pad && i > 0 && keys[i - 1] == VBD_SENT) return;
    // off[v + 1] = index of the first key with vertex > v
    const long long vp = i > 0 ? (long long)(keys[i - 1] >> 32) : -1;
    for (long long u = vp + 1; u <= v && u <= nsolve; ++u) off[u] = i;
    if (i == m - 1)
        for (long long u = v + 1; u <= nsolve; ++u) off[u] = m;
}


// contact penalty energy sum_c 1/2 k_c max(0, d)^2 with the detection-time weights
// (_assembly.py:49-56, Contact.gap contact.py:70-74); gap_max[block] = the block's largest
// gap d, for the max_penetration metric (solver.py:327-332)
template <typename R>
__global__ void __launch_bounds__(256) k_energy_contact(const int4* __restrict__ cidx,
                                                        const typename Vec4<R>::T* __restrict__ creal, int n,
                                                        const typename Vec4<R>::T* __restrict__ x, double* partial,
                                                        double* gap_max)
{
    __shared__ double red[256], mx[256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0, d = 0.0;
    if (i < n && cidx[i].x >= 0) {  // (padding records of the graph-mode arrays: idx.x = -1)
        const int4 id = cidx[i];
        const int ids[4] = {id.x, id.y, id.z, id.w};
        const typename Vec4<R>::T g = creal[4 * i], nk = creal[4 * i + 1];
        const double gam[4] = {g.x, g.y, g.z, g.w};
        D3 acc = gam[0] * ld3<R>(x, ids[0]);
        for (int k = 1; k < 4; ++k) acc = acc + gam[k] * ld3<R>(x, ids[k]);
        d = fmax(0.0, -(acc.x * nk.x + acc.y * nk.y + acc.z * nk.z));
        e = 0.5 * (double)nk.w * d * d;
    }
    red[threadIdx.x] = e;
    mx[threadIdx.x] = d;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[threadIdx.x] += red[threadIdx.x + o];
            mx[threadIdx.x] = fmax(mx[threadIdx.x], mx[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = red[0];
        gap_max[blockIdx.x] = mx[0];
    }
}
