/*
 * vbd_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never shipped,
 * never called by the product path).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Plain-C fp64 restatement of the reference VBD colour pass (tets, springs,
 * contacts with friction, fixed / subspace / world-box constraints, mode 0 block-Newton,
 * mode 1 diagonal GD, optional 17-trial local line search), written so that its floating-point
 * operation order is the reference's, hence bit-identical to the reference's
 * compiled kernel when built without FP contraction:
 *
 *   _tet_fc          <- /root/reference/pkg/src/vbdsim/_native.pyx:175-198
 *   _local_energy    <- _native.pyx:201-258 (inertia, tet, spring, box terms)
 *   _assemble        <- _native.pyx:261-317 (inertia + SNH tets + damping),
 *                       319-349 (springs), 351-399 (contacts + friction),
 *                       401-409 (world box)
 *   _contact_gamma   <- _native.pyx:134-172, _closest_bary <- :79-131
 *   _solve_vertex    <- _native.pyx:412-494 (fixed skip, mode 1, subspace
 *                       1D/2D solve, adjugate solve with relative det guard,
 *                       line search)
 *   color_pass       <- _native.pyx:513-589 (aux buffer + serial merge)
 *   greedy_color     <- /root/reference/pkg/src/vbdsim/mesh.py:270-302
 *   beam connectivity<- /root/reference/pkg/src/vbdsim/harness.py:28-67
 *
 * Parity is pinned in tests/test_oracle.py against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py) and, live, against the
 * reference's own compiled kernel built into oracle/_ref/ (oracle/Makefile).
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ORACLE_F32 (liboracle_f32.so): the same restatement with every real -- arrays, scalars and
 * literals (-fsingle-precision-constant) -- in binary32.  It is the fp32-arithmetic SENSITIVITY
 * yardstick for ill-conditioned inputs (tests/test_gpu_configs.py, C2 extreme init), never a
 * parity reference. */
#ifdef ORACLE_F32
typedef float f64;
#else
typedef double f64;
#endif
typedef int64_t i64;

#define KIND_FIXED 1
#define KIND_SUBSPACE 2

typedef struct {
    const f64 *x, *xt, *y, *masses;
    const i64 *tets;
    const f64 *tet_w, *tet_vol, *tet_mu, *tet_lam, *tet_kd;
    const i64 *t_off, *t_id, *t_slot;
    const uint8_t *kind;
    f64 h, eps_det;
    int mode, line_search;
    /* springs (_system.py:117-123) and constraints (_system.py:76-83); NULL = none */
    const i64 *springs, *s_off, *s_id, *s_slot;
    const f64 *sp_l0, *sp_k, *sp_kd;
    const i64 *sub_dim;
    const f64 *sub_basis, *box_k, *box_lo, *box_hi;
    /* contacts (ContactArrays, _system.py:86-96); cv_off NULL = none */
    const i64 *c_idx, *cv_off, *cv_cid, *cv_slot;
    const f64 *c_gamma, *c_n, *c_t, *c_kc;
    const uint8_t *c_refresh;
    f64 mu_c, eps_u;
} osys;

/* Voronoi-region closest point on triangle abc, barycentric (_native.pyx:79-131). */
static void closest_bary(const f64 *p, const f64 *a, const f64 *b, const f64 *c, f64 *bary)
{
    f64 ab[3], ac[3], ap[3], bp[3], cp[3];
    for (int k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
    }
    f64 d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    f64 d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    if (d1 <= 0.0 && d2 <= 0.0) { bary[0] = 1.0; bary[1] = 0.0; bary[2] = 0.0; return; }
    for (int k = 0; k < 3; ++k) bp[k] = p[k] - b[k];
    f64 d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    f64 d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    if (d3 >= 0.0 && d4 <= d3) { bary[0] = 0.0; bary[1] = 1.0; bary[2] = 0.0; return; }
    f64 vc = d1 * d4 - d3 * d2, v, w;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        v = d1 / (d1 - d3);
        bary[0] = 1.0 - v; bary[1] = v; bary[2] = 0.0;
        return;
    }
    for (int k = 0; k < 3; ++k) cp[k] = p[k] - c[k];
    f64 d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    f64 d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    if (d6 >= 0.0 && d5 <= d6) { bary[0] = 0.0; bary[1] = 0.0; bary[2] = 1.0; return; }
    f64 vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        w = d2 / (d2 - d6);
        bary[0] = 1.0 - w; bary[1] = 0.0; bary[2] = w;
        return;
    }
    f64 va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        bary[0] = 0.0; bary[1] = 1.0 - w; bary[2] = w;
        return;
    }
    f64 denom = 1.0 / (va + vb + vc);
    v = vb * denom;
    w = vc * denom;
    bary[0] = 1.0 - v - w; bary[1] = v; bary[2] = w;
}

/* Signed contact weights; DCD vertex-triangle anchors follow the current closest point
 * (_native.pyx:134-172). */
static void contact_gamma(const osys *s, i64 cid, f64 *gam)
{
    for (int k = 0; k < 4; ++k) gam[k] = s->c_gamma[cid * 4 + k];
    if (!s->c_refresh[cid]) return;
    i64 v = s->c_idx[cid * 4 + 0], t0 = s->c_idx[cid * 4 + 1], t1 = s->c_idx[cid * 4 + 2],
        t2 = s->c_idx[cid * 4 + 3];
    f64 e1[3], e2[3], nrm[3], bary[3], l1 = 0.0, l2 = 0.0, nn, scale;
    for (int k = 0; k < 3; ++k) {
        e1[k] = s->x[t1 * 3 + k] - s->x[t0 * 3 + k];
        e2[k] = s->x[t2 * 3 + k] - s->x[t0 * 3 + k];
        l1 = l1 + e1[k] * e1[k];
        l2 = l2 + e2[k] * e2[k];
    }
    nrm[0] = e1[1] * e2[2] - e1[2] * e2[1];
    nrm[1] = e1[2] * e2[0] - e1[0] * e2[2];
    nrm[2] = e1[0] * e2[1] - e1[1] * e2[0];
    nn = sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
    scale = l1 > l2 ? sqrt(l1) : sqrt(l2);
    if (scale < 1e-30) scale = 1e-30;
    if (nn < (1e-12 * scale) * scale) return;
    closest_bary(&s->x[v * 3], &s->x[t0 * 3], &s->x[t1 * 3], &s->x[t2 * 3], bary);
    gam[0] = 1.0;
    gam[1] = -bary[0];
    gam[2] = -bary[1];
    gam[3] = -bary[2];
}

/* F = sum_k x_k w_k^T with vertex i at p; cofactor; det by column-0 expansion
 * (_native.pyx:175-198). */
static void tet_fc(const osys *s, i64 t, i64 i, const f64 *p, f64 *F, f64 *C, f64 *J)
{
    for (int k = 0; k < 9; ++k) F[k] = 0.0;
    for (int k = 0; k < 4; ++k) {
        i64 vid = s->tets[t * 4 + k];
        const f64 *pos = (vid == i) ? p : &s->x[vid * 3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                F[a * 3 + b] += pos[a] * s->tet_w[t * 12 + k * 3 + b];
    }
    C[0] = F[4] * F[8] - F[7] * F[5];
    C[3] = F[7] * F[2] - F[1] * F[8];
    C[6] = F[1] * F[5] - F[4] * F[2];
    C[1] = F[5] * F[6] - F[8] * F[3];
    C[4] = F[8] * F[0] - F[2] * F[6];
    C[7] = F[2] * F[3] - F[5] * F[0];
    C[2] = F[3] * F[7] - F[6] * F[4];
    C[5] = F[6] * F[1] - F[0] * F[7];
    C[8] = F[0] * F[4] - F[3] * F[1];
    *J = F[0] * C[0] + F[3] * C[3] + F[6] * C[6];
}

/* G_i with vertex i at p (inertia + SNH tets), _native.pyx:201-258. */
static f64 local_energy(const osys *s, i64 i, const f64 *p)
{
    f64 e = 0.0, h2 = s->h * s->h, F[9], C[9], J;
    for (int a = 0; a < 3; ++a) {
        f64 d = p[a] - s->y[i * 3 + a];
        e = e + ((0.5 * (s->masses[i] / h2)) * d) * d;
    }
    for (i64 kk = s->t_off[i]; kk < s->t_off[i + 1]; ++kk) {
        i64 t = s->t_id[kk];
        tet_fc(s, t, i, p, F, C, &J);
        f64 ic = 0.0;
        for (int k = 0; k < 9; ++k) ic += F[k] * F[k];
        f64 mu = s->tet_mu[t], lam = s->tet_lam[t];
        f64 g = 1.0 + mu / lam;
        f64 psi = ((0.5 * mu) * (ic - 3.0)) + (((0.5 * lam) * (J - g)) * (J - g));
        e = e + s->tet_vol[t] * psi;
    }
    if (s->springs)
        for (i64 kk = s->s_off[i]; kk < s->s_off[i + 1]; ++kk) {
            i64 sp = s->s_id[kk];
            i64 oth = s->springs[sp * 2 + (1 - s->s_slot[kk])];
            f64 length = 0.0, d;
            for (int a = 0; a < 3; ++a) {
                d = p[a] - s->x[oth * 3 + a];
                length = length + d * d;
            }
            length = sqrt(length);
            if (length < 1e-12 * s->sp_l0[sp])
                e = e + ((0.5 * s->sp_k[sp]) * s->sp_l0[sp]) * s->sp_l0[sp];
            else {
                d = length - s->sp_l0[sp];
                e = e + ((0.5 * s->sp_k[sp]) * d) * d;
            }
        }
    if (s->cv_off) /* _native.pyx:239-249 */
        for (i64 kk = s->cv_off[i]; kk < s->cv_off[i + 1]; ++kk) {
            i64 cid = s->cv_cid[kk];
            f64 gam[4], d = 0.0;
            contact_gamma(s, cid, gam);
            for (int k = 0; k < 4; ++k) {
                i64 oth = s->c_idx[cid * 4 + k];
                for (int a = 0; a < 3; ++a) {
                    f64 tmp = (oth == i && k == s->cv_slot[kk]) ? p[a] : s->x[oth * 3 + a];
                    d = d - (gam[k] * s->c_n[cid * 3 + a]) * tmp;
                }
            }
            if (d > 0.0) e = e + ((0.5 * s->c_kc[cid]) * d) * d;
        }
    if (s->box_k && s->box_k[i] > 0.0)
        for (int a = 0; a < 3; ++a) {
            f64 d = s->box_lo[i * 3 + a] - p[a];
            if (d > 0.0) e = e + ((0.5 * s->box_k[i]) * d) * d;
            d = p[a] - s->box_hi[i * 3 + a];
            if (d > 0.0) e = e + ((0.5 * s->box_k[i]) * d) * d;
        }
    return e;
}

/* force f = -grad G_i and 3x3 Hessian at the current x, _native.pyx:261-317. */
static void assemble(const osys *s, i64 i, f64 *f, f64 *H)
{
    f64 h2 = s->h * s->h, mih2 = s->masses[i] / h2;
    f64 F[9], C[9], He[9], w[3], cw[3], J;
    for (int a = 0; a < 3; ++a) {
        f[a] = mih2 * (s->y[i * 3 + a] - s->x[i * 3 + a]);
        for (int b = 0; b < 3; ++b) H[a * 3 + b] = (a == b) ? mih2 : 0.0;
    }
    for (i64 kk = s->t_off[i]; kk < s->t_off[i + 1]; ++kk) {
        i64 t = s->t_id[kk], slot = s->t_slot[kk];
        tet_fc(s, t, i, &s->x[i * 3], F, C, &J);
        f64 mu = s->tet_mu[t], lam = s->tet_lam[t];
        f64 g = 1.0 + mu / lam;
        f64 vol = s->tet_vol[t];
        f64 wsq = 0.0;
        for (int a = 0; a < 3; ++a) {
            w[a] = s->tet_w[t * 12 + slot * 3 + a];
            wsq += w[a] * w[a];
        }
        for (int a = 0; a < 3; ++a) {
            cw[a] = 0.0;
            for (int b = 0; b < 3; ++b) cw[a] += C[a * 3 + b] * w[b];
        }
        f64 coef = lam * (J - g);
        for (int a = 0; a < 3; ++a) {
            f64 tmp = 0.0;
            for (int b = 0; b < 3; ++b) tmp = tmp + ((mu * F[a * 3 + b]) + (coef * C[a * 3 + b])) * w[b];
            f[a] -= vol * tmp;
        }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                f64 diag = (a == b) ? mu * wsq : 0.0;
                He[a * 3 + b] = vol * (((lam * cw[a]) * cw[b]) + diag);
            }
        f64 dsc = s->tet_kd[t] / s->h;
        for (int a = 0; a < 3; ++a) {
            f64 tmp = 0.0;
            for (int b = 0; b < 3; ++b) tmp = tmp + He[a * 3 + b] * (s->x[i * 3 + b] - s->xt[i * 3 + b]);
            f[a] -= dsc * tmp;
        }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) H[a * 3 + b] = H[a * 3 + b] + (1.0 + dsc) * He[a * 3 + b];
    }
    if (s->springs) /* _native.pyx:319-349 */
        for (i64 kk = s->s_off[i]; kk < s->s_off[i + 1]; ++kk) {
            i64 sp = s->s_id[kk];
            i64 oth = s->springs[sp * 2 + (1 - s->s_slot[kk])];
            f64 dvec[3], length = 0.0;
            for (int a = 0; a < 3; ++a) {
                dvec[a] = s->x[i * 3 + a] - s->x[oth * 3 + a];
                length = length + dvec[a] * dvec[a];
            }
            length = sqrt(length);
            f64 k = s->sp_k[sp], l0 = s->sp_l0[sp];
            if (length < 1e-12 * l0) {
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) He[a * 3 + b] = (a == b) ? k : 0.0;
            } else {
                for (int a = 0; a < 3; ++a) dvec[a] = dvec[a] / length;
                f64 coef = 1.0 - l0 / length;
                for (int a = 0; a < 3; ++a) {
                    f[a] = f[a] - (k * (length - l0)) * dvec[a];
                    for (int b = 0; b < 3; ++b)
                        He[a * 3 + b] = k * (dvec[a] * dvec[b] + coef * (((a == b) ? 1.0 : 0.0) - dvec[a] * dvec[b]));
                }
            }
            f64 dsc = s->sp_kd[sp] / s->h;
            for (int a = 0; a < 3; ++a) {
                f64 tmp = 0.0;
                for (int b = 0; b < 3; ++b) tmp = tmp + He[a * 3 + b] * (s->x[i * 3 + b] - s->xt[i * 3 + b]);
                f[a] = f[a] - dsc * tmp;
            }
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) H[a * 3 + b] = H[a * 3 + b] + (1.0 + dsc) * He[a * 3 + b];
        }
    if (s->cv_off) /* _native.pyx:351-399 */
        for (i64 kk = s->cv_off[i]; kk < s->cv_off[i + 1]; ++kk) {
            i64 cid = s->cv_cid[kk], slot = s->cv_slot[kk];
            f64 gam[4], d = 0.0, dvec[3], u[2], tvec[3];
            contact_gamma(s, cid, gam);
            for (int k = 0; k < 4; ++k) {
                i64 oth = s->c_idx[cid * 4 + k];
                for (int a = 0; a < 3; ++a) d = d - (gam[k] * s->c_n[cid * 3 + a]) * s->x[oth * 3 + a];
            }
            if (d <= 0.0) continue;
            const f64 *n = &s->c_n[cid * 3], *ct = &s->c_t[cid * 6];
            f64 kc = s->c_kc[cid];
            f64 coef = (kc * d) * gam[slot];
            for (int a = 0; a < 3; ++a) f[a] = f[a] + coef * n[a];
            coef = (kc * gam[slot]) * gam[slot];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) H[a * 3 + b] = H[a * 3 + b] + (coef * n[a]) * n[b];
            if (s->mu_c > 0.0) {
                f64 lamc = kc * d, ratio;
                for (int a = 0; a < 3; ++a) dvec[a] = 0.0;
                for (int k = 0; k < 4; ++k) {
                    i64 oth = s->c_idx[cid * 4 + k];
                    for (int a = 0; a < 3; ++a) dvec[a] = dvec[a] + gam[k] * (s->x[oth * 3 + a] - s->xt[oth * 3 + a]);
                }
                for (int k = 0; k < 2; ++k) {
                    u[k] = 0.0;
                    for (int a = 0; a < 3; ++a) u[k] = u[k] + ct[a * 2 + k] * dvec[a];
                }
                f64 unorm = sqrt(u[0] * u[0] + u[1] * u[1]);
                if (unorm < 1e-14) {
                    ratio = 2.0 / s->eps_u;
                } else {
                    f64 r = unorm / s->eps_u;
                    f64 f1 = unorm >= s->eps_u ? 1.0 : 2.0 * r - r * r;
                    ratio = f1 / unorm;
                    coef = ((-s->mu_c * lamc) * gam[slot]) * ratio;
                    for (int a = 0; a < 3; ++a) {
                        tvec[a] = ct[a * 2 + 0] * u[0] + ct[a * 2 + 1] * u[1];
                        f[a] = f[a] + coef * tvec[a];
                    }
                }
                coef = (((s->mu_c * lamc) * gam[slot]) * gam[slot]) * ratio;
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        H[a * 3 + b] = H[a * 3 + b] + coef * (ct[a * 2 + 0] * ct[b * 2 + 0] + ct[a * 2 + 1] * ct[b * 2 + 1]);
            }
        }
    if (s->box_k && s->box_k[i] > 0.0) /* _native.pyx:401-409 */
        for (int a = 0; a < 3; ++a) {
            f64 tmp = s->x[i * 3 + a];
            if (tmp < s->box_lo[i * 3 + a]) {
                f[a] = f[a] - s->box_k[i] * (tmp - s->box_lo[i * 3 + a]);
                H[a * 4] = H[a * 4] + s->box_k[i];
            } else if (tmp > s->box_hi[i * 3 + a]) {
                f[a] = f[a] - s->box_k[i] * (tmp - s->box_hi[i * 3 + a]);
                H[a * 4] = H[a * 4] + s->box_k[i];
            }
        }
}

/* one vertex solve into out[3], _native.pyx:412-494. */
static void solve_vertex(const osys *s, i64 i, f64 *out)
{
    f64 f[3], H[9], d[3] = {0.0, 0.0, 0.0}, adj[9];
    for (int a = 0; a < 3; ++a) out[a] = s->x[i * 3 + a];
    if (s->kind && s->kind[i] == KIND_FIXED) return;
    assemble(s, i, f, H);
    if (s->mode == 1) {
        for (int a = 0; a < 3; ++a)
            if (H[a * 3 + a] != 0.0) d[a] = f[a] / H[a * 3 + a];
    } else if (s->kind && s->kind[i] == KIND_SUBSPACE) { /* _native.pyx:435-463 */
        const f64 *B = &s->sub_basis[i * 6];
        i64 dim = s->sub_dim[i];
        f64 rhs[2], amat[4], det, tr, q0, q1;
        for (int a = 0; a < dim; ++a) {
            rhs[a] = 0.0;
            for (int k = 0; k < 3; ++k) rhs[a] = rhs[a] + B[k * 2 + a] * f[k];
            for (int b = 0; b < dim; ++b) {
                amat[a * 2 + b] = 0.0;
                for (int k = 0; k < 3; ++k) {
                    q0 = 0.0;
                    for (int t = 0; t < 3; ++t) q0 = q0 + H[k * 3 + t] * B[t * 2 + b];
                    amat[a * 2 + b] = amat[a * 2 + b] + B[k * 2 + a] * q0;
                }
            }
        }
        if (dim == 1) {
            det = amat[0];
            tr = amat[0];
            if (fabs(det) > s->eps_det * fabs(tr)) {
                q0 = rhs[0] / amat[0];
                for (int a = 0; a < 3; ++a) d[a] = B[a * 2] * q0;
            }
        } else {
            det = amat[0] * amat[3] - amat[1] * amat[2];
            tr = 0.5 * (amat[0] + amat[3]);
            if (fabs(det) > (s->eps_det * tr) * tr) {
                q0 = (amat[3] * rhs[0] - amat[1] * rhs[1]) / det;
                q1 = (amat[0] * rhs[1] - amat[2] * rhs[0]) / det;
                for (int a = 0; a < 3; ++a) d[a] = B[a * 2] * q0 + B[a * 2 + 1] * q1;
            }
        }
    } else {
        adj[0] = H[4] * H[8] - H[5] * H[7];
        adj[1] = H[2] * H[7] - H[1] * H[8];
        adj[2] = H[1] * H[5] - H[2] * H[4];
        adj[3] = H[5] * H[6] - H[3] * H[8];
        adj[4] = H[0] * H[8] - H[2] * H[6];
        adj[5] = H[2] * H[3] - H[0] * H[5];
        adj[6] = H[3] * H[7] - H[4] * H[6];
        adj[7] = H[1] * H[6] - H[0] * H[7];
        adj[8] = H[0] * H[4] - H[1] * H[3];
        f64 det = H[0] * adj[0] + H[1] * adj[3] + H[2] * adj[6];
        f64 tr = ((H[0] + H[4]) + H[8]) / 3.0;
        if (fabs(det) > ((s->eps_det * tr) * tr) * tr)
            for (int a = 0; a < 3; ++a)
                d[a] = (adj[a * 3 + 0] * f[0] + adj[a * 3 + 1] * f[1] + adj[a * 3 + 2] * f[2]) / det;
    }
    if (s->line_search && s->mode == 0) {
        f64 e0 = local_energy(s, i, &s->x[i * 3]), alpha = 1.0, cand[3];
        for (int trial = 0; trial < 17; ++trial) {
            for (int a = 0; a < 3; ++a) cand[a] = s->x[i * 3 + a] + alpha * d[a];
            if (local_energy(s, i, cand) <= e0) {
                for (int a = 0; a < 3; ++a) out[a] = cand[a];
                return;
            }
            alpha *= 0.5;
        }
        return;
    }
    for (int a = 0; a < 3; ++a) out[a] = s->x[i * 3 + a] + d[a];
}

/* Aux-buffer colour pass (_native.pyx:513-589): every vertex of `group` reads
 * the main buffer x, results land in a scratch buffer merged afterwards, so the
 * output is independent of thread count.  Returns 0, or -1 on bad args. */
int oracle_color_pass(i64 n_vertices, f64 *x, const f64 *xt, const f64 *y, const f64 *masses,
                      const i64 *tets, const f64 *tet_w, const f64 *tet_vol, const f64 *tet_mu,
                      const f64 *tet_lam, const f64 *tet_kd, const i64 *t_off, const i64 *t_id,
                      const i64 *t_slot, const uint8_t *kind, f64 h, const i64 *group, i64 ng,
                      int mode, int line_search, f64 eps_det, int n_threads)
{
    (void)n_vertices;
    if (ng <= 0) return 0;
    osys s;
    memset(&s, 0, sizeof s);
    s.x = x; s.xt = xt; s.y = y; s.masses = masses; s.tets = tets; s.tet_w = tet_w;
    s.tet_vol = tet_vol; s.tet_mu = tet_mu; s.tet_lam = tet_lam; s.tet_kd = tet_kd;
    s.t_off = t_off; s.t_id = t_id; s.t_slot = t_slot; s.kind = kind; s.h = h;
    s.eps_det = eps_det; s.mode = mode; s.line_search = line_search;
    f64 *out = (f64 *)malloc((size_t)ng * 3 * sizeof(f64));
    if (!out) return -1;
#ifdef _OPENMP
    int nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
#endif
    for (i64 k = 0; k < ng; ++k) solve_vertex(&s, group[k], &out[k * 3]);
    for (i64 k = 0; k < ng; ++k) {
        i64 v = group[k];
        x[v * 3 + 0] = out[k * 3 + 0];
        x[v * 3 + 1] = out[k * 3 + 1];
        x[v * 3 + 2] = out[k * 3 + 2];
    }
    free(out);
    (void)n_threads;
    return 0;
}

/* The same pass with springs and constraints (any pointer may be NULL). */
int oracle_color_pass_ex(i64 n_vertices, f64 *x, const f64 *xt, const f64 *y, const f64 *masses,
                         const i64 *tets, const f64 *tet_w, const f64 *tet_vol, const f64 *tet_mu,
                         const f64 *tet_lam, const f64 *tet_kd, const i64 *t_off, const i64 *t_id,
                         const i64 *t_slot, const uint8_t *kind, f64 h, const i64 *group, i64 ng,
                         int mode, int line_search, f64 eps_det, int n_threads,
                         const i64 *springs, const f64 *sp_l0, const f64 *sp_k, const f64 *sp_kd,
                         const i64 *s_off, const i64 *s_id, const i64 *s_slot, const i64 *sub_dim,
                         const f64 *sub_basis, const f64 *box_k, const f64 *box_lo, const f64 *box_hi,
                         const i64 *c_idx, const f64 *c_gamma, const uint8_t *c_refresh, const f64 *c_n,
                         const f64 *c_t, const f64 *c_kc, const i64 *cv_off, const i64 *cv_cid,
                         const i64 *cv_slot, f64 mu_c, f64 eps_v)
{
    (void)n_vertices;
    if (ng <= 0) return 0;
    osys s = {x, xt, y, masses, tets, tet_w, tet_vol, tet_mu, tet_lam, tet_kd,
              t_off, t_id, t_slot, kind, h, eps_det, mode, line_search,
              springs, s_off, s_id, s_slot, sp_l0, sp_k, sp_kd, sub_dim, sub_basis,
              box_k, box_lo, box_hi, c_idx, cv_off, cv_cid, cv_slot, c_gamma, c_n, c_t, c_kc,
              c_refresh, mu_c, eps_v * h};
    f64 *out = (f64 *)malloc((size_t)ng * 3 * sizeof(f64));
    if (!out) return -1;
#ifdef _OPENMP
    int nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
#endif
    for (i64 k = 0; k < ng; ++k) solve_vertex(&s, group[k], &out[k * 3]);
    for (i64 k = 0; k < ng; ++k) {
        i64 v = group[k];
        x[v * 3 + 0] = out[k * 3 + 0];
        x[v * 3 + 1] = out[k * 3 + 1];
        x[v * 3 + 2] = out[k * 3 + 2];
    }
    free(out);
    (void)n_threads;
    return 0;
}

/* Local energy G_i at p (exposed for the line-search parity tests). */
f64 oracle_local_energy(const f64 *x, const f64 *y, const f64 *masses, const i64 *tets,
                        const f64 *tet_w, const f64 *tet_vol, const f64 *tet_mu,
                        const f64 *tet_lam, const i64 *t_off, const i64 *t_id, f64 h, i64 i,
                        const f64 *p)
{
    osys s;
    memset(&s, 0, sizeof s);
    s.x = x; s.y = y; s.masses = masses; s.tets = tets; s.tet_w = tet_w; s.tet_vol = tet_vol;
    s.tet_mu = tet_mu; s.tet_lam = tet_lam; s.t_off = t_off; s.t_id = t_id; s.h = h;
    return local_energy(&s, i, p);
}

/* Sequential greedy colouring, mesh.py:270-302: visit vertices in `order`
 * (default: descending degree, ties by index), give each the smallest colour
 * not used by an already-coloured neighbour.  Returns the number of colours. */
static const i64 *g_deg;
static int cmp_order(const void *pa, const void *pb)
{
    i64 a = *(const i64 *)pa, b = *(const i64 *)pb;
    if (g_deg[a] != g_deg[b]) return g_deg[a] > g_deg[b] ? -1 : 1;
    return (a < b) ? -1 : (a > b);
}

i64 oracle_greedy_color(i64 n, const i64 *noff, const i64 *nids, const i64 *order_in, i64 *color_of)
{
    i64 *order = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    i64 *deg = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    unsigned char *taken = NULL;
    i64 cap = 0, ncol = 0;
    for (i64 v = 0; v < n; ++v) {
        deg[v] = noff[v + 1] - noff[v];
        color_of[v] = -1;
        order[v] = order_in ? order_in[v] : v;
    }
    if (!order_in) {
        g_deg = deg;
        qsort(order, (size_t)n, sizeof(i64), cmp_order);
    }
    for (i64 k = 0; k < n; ++k) {
        i64 v = order[k];
        i64 need = deg[v] + 2;
        if (need > cap) {
            cap = need * 2;
            taken = (unsigned char *)realloc(taken, (size_t)cap);
        }
        memset(taken, 0, (size_t)need);
        for (i64 e = noff[v]; e < noff[v + 1]; ++e) {
            i64 c = color_of[nids[e]];
            if (c >= 0 && c < need) taken[c] = 1;
        }
        i64 c = 0;
        while (taken[c]) ++c;
        color_of[v] = c;
        if (c + 1 > ncol) ncol = c + 1;
    }
    free(order);
    free(deg);
    free(taken);
    return ncol;
}

/* Connectivity of generate_beam (harness.py:28-67): vertex id (ax*ny+ay)*nz+az,
 * 5 tets per hex cell alternated by cell parity; corner index 4dx+2dy+dz.
 * Writes (nx-1)(ny-1)(nz-1)*5 rows of 4 (before the orientation fix-up done by
 * build_tet_mesh). */
static const int CELL_EVEN[5][4] = {{0, 3, 5, 6}, {1, 0, 3, 5}, {2, 0, 3, 6}, {4, 0, 5, 6}, {7, 3, 5, 6}};
static const int CELL_ODD[5][4] = {{1, 2, 4, 7}, {0, 1, 2, 4}, {3, 1, 2, 7}, {5, 1, 4, 7}, {6, 2, 4, 7}};

void oracle_beam_tets(i64 nx, i64 ny, i64 nz, i64 *tets)
{
    i64 r = 0;
    for (i64 cx = 0; cx < nx - 1; ++cx)
        for (i64 cy = 0; cy < ny - 1; ++cy)
            for (i64 cz = 0; cz < nz - 1; ++cz) {
                i64 corner[8];
                for (int dx = 0; dx < 2; ++dx)
                    for (int dy = 0; dy < 2; ++dy)
                        for (int dz = 0; dz < 2; ++dz)
                            corner[dx * 4 + dy * 2 + dz] = ((cx + dx) * ny + (cy + dy)) * nz + (cz + dz);
                const int(*pat)[4] = ((cx + cy + cz) % 2 == 0) ? CELL_EVEN : CELL_ODD;
                for (int t = 0; t < 5; ++t, ++r)
                    for (int k = 0; k < 4; ++k) tets[r * 4 + k] = corner[pat[t][k]];
            }
}
