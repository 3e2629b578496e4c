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
    const PL* ent;           // entry planes
    long long E;             // plane stride (entries)
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
template <typename R, int W>
__device__ R local_energy(const K1Args<R>& a, long long beg, long long end, int lane, unsigned gmask,
                          const R* p, const typename Vec4<R>::T& y4)
{
    typedef typename Vec4<R>::T R4;
    R e = R(0);
    for (long long k = beg + lane; k < end; k += W) {
        const Entry<R> en = Entry<R>::load(a.ent, a.E, k);
        const R4 q0 = a.pos[en.n[0]], q1 = a.pos[en.n[1]], q2 = a.pos[en.n[2]];
        const R e0[3] = {q0.x - p[0], q0.y - p[1], q0.z - p[2]};
        const R e1[3] = {q1.x - p[0], q1.y - p[1], q1.z - p[2]};
        const R e2[3] = {q2.x - p[0], q2.y - p[1], q2.z - p[2]};
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
        const Material<R> m = a.mat[en.mat];
        const R psi = (R(0.5) * m.mu) * (ic - R(3)) + (R(0.5) * m.lam) * (J - m.gamma) * (J - m.gamma);
        e += en.V * psi;
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) e += __shfl_xor_sync(gmask, e, o, W);
    R ein = R(0);
    const R d0 = p[0] - y4.x, d1 = p[1] - y4.y, d2 = p[2] - y4.z;
    ein = ein + ((R(0.5) * y4.w) * d0) * d0;
    ein = ein + ((R(0.5) * y4.w) * d1) * d1;
    ein = ein + ((R(0.5) * y4.w) * d2) * d2;
    return ein + e;
}

template <typename R, int W, int U, bool UM, bool LS = false>
__device__ __forceinline__ void k1_vertex_impl(const K1Args<R>& a, int g, int lane)
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
    Material<R> mv;
    if (UM) mv = a.mat[a.vmat[v]];
    // U entries per lane per iteration: all their loads (entry planes, then the 3U
    // neighbour gathers) are issued before any math, for memory-level parallelism.
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
                const R e0[3] = {p[u][0].x - xi[0], p[u][0].y - xi[1], p[u][0].z - xi[2]};
                const R e1[3] = {p[u][1].x - xi[0], p[u][1].y - xi[1], p[u][1].z - xi[2]};
                const R e2[3] = {p[u][2].x - xi[0], p[u][2].y - xi[1], p[u][2].z - xi[2]};
                if (UM) {
                    tet_contrib<R, false>(e0, e1, e2, e[u].w, e[u].V, mv, dx, f, H);
                } else {
                    const Material<R> m = a.mat[e[u].mat];
                    tet_contrib<R, true>(e0, e1, e2, e[u].w, e[u].V, m, dx, f, H);
                }
            }
        }
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int q = 0; q < 3; ++q) f[q] += __shfl_xor_sync(gmask, f[q], o, W);
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] += __shfl_xor_sync(gmask, H[q], o, W);
    }
    if (!LS && lane != 0) return;
    if (UM && end > beg) {
        // hoisted Rayleigh damping (_native.pyx:309-317 summed over the vertex's tets):
        // f -= dsc (sum He) dx,  H = (1 + dsc) sum He
        const R hd0 = H[0] * dx[0] + H[1] * dx[1] + H[2] * dx[2];
        const R hd1 = H[1] * dx[0] + H[3] * dx[1] + H[4] * dx[2];
        const R hd2 = H[2] * dx[0] + H[4] * dx[1] + H[5] * dx[2];
        f[0] -= mv.dsc * hd0;
        f[1] -= mv.dsc * hd1;
        f[2] -= mv.dsc * hd2;
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] *= mv.opd;
    }
    const R4 y4 = a.y[v];
    const R mih2 = y4.w;  // inertia term, _native.pyx:278-281
    f[0] += mih2 * (y4.x - xi[0]);
    f[1] += mih2 * (y4.y - xi[1]);
    f[2] += mih2 * (y4.z - xi[2]);
    H[0] += mih2;
    H[3] += mih2;
    H[5] += mih2;
    R d[3];
    block_solve<R>(f, H, a.eps_det, a.mode, d);
    R4 nx = xi4;
    if (LS && a.mode == 0) {
        // 17-trial backtracking on G_i (_native.pyx:481-492); every lane of the group runs
        // the same trials on the same reduced energies
        const R e0 = local_energy<R, W>(a, beg, end, lane, gmask, xi, y4);
        R alpha = R(1);
        for (int trial = 0; trial < 17; ++trial) {
            const R cand[3] = {xi[0] + alpha * d[0], xi[1] + alpha * d[1], xi[2] + alpha * d[2]};
            if (local_energy<R, W>(a, beg, end, lane, gmask, cand, y4) <= e0) {
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
                __threadfence_system();
            } else if (j < a.nb[0] + a.nb[1]) {
                a.peer_pos[1][a.peer_off[1] + (j - a.nb[0])] = nx;
                __threadfence_system();
            }
        }
    }
    if (a.flag && !finite3(nx.x, nx.y, nx.z))
        atomicMin(a.flag, StepFlag::key((unsigned)*a.stepctr, (unsigned)a.iter, (unsigned)a.perm[v]));
}

template <typename R, int W, int U>
__device__ __forceinline__ void k1_vertex(const K1Args<R>& a, int g, int lane)
{
    if (a.vmat) k1_vertex_impl<R, W, U, true>(a, g, lane);
    else k1_vertex_impl<R, W, U, false>(a, g, lane);
}

// K1 with the local line search (protocol path, line_search=True)
template <typename R>
__global__ void __launch_bounds__(256) k1_color_pass_ls(const K1Args<R> a)
{
    const int g = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) / 4);
    if (g < a.count) k1_vertex_impl<R, 4, 1, false, true>(a, g, threadIdx.x & 3);
}

// One group of W lanes per vertex; lane j handles entries j, j+W, ... of its vertex and the
// group reduces f (3) and H (6) with a fixed xor-butterfly (bitwise deterministic).
template <typename R, int W, int U, int MINB, bool PF, bool UM>
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
                for (int pl = 0; pl < EntryPlanes<R>::P; ++pl) {
                    const void* src = reinterpret_cast<const char*>(a.ent) + 16 * (pl * a.E + e0);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes)
                                 : "memory");
                }
        }
    }
    if (g < a.count) k1_vertex_impl<R, W, U, UM>(a, g, lane);
}

// ---------------------------------------------------------------------------------------
// K1 (pipelined, fp32, range mode): persistent CTAs walk tiles of 256/W vertices of the
// colour range; every warp streams its lanes' entries (and, at a tile start, x / x_t of the
// lane's vertex) into shared memory with per-lane cp.async (LDGSTS) S-1 items ahead of the
// one it computes, so the entry latency leaves the dependency chain and only the neighbour
// gathers remain.  An item = one iteration of the warp: U entries per lane.  Each lane only
// reads its own shared-memory slots, so no barrier is needed between copy and use.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;  // src-size 0 -> zero fill, no global read
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int W, int U, int S>
struct PipeSmem {
    static constexpr int SLOTS = 3 * U + 2;  // U entries x 3 planes, then x and x_t
    float4 buf[8][S][SLOTS][32];
};

template <int W, int U, int S, bool UM>
__global__ void __launch_bounds__(256, 3) k1_color_pass_pipe(const K1Args<float> a, int ntiles)
{
    constexpr int VPB = 256 / W;   // vertices per tile
    constexpr int VPW = 32 / W;    // vertices per warp
    constexpr int SL = PipeSmem<W, U, S>::SLOTS;
    extern __shared__ float4 dyn_smem[];
    auto& sm = *reinterpret_cast<PipeSmem<W, U, S>*>(dyn_smem);
    const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
    const int lane = l32 & (W - 1), sub = l32 / W;
    const unsigned gmask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (l32 & ~(W - 1)));
    const long long E = a.E;
    const float4* __restrict__ ent = a.ent;

    // tile descriptor of this lane's vertex
    struct Desc {
        int v;        // vertex (colour-major id) or -1
        long long beg, end;
        int rounds;   // warp-uniform
    };
    auto describe = [&](int tile) {
        Desc d;
        const int g = tile * VPB + warp * VPW + sub;
        d.v = (tile < ntiles && g < a.count) ? a.vbeg + g : -1;
        d.beg = d.v >= 0 ? a.off[d.v] : 0;
        d.end = d.v >= 0 ? a.off[d.v + 1] : 0;
        int r = (int)((d.end - d.beg + W * U - 1) / (W * U));
        r = __reduce_max_sync(0xffffffffu, r);
        d.rounds = r < 1 ? 1 : r;
        return d;
    };
    auto issue = [&](const Desc& d, int it, int stage) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = d.beg + lane + (long long)(it * U + u) * W;
            const bool ok = d.v >= 0 && k < d.end;
            const long long ks = ok ? k : 0;
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                cp_async16(&sm.buf[warp][stage][pl * U + u][l32], ent + pl * E + ks, ok);
        }
        if (it == 0) {
            const int vv = d.v >= 0 ? d.v : 0;
            cp_async16(&sm.buf[warp][stage][3 * U][l32], a.pos + vv, d.v >= 0);
            cp_async16(&sm.buf[warp][stage][3 * U + 1][l32], a.xt + vv, d.v >= 0);
        }
        cp_async_commit();
    };

    int tile = blockIdx.x;
    if (tile >= ntiles) return;
    Desc cur = describe(tile);
    Desc nxt = describe(tile + gridDim.x);
    // prologue: items 0 .. S-2
    int itile = tile, iit = 0;     // issue cursor
    Desc icur = cur, inxt = nxt;
    int stage_issue = 0;
    for (int p = 0; p < S - 1; ++p) {
        if (itile < ntiles) issue(icur, iit, stage_issue);
        else cp_async_commit();
        stage_issue = (stage_issue + 1) % S;
        if (++iit == icur.rounds) {
            iit = 0;
            itile += gridDim.x;
            icur = inxt;
            inxt = describe(itile + gridDim.x);
        }
    }
    int it = 0, stage = 0;
    float xi[3] = {0.f, 0.f, 0.f}, dx[3] = {0.f, 0.f, 0.f};
    float f[3], H[6];
    Material<float> mv;
    while (tile < ntiles) {
        // issue the item S-1 ahead
        if (itile < ntiles) issue(icur, iit, stage_issue);
        else cp_async_commit();
        stage_issue = (stage_issue + 1) % S;
        if (++iit == icur.rounds) {
            iit = 0;
            itile += gridDim.x;
            icur = inxt;
            inxt = describe(itile + gridDim.x);
        }
        cp_async_wait<S - 1>();  // this lane's copies of the current item have landed
        if (it == 0) {
            const float4 x4 = sm.buf[warp][stage][3 * U][l32];
            const float4 t4 = sm.buf[warp][stage][3 * U + 1][l32];
            xi[0] = x4.x; xi[1] = x4.y; xi[2] = x4.z;
            dx[0] = x4.x - t4.x; dx[1] = x4.y - t4.y; dx[2] = x4.z - t4.z;
#pragma unroll
            for (int q = 0; q < 3; ++q) f[q] = 0.f;
#pragma unroll
            for (int q = 0; q < 6; ++q) H[q] = 0.f;
            if (UM && cur.v >= 0) mv = a.mat[a.vmat[cur.v]];
        }
        float4 pos[U][3];
        Entry<float> e[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long k = cur.beg + lane + (long long)(it * U + u) * W;
            ok[u] = cur.v >= 0 && k < cur.end;
            const float4 p0 = sm.buf[warp][stage][u][l32];
            const float4 p1 = sm.buf[warp][stage][U + u][l32];
            const float4 p2 = sm.buf[warp][stage][2 * U + u][l32];
            const unsigned u0 = __float_as_uint(p0.x), u1 = __float_as_uint(p0.y), u2 = __float_as_uint(p0.z);
            e[u].n[0] = (int)(u0 & VBD_ID_MASK);
            e[u].n[1] = (int)(u1 & VBD_ID_MASK);
            e[u].n[2] = (int)(u2 & VBD_ID_MASK);
            e[u].mat = (int)((u0 >> VBD_ID_BITS) | ((u1 >> VBD_ID_BITS) << 3) | ((u2 >> VBD_ID_BITS) << 6));
            e[u].w[0] = p0.w;
            e[u].w[1] = p1.x; e[u].w[2] = p1.y; e[u].w[3] = p1.z; e[u].w[4] = p1.w;
            e[u].w[5] = p2.x; e[u].w[6] = p2.y; e[u].w[7] = p2.z; e[u].w[8] = p2.w;
            if (ok[u]) {
                pos[u][0] = a.pos[e[u].n[0]];
                pos[u][1] = a.pos[e[u].n[1]];
                pos[u][2] = a.pos[e[u].n[2]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const float* w = e[u].w;
            const float dd = w[0] * (w[4] * w[8] - w[5] * w[7]) - w[1] * (w[3] * w[8] - w[5] * w[6]) +
                             w[2] * (w[3] * w[7] - w[4] * w[6]);
            const float V = __fdividef(1.0f / 6.0f, fabsf(dd));
            const float e0[3] = {pos[u][0].x - xi[0], pos[u][0].y - xi[1], pos[u][0].z - xi[2]};
            const float e1[3] = {pos[u][1].x - xi[0], pos[u][1].y - xi[1], pos[u][1].z - xi[2]};
            const float e2[3] = {pos[u][2].x - xi[0], pos[u][2].y - xi[1], pos[u][2].z - xi[2]};
            if (UM) {
                tet_contrib<float, false>(e0, e1, e2, w, V, mv, dx, f, H);
            } else {
                const Material<float> m = a.mat[e[u].mat];
                tet_contrib<float, true>(e0, e1, e2, w, V, m, dx, f, H);
            }
        }
        stage = (stage + 1) % S;
        if (++it < cur.rounds) continue;
        // vertex finished: group reduction, inertia, guarded solve, in-place write
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q) f[q] += __shfl_xor_sync(gmask, f[q], o, W);
#pragma unroll
            for (int q = 0; q < 6; ++q) H[q] += __shfl_xor_sync(gmask, H[q], o, W);
        }
        if (lane == 0 && cur.v >= 0) {
            const int v = cur.v;
            if (UM && cur.end > cur.beg) {
                const float hd0 = H[0] * dx[0] + H[1] * dx[1] + H[2] * dx[2];
                const float hd1 = H[1] * dx[0] + H[3] * dx[1] + H[4] * dx[2];
                const float hd2 = H[2] * dx[0] + H[4] * dx[1] + H[5] * dx[2];
                f[0] -= mv.dsc * hd0;
                f[1] -= mv.dsc * hd1;
                f[2] -= mv.dsc * hd2;
#pragma unroll
                for (int q = 0; q < 6; ++q) H[q] *= mv.opd;
            }
            const float4 y4 = a.y[v];
            const float mih2 = y4.w;
            f[0] += mih2 * (y4.x - xi[0]);
            f[1] += mih2 * (y4.y - xi[1]);
            f[2] += mih2 * (y4.z - xi[2]);
            H[0] += mih2;
            H[3] += mih2;
            H[5] += mih2;
            float d[3];
            block_solve<float>(f, H, a.eps_det, a.mode, d);
            const float4 nx = make_float4(xi[0] + d[0], xi[1] + d[1], xi[2] + d[2], 0.f);
            a.pos[v] = nx;
            if (a.flag && !finite3(nx.x, nx.y, nx.z))
                atomicMin(a.flag, StepFlag::key((unsigned)*a.stepctr, (unsigned)a.iter, (unsigned)a.perm[v]));
        }
        it = 0;
        tile += gridDim.x;
        cur = nxt;
        nxt = describe(tile + gridDim.x);
    }
    cp_async_wait<0>();
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
};

template <typename R>
__device__ __forceinline__ void k2_vertex(const StepArgs<R>& s, int i)
{
    typedef typename Vec4<R>::T R4;
    const R4 xt = s.xt[i], vt = s.vt[i];
    const R h = (R)s.h, hh = (R)s.hh;
    const R ax = (R)s.a[0], ay = (R)s.a[1], az = (R)s.a[2];
    R4 y;
    y.x = xt.x + h * vt.x + hh * ax;
    y.y = xt.y + h * vt.y + hh * ay;
    y.z = xt.z + h * vt.z + hh * az;
    y.w = s.mass[i] / hh;
    R4 x = xt;
    x.w = R(0);
    if (i < s.nfree_all) {
        if (s.init_mode == 1 || (s.init_mode == 3 && s.anorm == 0.0)) {
            x.x = xt.x + h * vt.x;
            x.y = xt.y + h * vt.y;
            x.z = xt.z + h * vt.z;
        } else if (s.init_mode == 2) {
            x.x = y.x; x.y = y.y; x.z = y.z;
        } else if (s.init_mode == 3) {
            const R4 vp = s.vprev[i];
            R atx = (vt.x - vp.x) / h, aty = (vt.y - vp.y) / h, atz = (vt.z - vp.z) / h;
            R comp = atx * (R)s.an[0] + aty * (R)s.an[1] + atz * (R)s.an[2];
            R at = comp / (R)s.anorm;
            at = at < R(0) ? R(0) : (at > R(1) ? R(1) : at);
            R sc = hh * at;
            x.x = xt.x + h * vt.x + sc * ax;
            x.y = xt.y + h * vt.y + sc * ay;
            x.z = xt.z + h * vt.z + sc * az;
        }
    } else if (s.flag && !finite3(x.x, x.y, x.z)) {  // fixed vertices never pass through K1
        atomicMin(s.flag, StepFlag::key((unsigned)*s.stepctr, 1u, (unsigned)s.perm[i]));
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

// K3: Chebyshev semi-iterative blend against the iterate two sweeps back, then copy the
// blended iterate into the history buffer that becomes x_prev1 (solver.py:221-232, 312-315),
// then the non-finite check of solver.py:282-288.
template <typename R>
__device__ __forceinline__ void k3_vertex(typename Vec4<R>::T* pos, typename Vec4<R>::T* hist,
                                          double omega, int blend, unsigned long long* flag,
                                          const int* perm, const int* stepctr, int iter, int i)
{
    typedef typename Vec4<R>::T R4;
    R4 x = pos[i];
    if (blend) {
        const R4 pp = hist[i];
        const R w = (R)omega;
        x.x = w * (x.x - pp.x) + pp.x;
        x.y = w * (x.y - pp.y) + pp.y;
        x.z = w * (x.z - pp.z) + pp.z;
        pos[i] = x;
    }
    hist[i] = x;
    if (flag && !finite3(x.x, x.y, x.z))
        atomicMin(flag, StepFlag::key((unsigned)*stepctr, (unsigned)iter, (unsigned)perm[i]));
}

template <typename R>
__global__ void k3_chebyshev(typename Vec4<R>::T* pos, typename Vec4<R>::T* hist, int n,
                             double omega, int blend, unsigned long long* flag,
                             const int* perm, const int* stepctr, int iter)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) k3_vertex<R>(pos, hist, omega, blend, flag, perm, stepctr, iter, i);
}

// K4: velocity commit (solver.py:319-323); skipped when the step reported a non-finite state.
template <typename R>
__device__ __forceinline__ void k4_vertex(typename Vec4<R>::T* pos, typename Vec4<R>::T* xt,
                                          typename Vec4<R>::T* vt, typename Vec4<R>::T* vprev,
                                          double h, int i)
{
    typedef typename Vec4<R>::T R4;
    const R4 x = pos[i], x0 = xt[i], v0 = vt[i];
    const R hr = (R)h;
    R4 v;
    v.x = (x.x - x0.x) / hr;
    v.y = (x.y - x0.y) / hr;
    v.z = (x.z - x0.z) / hr;
    v.w = R(0);
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

template <typename R>
__global__ void k_load_vec(const double* __restrict__ src, typename Vec4<R>::T* dst,
                           const int* __restrict__ perm, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long o = perm[i];
    typename Vec4<R>::T v;
    v.x = (R)src[3 * o];
    v.y = (R)src[3 * o + 1];
    v.z = (R)src[3 * o + 2];
    v.w = R(0);
    dst[i] = v;
}

template <typename R>
__global__ void k_store_vec(const typename Vec4<R>::T* __restrict__ src, double* dst,
                            const int* __restrict__ inv, int n)
{
    int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    typename Vec4<R>::T v = src[inv[o]];
    dst[3LL * o] = (double)v.x;
    dst[3LL * o + 1] = (double)v.y;
    dst[3LL * o + 2] = (double)v.z;
}

template <typename R>
__global__ void k_set_targets(const int* __restrict__ ids, const double* __restrict__ xyz, int n,
                              typename Vec4<R>::T* xt, typename Vec4<R>::T* pos)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    typename Vec4<R>::T v;
    v.x = (R)xyz[3 * k];
    v.y = (R)xyz[3 * k + 1];
    v.z = (R)xyz[3 * k + 2];
    v.w = R(0);
    xt[ids[k]] = v;
    pos[ids[k]] = v;
}

template <typename R>
__global__ void k_fill_mih2(typename Vec4<R>::T* y, const R* mass, int n, double hh)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i].w = mass[i] / (R)hh;
}

// halo exchange for slab-decomposed scenes: gather/scatter the positions of a vertex list
// Neighbour phase barrier over peer memory (slab P2P halo).  flags[0] of a context is
// written by its left neighbour, flags[1] by its right one; values are monotonically
// increasing phase stamps base + phase, base = phases of all previous steps (identical on
// every rank because every rank runs the same phase sequence).
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
