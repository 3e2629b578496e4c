// vbd_resident.cuh -- K1R: the whole time step of a SMALL scene in one launch, with the scene
// resident in shared memory (solver.py:291-324 for scenes whose colour passes are a few
// microseconds of work: launch latency, not bandwidth, bounds them on the per-colour graph).
//
// Every CTA owns, per colour, a contiguous run of 8-vertex groups (4 lanes per vertex) and
// keeps their entry slots {n0, n1, n2, kind} (int4, [round][lane] per group), x_t, y and the
// per-vertex sum V mu |w|^2 in shared memory for the whole step; the kind table is staged too.
// Between phases the CTAs synchronise with one barrier:
//   * REPL (one thread-block cluster, <= 16 CTAs): every CTA holds a REPLICA of all positions
//     in shared memory.  A colour pass reads neighbours from the local replica only and pushes
//     each new position into every CTA's replica through distributed shared memory
//     (st.shared::cluster), then barrier.cluster (release / acquire) ends the pass.  No global
//     memory is touched between K2 and K4.
//   * GLOB (one CTA per SM, co-resident by cooperative launch): positions stay in global memory
//     (L2-resident at these sizes, read with ld.global.cg) and a sense-reversing grid barrier
//     on a global {count, generation} pair ends each phase.
// The per-vertex arithmetic is the K1 one (tet_contrib_ec[_xy], vertex_terms, block_solve) with
// 4 lanes per vertex and the same lane partial sums and butterfly as the 4-lane K1 variants,
// and K2 / K3 / K4 run the same vertex bodies: results are bitwise equal to the graph path.
#pragma once
#include <cooperative_groups.h>

#include "vbd_kernels.cuh"

#define VBD_RES_THREADS 512  // 16 warps: 16 groups of 8 vertices in flight per CTA
#define VBD_RES_U 2          // entries per lane in flight per sweep iteration (rounds padded to it; 4 at 384 threads measured slower: 2.81 vs 2.50 us per C1 pass)
#define VBD_RES_MAX_COLORS 16

struct ResGroup {
    int v0, nv;  // first colour-major vertex, vertices (<= 8)
    int sbase;   // first slot (int4) of the group in the CTA's slot array
    int rounds;  // slot rounds (even); slot (i, lane) = sbase + 32 i + lane
};

template <typename R> struct ResArgs {
    K1Args<R> a;    // kinds, vsv, eps_det, mode, flag (K1 check when rho == 0), perm, stepctr
    StepArgs<R> s;  // K2 / K3 / K4 state
    const int4* slots;          // all CTAs' slots, CTA k at slot_beg[k]
    const long long* slot_beg;  // (ncta + 1)
    const ResGroup* groups;     // all CTAs' groups, CTA k at grp_beg[k]
    const int* grp_beg;         // (ncta + 1)
    const int* col_grp;         // per CTA: (ncolors + 1) group offsets (relative to grp_beg[k])
    int ncolors, n_max, cheb;
    const double* omegas;       // (n_max + 1), device
    int nkinds;
    int slot_cap, grp_cap;      // max slots / groups of one CTA (shared memory sizing)
    unsigned* bar;              // GLOB: {count, generation}
    int ncta;
    const unsigned short* push; // REPL: per vertex, the CTAs whose replica must see its updates
                                // (owners of its neighbours, its own CTA, its K3 / K4 chunk CTA)
    int dbg;                    // timing experiments only (VBD_RES_DBG, wrong results): 1 no DSMEM
                                // pushes, 2 no entry sweep, 3 neither; 8: CTA 0's pass timeline
                                // (clock64, results unchanged) into prof
    long long* prof;            // dbg & 8: per pass {start, last sweep end, last push end, barrier exit,
                                // longest single group's sweep end -> push end}
};

// shared memory of one CTA (bytes; every region 16-byte aligned)
template <typename R> struct ResSmem {
    typedef typename Vec4<R>::T R4;
    int nk, n, slot_cap, grp_cap, ncolors;
    bool repl;
    // kind records, then (fp32, displacement state) the kinds' rest edges, 3 float4 each
    __host__ __device__ size_t recs_bytes() const { return ((size_t)(nk + 1) * KindRec<R>::HOT * sizeof(R) + 15) & ~(size_t)15; }
    __host__ __device__ size_t kinds_bytes() const { return recs_bytes() + (sizeof(R) == 4 ? (size_t)(nk + 1) * 48 : 0); }
    __host__ __device__ size_t off_rep() const { return kinds_bytes(); }
    __host__ __device__ size_t off_slots() const { return off_rep() + (repl ? (size_t)(n + 1) * sizeof(R4) : 0); }
    __host__ __device__ size_t off_xt() const { return off_slots() + (size_t)slot_cap * 16; }
    __host__ __device__ size_t off_y() const { return off_xt() + (size_t)grp_cap * 8 * sizeof(R4); }
    __host__ __device__ size_t off_sv() const { return off_y() + (size_t)grp_cap * 8 * sizeof(R4); }
    __host__ __device__ size_t off_grp() const { return (off_sv() + (size_t)grp_cap * 8 * sizeof(R) + 15) & ~(size_t)15; }
    __host__ __device__ size_t off_cg() const { return off_grp() + (size_t)grp_cap * sizeof(ResGroup); }
    __host__ __device__ size_t total() const { return off_cg() + (size_t)(ncolors + 1) * 4; }
};

__device__ __forceinline__ float4 ldcg4(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ double4 ldcg4(const double4* p)
{
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p)), b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void stcg4(float4* p, float4 v) { __stcg(p, v); }
__device__ __forceinline__ void stcg4(double4* p, double4 v)
{
    __stcg(reinterpret_cast<double2*>(p), make_double2(v.x, v.y));
    __stcg(reinterpret_cast<double2*>(p) + 1, make_double2(v.z, v.w));
}

// sense-reversing grid barrier (GLOB): the last arriver resets the count and publishes a new
// generation (release); the others spin on it (acquire).  bar.sync orders the CTA around it.
__device__ __forceinline__ void res_grid_barrier(unsigned* bar, unsigned ncta)
{
    // one monotonic 64-bit arrival counter (a multiple of ncta between barriers): each CTA adds
    // 1 (release) and polls (acquire) until the count reaches the next multiple -- one atomic
    // round trip per CTA, no generation word and no reset store
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* c = reinterpret_cast<unsigned long long*>(bar);
        unsigned long long old;
        asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
        const unsigned long long target = (old / ncta + 1) * ncta;
        unsigned long long cur = old + 1;
        while (cur < target) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(c) : "memory");
    }
    __syncthreads();
}

template <typename R, bool UM, bool REPL>
__global__ void __launch_bounds__(VBD_RES_THREADS, 1) k_step_resident(const ResArgs<R> ra)
{
    namespace cg = cooperative_groups;
    typedef typename Vec4<R>::T R4;
    typedef typename PlaneT<R>::T PL;
    constexpr int HOT = KindRec<R>::HOT, QH = KindRec<R>::QH, Q = KindRec<R>::Q;
    constexpr int QS = UM ? 8 * (int)sizeof(R) / 16 : QH;  // chunks the entry loop reads
    constexpr bool PACK = sizeof(R) == 4 && UM;
    extern __shared__ __align__(128) unsigned char smem[];
    const K1Args<R>& a = ra.a;
    const StepArgs<R>& s = ra.s;
    const int cta = REPL ? (int)cg::this_cluster().block_rank() : (int)blockIdx.x;
    const int ncta = ra.ncta;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int NW = VBD_RES_THREADS / 32;
    const int n = s.n;
    const ResSmem<R> L{ra.nkinds, n, ra.slot_cap, ra.grp_cap, ra.ncolors, REPL};
    PL* skind = reinterpret_cast<PL*>(smem);
    R4* rep = reinterpret_cast<R4*>(smem + L.off_rep());
    int4* sslot = reinterpret_cast<int4*>(smem + L.off_slots());
    R4* sxt = reinterpret_cast<R4*>(smem + L.off_xt());
    R4* sy = reinterpret_cast<R4*>(smem + L.off_y());
    R* ssv = reinterpret_cast<R*>(smem + L.off_sv());
    ResGroup* sgrp = reinterpret_cast<ResGroup*>(smem + L.off_grp());
    int* scg = reinterpret_cast<int*>(smem + L.off_cg());

    auto barrier = [&]() {
        if constexpr (REPL) cg::this_cluster().sync();
        else res_grid_barrier(ra.bar, (unsigned)ncta);
    };
    auto xget = [&](int i) -> R4 {  // current position of vertex i (any CTA's latest write)
        if constexpr (REPL) return rep[i];
        else return ldcg4(s.pos + i);
    };

    // ---- step constants into shared memory
    for (int i = tid; i < ra.nkinds * QH; i += blockDim.x) skind[i] = a.kinds[(i / QH) * Q + i % QH];
    for (int i = tid; i < QH; i += blockDim.x) skind[ra.nkinds * QH + i] = PL{};  // padding: zero record
    constexpr bool DISP = sizeof(R) == 4;  // fp32: displacement state, rest edges per kind
    float4* sedge = reinterpret_cast<float4*>(smem + L.recs_bytes());
    if constexpr (DISP) {
        for (int i = tid; i < ra.nkinds * 3; i += blockDim.x) sedge[i] = a.kedge[i];
        for (int i = tid; i < 3; i += blockDim.x) sedge[ra.nkinds * 3 + i] = float4{};
    }
    const long long sb0 = ra.slot_beg[cta], ns = ra.slot_beg[cta + 1] - sb0;
    for (long long i = tid; i < ns; i += blockDim.x) sslot[i] = ra.slots[sb0 + i];
    const int gb0 = ra.grp_beg[cta], ng = ra.grp_beg[cta + 1] - gb0;
    for (int i = tid; i < ng; i += blockDim.x) sgrp[i] = ra.groups[gb0 + i];
    for (int i = tid; i <= ra.ncolors; i += blockDim.x) scg[i] = ra.col_grp[cta * (ra.ncolors + 1) + i];

    // push a new position of vertex v into the replicas of the CTAs in m (DSMEM stores); a
    // colour pass ends with barrier.cluster (release / acquire)
    auto push_to = [&](unsigned m, int v, const R4& x) {
        const unsigned la = smem_u32(rep + v);
        while (m) {
            const int r = __ffs(m) - 1;
            m &= m - 1;
            unsigned ca;  // the rank's copy of this address (mapa), stored with st.shared::cluster
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ca) : "r"(la), "r"(r));
            if constexpr (sizeof(R) == 4) {
                asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ca), "f"((float)x.x),
                             "f"((float)x.y), "f"((float)x.z), "f"((float)x.w)
                             : "memory");
            } else {
                asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ca), "d"((double)x.x),
                             "d"((double)x.y)
                             : "memory");
                asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ca + 16), "d"((double)x.z),
                             "d"((double)x.w)
                             : "memory");
            }
        }
    };

    // ---- K2 over this CTA's elementwise chunk
    const int lo = (int)((long long)n * cta / ncta), hi = (int)((long long)n * (cta + 1) / ncta);
    for (int i = lo + tid; i < hi; i += blockDim.x) k2_vertex<R>(s, i);
    barrier();
    // owned per-vertex state; REPL: the replica (+ a zero position for padding slots)
    for (int k = tid; k < ng * 8; k += blockDim.x) {
        const ResGroup g = sgrp[k >> 3];
        const int vi = k & 7;
        const int v = g.v0 + (vi < g.nv ? vi : 0);
        sxt[k] = ldcg4(s.xt + v);
        sy[k] = ldcg4(s.y + v);
        ssv[k] = UM ? a.vsv[v] : R(0);
    }
    if constexpr (REPL) {
        for (int i = tid; i < n; i += blockDim.x) rep[i] = ldcg4(s.pos + i);
        if (tid == 0) rep[n] = R4{};
    }
    __syncthreads();

    const unsigned kb = smem_u32(skind);
    const int vi = lane & 7, j = lane >> 3;  // lane = 8 j + vi serves entry positions j, j + 4, ...
    const R4 zero4{};
    __shared__ unsigned long long prof_t[3];
    const bool prof = (ra.dbg & 8) && cta == 0 && ra.prof;
    int pass = 0;
    for (int it = 1; it <= ra.n_max; ++it) {
        for (int c = 0; c < ra.ncolors; ++c) {
            if (prof && tid == 0) {
                prof_t[0] = prof_t[1] = prof_t[2] = 0;
                ra.prof[5 * pass] = (long long)clock64();
            }
            if (prof) __syncthreads();
            for (int gi = scg[c] + warp; gi < scg[c + 1]; gi += NW) {
                const ResGroup g = sgrp[gi];
                const bool act = vi < g.nv;
                const int v = g.v0 + (act ? vi : 0);
                const int k = gi * 8 + vi;
                const R4 xi4 = xget(v), xt4 = sxt[k], y4 = sy[k];
                // the vertex's push set, loaded before the sweep (its latency off the critical path)
                const unsigned pmask = REPL ? (unsigned)__ldg(ra.push + v) : 0u;
                const R xi[3] = {xi4.x, xi4.y, xi4.z};
                const R dx[3] = {xi[0] - xt4.x, xi[1] - xt4.y, xi[2] - xt4.z};
                R f[3] = {R(0), R(0), R(0)}, H[6] = {R(0), R(0), R(0), R(0), R(0), R(0)}, sv = R(0);
                AccXY acc;
                acc.zero();
                const float2 nxy = make_float2(-(float)xi[0], -(float)xi[1]);
                const float nz = -(float)xi[2];
                const int4* sl = sslot + g.sbase + lane;
                auto pos_of = [&](int id) -> R4 {
                    if constexpr (REPL) return rep[id];
                    else {
                        const R4 p = ldcg4(s.pos + (id < n ? id : 0));
                        return id < n ? p : zero4;
                    }
                };
                const int grounds = (ra.dbg & 2) ? 0 : g.rounds;
                for (int i0 = 0; i0 < grounds; i0 += VBD_RES_U) {
                    int4 e[VBD_RES_U];
                    R4 p[VBD_RES_U][3];
#pragma unroll
                    for (int u = 0; u < VBD_RES_U; ++u) {
                        e[u] = sl[32 * (i0 + u)];
                        p[u][0] = pos_of(e[u].x);
                        p[u][1] = pos_of(e[u].y);
                        p[u][2] = pos_of(e[u].z);
                    }
#pragma unroll
                    for (int u = 0; u < VBD_RES_U; ++u) {
                        R r[HOT];
                        const unsigned rp = kb + (unsigned)e[u].w * (unsigned)(HOT * sizeof(R));
                        float4 ex[3];
                        if constexpr (DISP) {
#pragma unroll
                            for (int q = 0; q < 3; ++q) ex[q] = sedge[3 * e[u].w + q];
                        }
#pragma unroll
                        for (int q = 0; q < QS; ++q) {
                            PL w;
                            lds_v(rp + 16u * q, w);
                            const R* wr = reinterpret_cast<const R*>(&w);
#pragma unroll
                            for (int z = 0; z < 16 / (int)sizeof(R); ++z) r[q * (16 / (int)sizeof(R)) + z] = wr[z];
                        }
                        if constexpr (PACK) {
                            tet_contrib_ec_xy(p[u][0], p[u][1], p[u][2], nxy, nz, ex[0], ex[1], ex[2],
                                              reinterpret_cast<const float*>(r), acc);
                        } else {
                            R e0[3], e1[3], e2[3];
                            edge3<R>(p[u][0], xi, ex[0], DISP, e0);
                            edge3<R>(p[u][1], xi, ex[1], DISP, e1);
                            edge3<R>(p[u][2], xi, ex[2], DISP, e2);
                            tet_contrib_ec<R, !UM>(e0, e1, e2, r, UM ? R(0) : r[9], UM ? R(1) : r[10], dx, f, H, sv);
                        }
                    }
                }
                if constexpr (PACK) {
                    f[0] = acc.f01.x;
                    f[1] = acc.f01.y;
                    f[2] = acc.f2;
                    H[0] = acc.h03.x;
                    H[1] = acc.h1;
                    H[2] = acc.h24.x;
                    H[3] = acc.h03.y;
                    H[4] = acc.h24.y;
                    H[5] = acc.h5;
                }
                R dsc = R(0), opd = R(1);
                if (UM && g.rounds > 0) {  // the record of this lane's round-0 slot (lane j = 0: entry 0)
                    const unsigned rp = kb + (unsigned)sl[0].w * (unsigned)(HOT * sizeof(R));
                    R r[HOT];
#pragma unroll
                    for (int q = 0; q < QH; ++q) {
                        PL w;
                        lds_v(rp + 16u * q, w);
                        const R* wr = reinterpret_cast<const R*>(&w);
#pragma unroll
                        for (int z = 0; z < 16 / (int)sizeof(R); ++z) r[q * (16 / (int)sizeof(R)) + z] = wr[z];
                    }
                    dsc = r[9];
                    opd = r[10];
                }
                const unsigned long long t_sw = prof ? (unsigned long long)clock64() : 0ull;
                if (prof && lane == 0) atomicMax(&prof_t[0], t_sw);
                // the 4 lanes of a vertex are vi + 8 j: butterfly j ^ 2, then j ^ 1 (4-lane K1 order)
#pragma unroll
                for (int o = 16; o >= 8; o >>= 1) {
#pragma unroll
                    for (int q = 0; q < 3; ++q) f[q] += __shfl_xor_sync(0xffffffffu, f[q], o);
#pragma unroll
                    for (int q = 0; q < 6; ++q) H[q] += __shfl_xor_sync(0xffffffffu, H[q], o);
                }
                R4 nx = xi4;
                if (j == 0) {
                    if (UM) {
                        H[0] = H[0] + ssv[k];
                        H[3] = H[3] + ssv[k];
                        H[5] = H[5] + ssv[k];
                    }
                    vertex_terms<R>(f, H, dx, xi, y4.x, y4.y, y4.z, y4.w, UM, dsc, opd);
                    R d[3];
                    block_solve<R>(f, H, a.eps_det, a.mode, d);
                    nx.x = xi[0] + d[0];
                    nx.y = xi[1] + d[1];
                    nx.z = xi[2] + d[2];
                    if (act && a.flag && !finite3(nx.x, nx.y, nx.z))
                        atomicMin(a.flag, StepFlag::key((unsigned)*a.stepctr, (unsigned)it, (unsigned)a.perm[v]));
                }
                nx.x = __shfl_sync(0xffffffffu, nx.x, vi);
                nx.y = __shfl_sync(0xffffffffu, nx.y, vi);
                nx.z = __shfl_sync(0xffffffffu, nx.z, vi);
                if constexpr (REPL) __syncwarp();  // inactive lanes read x of the group's first vertex
                if (act) {
                    if constexpr (REPL) {  // lane j pushes to every 4th CTA of the reader set
                        push_to((ra.dbg & 1) ? 0u : pmask & (0x1111u << j), v, nx);
                    } else if (j == 0) {
                        stcg4(s.pos + v, nx);
                    }
                }
                if (prof) {
                    __syncwarp();
                    if (lane == 0) atomicMax(&prof_t[2], (unsigned long long)clock64() - t_sw);
                }
            }
            // K3 of this iteration (after its last colour pass): the history copy and the
            // finite check of the chunk; with a blend it is a pass of its own
            R4* hist = (it % 2 == 1) ? s.hb : s.ha;
            const double w = ra.cheb ? ra.omegas[it] : 1.0;
            const bool blend = ra.cheb && it >= 2 && w != 1.0;
            auto k3_copy = [&]() {
                for (int i = lo + tid; i < hi; i += blockDim.x) {
                    const R4 x = xget(i);
                    hist[i] = x;
                    if (s.flag && !finite3(x.x, x.y, x.z))
                        atomicMin(s.flag, StepFlag::key((unsigned)*s.stepctr, (unsigned)it, (unsigned)s.perm[i]));
                }
            };
            const bool copy_here = ra.cheb && !blend && c == ra.ncolors - 1;
            if (prof && lane == 0) atomicMax(&prof_t[1], (unsigned long long)clock64());
            barrier();
            if (prof && tid == 0) {
                ra.prof[5 * pass + 1] = (long long)prof_t[0];
                ra.prof[5 * pass + 2] = (long long)prof_t[1];
                ra.prof[5 * pass + 3] = (long long)clock64();
                ra.prof[5 * pass + 4] = (long long)prof_t[2];
            }
            ++pass;
            if (copy_here) {
                k3_copy();
                barrier();
            }
            if (blend && c == ra.ncolors - 1) {  // K3 blend pass over the elementwise chunk
                for (int i = lo + tid; i < hi; i += blockDim.x) {
                    R4 x = k3_blend<R>(xget(i), hist[i], w);
                    if constexpr (REPL) push_to(ra.push[i], i, x);
                    else stcg4(s.pos + i, x);
                    hist[i] = x;
                    if (s.flag && !finite3(x.x, x.y, x.z))
                        atomicMin(s.flag, StepFlag::key((unsigned)*s.stepctr, (unsigned)it, (unsigned)s.perm[i]));
                }
                barrier();
            }
        }
    }
    if constexpr (REPL) cg::this_cluster().sync();  // every flag report and remote store settled
    // ---- K4 (the final iterate is stored either way; the commit only without a non-finite report)
    const bool ok = !s.flag || *reinterpret_cast<volatile unsigned long long*>(s.flag) == StepFlag::NONE;
    for (int i = lo + tid; i < hi; i += blockDim.x) {
        const R4 x = xget(i);
        if constexpr (REPL) s.pos[i] = x;
        if (ok) {
            const R4 x0 = s.xt[i], v0 = s.vt[i];
            s.vprev[i] = v0;
            s.vt[i] = k4_velocity<R>(x, x0, s.h);
            s.xt[i] = x;
        }
    }
    if (cta == 0 && tid == 0) atomicAdd(s.stepctr, 1);
}
