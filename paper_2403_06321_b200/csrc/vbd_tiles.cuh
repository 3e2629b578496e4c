// vbd_tiles.cuh -- K1T: the colour pass as a warp-specialised, TMA-fed tile pipeline.
//
// A colour range is cut into tiles of 256 / W consecutive vertices (Morton-compact in space;
// W = lanes per vertex, 8 consumer warps per tile).  Each tile carries, built once at pack time:
//   * its sorted list of distinct neighbour vertices (the other-colour positions it reads),
//   * its entries re-encoded against that list: 8 bytes of shared-memory byte offsets
//     {u16 n0, u16 n1, u16 n2, u16 kind}, laid out per consumer warp as [round i][lane] slots:
//     lane = (32 / W) j + vi serves entry position W i + j of the warp's vertex vi.  Rounds are
//     padded to even counts; padding slots point at a zero position and a zero kind record,
//     whose contribution is exactly +0, so the sweep has no validity branches.  A warp's
//     slot reads are contiguous, and the 8 lanes of a quarter-warp (same position, 8 vertices
//     of one class) read the same kind record: shared-memory broadcast.
// K1T is persistent: per CTA one producer warp and 8 consumer warps (W lanes per vertex).
// The producer fills a ring of shared-memory stages for tile t + grid: one elected lane
// issues cp.async.bulk (TMA) copies of the tile's entry range and of x / x_t / y of its 64
// vertices, all 32 lanes gather the neighbour positions (and CSR offsets) with cp.async,
// and the stage's mbarrier completes on the byte count + the 32 cp.async arrivals.  The
// consumers wait on the mbarrier, sweep their vertices with shared-memory loads only
// (entries, neighbour positions, kind records), solve, store x in place, and release the
// stage.  The arithmetic is tet_contrib_core / vertex_terms / block_solve: bitwise equal to
// every other K1 variant.
#pragma once
#include "vbd_kernels.cuh"
#include "vbd_grid_classes.cuh"

#define VBD_TILE_SORT 32768  // max neighbour references (3 per entry) per tile for the build

// ---------------------------------------------------------------------------------------
// build: one CTA (256 threads) per tile.  FILL = false: count distinct neighbours;
// FILL = true: write the sorted list at loff[t] and the 8-byte tile entries.

#define VBD_TILE_U 2  // rounds per consumer loop iteration (slot counts padded to it)

// rounds (entry slots per lane) of consumer warp w of a tile: max over its 32 / W vertices
// of ceil(degree / W)
__device__ __forceinline__ int tile_warp_rounds(const long long* __restrict__ eoff, int v0, int nv, int w, int W)
{
    const int vpw = 32 / W;
    int r = 0;
    for (int vi = 0; vi < vpw; ++vi) {
        const int lv = vpw * w + vi;
        if (lv >= nv) break;
        const int d = (int)(eoff[v0 + lv + 1] - eoff[v0 + lv]);
        r = max(r, (d + W - 1) / W);
    }
    return (r + VBD_TILE_U - 1) / VBD_TILE_U * VBD_TILE_U;
}

// build: one CTA (256 threads) per tile.  FILL = false: count distinct neighbours (cnt[2t])
// and entry slots (cnt[2t+1]); FILL = true: write the sorted neighbour list at lbase[t] and
// the slots at sbase[t].
template <bool FILL>
__global__ void __launch_bounds__(256) k_tile_nbrs(const int* __restrict__ tv0, const int* __restrict__ tnv,
                                                   const long long* __restrict__ eoff,
                                                   const int4* __restrict__ cent, long long* cnt,
                                                   const long long* __restrict__ lbase,
                                                   const long long* __restrict__ sbase, int* __restrict__ tnbr,
                                                   uint2* __restrict__ tent, int W, unsigned r4b,
                                                   unsigned pad_pos, unsigned kstride, unsigned pad_kind, int* err,
                                                   long long* __restrict__ slot_entry = nullptr,
                                                   const signed char* __restrict__ tw = nullptr)
{
    extern __shared__ int keys[];  // next power of two >= max references per tile
    __shared__ int part[257];
    __shared__ int wslot[9];
    const int t = blockIdx.x, tid = threadIdx.x;
    if (tw) W = tw[t];  // class tiles: one lane per vertex
    const int v0 = tv0[t], nv = tnv[t];
    const long long e0 = eoff[v0], e1 = eoff[v0 + nv];
    const int nref = (int)(3 * (e1 - e0));
    if (nref > VBD_TILE_SORT) {
        if (tid == 0) atomicExch(err, 1);
        return;
    }
    if (tid == 0) {
        int sb = 0;
        for (int w = 0; w < 8; ++w) {
            wslot[w] = sb;
            sb += 32 * tile_warp_rounds(eoff, v0, nv, w, W);
        }
        wslot[8] = sb;
    }
    int P = 256;
    while (P < nref) P <<= 1;
    for (int i = tid; i < P; i += 256) {
        int k = 0x7fffffff;
        if (i < nref) {
            const int4 e = cent[e0 + i / 3];
            const int r = i % 3;
            k = r == 0 ? e.x : (r == 1 ? e.y : e.z);
        }
        keys[i] = k;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P; i += 256) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    // distinct keys: chunked count + serial scan of the 256 partial counts
    const int chunk = P / 256;
    const int i0 = tid * chunk;
    int c = 0;
    for (int i = i0; i < i0 + chunk; ++i)
        if (i < nref && (i == 0 || keys[i] != keys[i - 1])) ++c;
    part[tid] = c;
    __syncthreads();
    if (tid == 0) {
        int s = 0;
        for (int i = 0; i < 256; ++i) {
            const int x = part[i];
            part[i] = s;
            s += x;
        }
        part[256] = s;
    }
    __syncthreads();
    const int nl = part[256];
    if (!FILL) {
        if (tid == 0) {
            cnt[2 * t] = nl;
            cnt[2 * t + 1] = wslot[8];
        }
        return;
    }
    const long long l0 = lbase[t];
    int o = part[tid];
    for (int i = i0; i < i0 + chunk; ++i)
        if (i < nref && (i == 0 || keys[i] != keys[i - 1])) tnbr[l0 + o++] = keys[i];
    __syncthreads();  // the list is visible to the whole CTA (global writes, bar.sync)
    const int* lst = tnbr + l0;
    const long long s0 = sbase[t];
    for (int sl = tid; sl < wslot[8]; sl += 256) {
        int w = 0;
        while (sl >= wslot[w + 1]) ++w;
        const int rel = sl - wslot[w];
        const int lane = rel & 31, i = rel >> 5;
        const int vpw = 32 / W;
        const int lv = vpw * w + lane % vpw, pos = W * i + lane / vpw;
        uint2 out = make_uint2(pad_pos | (pad_pos << 16), pad_pos | (pad_kind << 16));
        long long ent = -1;
        if (lv < nv) {
            const long long k = eoff[v0 + lv] + pos;
            if (k < eoff[v0 + lv + 1]) {
                ent = k;
                const int4 e = cent[k];
                unsigned loc[3];
                const int ids[3] = {e.x, e.y, e.z};
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    int lo = 0, hi = nl - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (lst[mid] < ids[r]) lo = mid + 1;
                        else hi = mid;
                    }
                    loc[r] = (unsigned)lo * r4b;  // byte offset into the stage's positions
                }
                out = make_uint2(loc[0] | (loc[1] << 16), loc[2] | (((unsigned)e.w * kstride) << 16));
            }
        }
        tent[s0 + sl] = out;
        if (slot_entry) slot_entry[s0 + sl] = ent;
    }
}

// K1T class tiles: the tile build's input for a grid-class vertex (vtpl >= 0) is R = ceil(NL / 3)
// pseudo entries {loc[3r], loc[3r + 1], loc[3r + 2], pad kind} -- its NL distinct neighbours in
// the class's local order (vbd_grid_classes.cuh), so the slots a lane reads are the shared-memory
// offsets of its neighbours (bank-placed like any slot); other vertices keep their entries.
// err: 1 a vertex does not match its class, 2 its kinds differ from its instance's records.
__global__ void k_class_pseudo(const long long* __restrict__ eoff, const int4* __restrict__ cent, long long nsolve,
                               const signed char* __restrict__ vtpl, const signed char* __restrict__ vins,
                               const long long* __restrict__ eoff2, int4* __restrict__ cent2,
                               const int* __restrict__ irec, const int* __restrict__ ckind, int pad_kind,
                               int* __restrict__ err)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nsolve) return;
    const long long k0 = eoff[i], o = eoff2[i];
    const int d = (int)(eoff[i + 1] - k0), tpl = vtpl[i];
    if (tpl < 0) {
        for (int q = 0; q < d; ++q) cent2[o + q] = cent[k0 + q];
        return;
    }
    const int b = vbd_gc_beg[tpl], ne = vbd_gc_beg[tpl + 1] - b, nl = vbd_gc_nl[tpl];
    if (d != ne) {
        atomicExch(err, 1);
        return;
    }
    int loc[VBD_GC_MAXNL];
    for (int q = 0; q < VBD_GC_MAXNL; ++q) loc[q] = -1;
    const int* kr = ckind + irec[vins[i]];
    for (int q = 0; q < ne; ++q) {
        const int4 e = cent[k0 + q];
        const int ids[3] = {e.x, e.y, e.z};
        for (int r = 0; r < 3; ++r) {
            const int li = vbd_gc_nbr[3 * (b + q) + r];
            if (loc[li] < 0) loc[li] = ids[r];
            else if (loc[li] != ids[r]) atomicExch(err, 1);
        }
        if (e.w != kr[q]) atomicExch(err, 2);
    }
    for (int r = 0; 3 * r < nl; ++r) {
        const int a = loc[3 * r];
        cent2[o + r] = make_int4(a, 3 * r + 1 < nl ? loc[3 * r + 1] : a, 3 * r + 2 < nl ? loc[3 * r + 2] : a, pad_kind);
    }
}

// class tiles: the tile build's degree of every solved vertex (pseudo rows for class vertices)
__global__ void k_class_deg(const long long* __restrict__ eoff, const signed char* __restrict__ vtpl, long long n,
                            long long* __restrict__ deg)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = vtpl[i];
    deg[i] = t < 0 ? eoff[i + 1] - eoff[i] : (long long)((vbd_gc_nl[t] + 2) / 3);
}

// K1T-X: {n0, n1, n2, 0} of every explicit fp32 entry (ids without the material bits)
__global__ void k_plane_ids(const float4* __restrict__ planes, long long E, int4* __restrict__ out)
{
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= E) return;
    const float4 a = planes[k];
    out[k] = make_int4((int)(__float_as_uint(a.x) & VBD_ID_MASK), (int)(__float_as_uint(a.y) & VBD_ID_MASK),
                       (int)(__float_as_uint(a.z) & VBD_ID_MASK), 0);
}

// K1T-X: the 9 slot-weight rows of every slot's entry, plane q at rows + q * S (padding: 0)
__global__ void k_slot_rows(const long long* __restrict__ slot_entry, long long S, const float4* __restrict__ planes,
                            long long E, float* __restrict__ rows)
{
    const long long sl = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (sl >= S) return;
    const long long k = slot_entry[sl];
    float w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (k >= 0) {
        const Entry<float> e = Entry<float>::load(planes, E, k);
        for (int q = 0; q < 9; ++q) w[q] = e.w[q];
    }
    for (int q = 0; q < 9; ++q) rows[q * S + sl] = w[q];
}

// Bank-aware placement of a tile's neighbour positions (one thread per tile, after FILL).
// A consumer LDS.128 is served per quarter-warp: its 8 lanes (8 vertices, same entry
// position, same tet corner k) take one wavefront only if their positions lie in 8 distinct
// 16-byte bank groups (slot index mod 8) or coincide.  The sorted list leaves that to chance
// (~2.1 wavefronts per quarter measured on C5).  Here every quarter-warp group, in sweep
// order, places its not-yet-placed neighbours into bank groups its placed members do not
// use, least-filled first, inside a list padded to nlp = 8 * (slots per bank); then each bank
// group is filled in sorted-id order.  The list is rewritten in position order (-1 = hole,
// skipped by the producer) and the slots' offsets remapped; positions only move in shared
// memory, so results are bitwise unchanged.
__global__ void k_tile_banks(const int* __restrict__ tv0, const int* __restrict__ tnv,
                             const long long* __restrict__ eoff, const long long* __restrict__ lbase,
                             const long long* __restrict__ sbase, const int* __restrict__ nls, int nt, int W,
                             unsigned r4b, unsigned pad_pos, int* __restrict__ tnbr, uint2* __restrict__ tent,
                             int* __restrict__ ids, int* __restrict__ asg, int given,
                             const signed char* __restrict__ tw = nullptr)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    if (tw) W = tw[t];
    const long long l0 = lbase[t], s0 = sbase[t];
    const int nl = nls[t], nlp = (int)(lbase[t + 1] - l0), cap = nlp / 8;
    const int pad_bank = (int)((pad_pos / r4b) & 7u);
    for (int u = 0; u < nl; ++u) {
        ids[l0 + u] = tnbr[l0 + u];
        if (!given) asg[l0 + u] = -1;
    }
    int fill[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int v0 = tv0[t], nv = tnv[t];
    long long slot = given ? sbase[t + 1] : s0;  // given: banks from k_tile_banks_dsatur
    for (int w = 0; w < 8 && !given; ++w) {
        const int rounds = tile_warp_rounds(eoff, v0, nv, w, W);
        for (int i = 0; i < rounds; ++i, slot += 32) {
            uint2 e[32];
            for (int l = 0; l < 32; ++l) e[l] = tent[slot + l];
            for (int k = 0; k < 3; ++k)
                for (int q = 0; q < 32; q += 8) {  // one quarter-warp group (8 lanes)
                    int u[8];
                    unsigned used = 0;
                    for (int l = 0; l < 8; ++l) {
                        const uint2 s = e[q + l];
                        const unsigned off = (k == 0 ? s.x : k == 1 ? s.x >> 16 : s.y) & 0xffffu;
                        u[l] = off == pad_pos ? -2 : (int)(off / r4b);
                        if (u[l] == -2) used |= 1u << pad_bank;
                        else if (asg[l0 + u[l]] >= 0) used |= 1u << asg[l0 + u[l]];
                    }
                    for (int l = 0; l < 8; ++l) {
                        if (u[l] < 0 || asg[l0 + u[l]] >= 0) continue;
                        int best = -1;
                        for (int b = 0; b < 8; ++b)  // a free bank group the group does not use yet
                            if (!(used >> b & 1u) && fill[b] < cap && (best < 0 || fill[b] < fill[best])) best = b;
                        if (best < 0)
                            for (int b = 0; b < 8; ++b)  // none: least-filled (a conflict)
                                if (fill[b] < cap && (best < 0 || fill[b] < fill[best])) best = b;
                        asg[l0 + u[l]] = best;
                        ++fill[best];
                        used |= 1u << best;
                    }
                }
        }
    }
    // positions: within each bank group in sorted-id order, so the producer's gather (lane i ->
    // position i) still walks nearly sorted ids (coalesced cp.async sources)
    int next[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    for (int u = 0; u < nl; ++u) {
        const int b = asg[l0 + u] & 7;  // (given banks are always set; & 7 keeps this total)
        asg[l0 + u] = next[b];
        next[b] += 8;
    }
    for (int p = 0; p < nlp; ++p) tnbr[l0 + p] = -1;
    for (int u = 0; u < nl; ++u) tnbr[l0 + asg[l0 + u]] = ids[l0 + u];
    auto remap = [&](unsigned off) {
        return off == pad_pos ? off : (unsigned)asg[l0 + off / r4b] * r4b;
    };
    for (long long sl = s0; sl < slot; ++sl) {
        uint2 s = tent[sl];
        s.x = remap(s.x & 0xffffu) | (remap(s.x >> 16) << 16);
        s.y = remap(s.y & 0xffffu) | (s.y & 0xffff0000u);
        tent[sl] = s;
    }
}

// Bank groups by DSATUR colouring of the tile's conflict graph (one warp per tile; run before
// k_tile_banks with given = 1).  Two neighbours conflict when they share a quarter-warp group
// (8 lanes x one tet corner of one slot block); the colours are the 8 bank groups, each
// holding at most nlp / 8 neighbours.  Repeatedly the uncoloured neighbour with the most
// distinct bank groups among its group-mates (then the most groups) takes the admissible bank
// group with the fewest coloured group-mates (then the least filled).  On C5-like tiles this
// leaves ~1.1x the ideal wavefronts where the sweep-order greedy left ~1.3x (prototype).
// Shared memory per warp: sat, col, cnt/cursor (4 B x V each), moff (4 B x (V + 1)),
// mlist (2 B x 3 slots).
__global__ void __launch_bounds__(32) k_tile_banks_dsatur(const long long* __restrict__ lbase,
                                                         const long long* __restrict__ sbase,
                                                         const int* __restrict__ nls, int nt, unsigned r4b,
                                                         unsigned pad_pos, const uint2* __restrict__ tent,
                                                         int* __restrict__ asg, int vmax, int mmax)
{
    extern __shared__ int sm[];
    const int t = blockIdx.x;
    if (t >= nt) return;
    const int lane = threadIdx.x;
    const long long l0 = lbase[t], s0 = sbase[t];
    const int V = nls[t], cap = (int)(lbase[t + 1] - l0) / 8;
    const int nslots = (int)(sbase[t + 1] - s0), ngroups = nslots / 8 * 3;
    const int pad_bank = (int)((pad_pos / r4b) & 7u);
    int* sat = sm;
    int* col = sat + vmax;
    int* cur = col + vmax;
    int* moff = cur + vmax;
    unsigned short* mlist = reinterpret_cast<unsigned short*>(moff + vmax + 1);
    if (V > vmax || 3 * nslots > mmax) {  // cannot happen (sized from the tile caps); keep greedy
        for (int u = lane; u < V; u += 32) asg[l0 + u] = -1;
        return;
    }
    auto member = [&](int gi, int l) -> int {  // neighbour index, -2 = padding position
        const uint2 e = tent[s0 + 8 * (gi / 3) + l];
        const int k = gi % 3;
        const unsigned off = (k == 0 ? e.x : k == 1 ? e.x >> 16 : e.y) & 0xffffu;
        return off == pad_pos ? -2 : (int)(off / r4b);
    };
    auto first = [&](const int* u, int l) {  // u[l] is the first lane of the group holding it
        for (int m = 0; m < l; ++m)
            if (u[m] == u[l]) return false;
        return true;
    };
    for (int u = lane; u < V; u += 32) {
        sat[u] = 0;
        col[u] = -1;
        cur[u] = 0;
    }
    __syncwarp();
    for (int gi = lane; gi < ngroups; gi += 32) {  // memberships (distinct per group)
        int u[8];
        bool pad = false;
        for (int l = 0; l < 8; ++l) {
            u[l] = member(gi, l);
            pad |= u[l] == -2;
        }
        for (int l = 0; l < 8; ++l)
            if (u[l] >= 0 && first(u, l)) {
                atomicAdd(&cur[u[l]], 1);
                if (pad) atomicOr(&sat[u[l]], 1 << pad_bank);
            }
    }
    __syncwarp();
    if (lane == 0) {
        int acc = 0;
        for (int u = 0; u < V; ++u) {
            moff[u] = acc;
            acc += cur[u];
            cur[u] = moff[u];
        }
        moff[V] = acc;
    }
    __syncwarp();
    for (int gi = lane; gi < ngroups; gi += 32) {
        int u[8];
        for (int l = 0; l < 8; ++l) u[l] = member(gi, l);
        for (int l = 0; l < 8; ++l)
            if (u[l] >= 0 && first(u, l)) mlist[atomicAdd(&cur[u[l]], 1)] = (unsigned short)gi;
    }
    __syncwarp();
    int fill[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // warp-uniform
    for (int step = 0; step < V; ++step) {
        // the uncoloured neighbour with the largest (saturation, memberships, -index)
        long long best = -1;
        for (int u = lane; u < V; u += 32)
            if (col[u] < 0) {
                const long long key = ((long long)__popc(sat[u]) << 40) | ((long long)(moff[u + 1] - moff[u]) << 20) |
                                      (long long)(0xfffff - u);
                best = key > best ? key : best;
            }
        for (int o = 16; o > 0; o >>= 1) {
            const long long other = __shfl_xor_sync(0xffffffffu, best, o);
            best = other > best ? other : best;
        }
        const int u = 0xfffff - (int)(best & 0xfffff);
        // coloured group-mates per bank group (distinct per group; padding counts as pad_bank)
        int c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int m = moff[u] + lane; m < moff[u + 1]; m += 32) {
            const int gi = mlist[m];
            int v[8];
            for (int l = 0; l < 8; ++l) v[l] = member(gi, l);
            for (int l = 0; l < 8; ++l) {
                if (v[l] == u || !first(v, l)) continue;
                const int b = v[l] == -2 ? pad_bank : col[v[l]];
                if (b >= 0) ++c[b];
            }
        }
#pragma unroll
        for (int b = 0; b < 8; ++b)
            for (int o = 16; o > 0; o >>= 1) c[b] += __shfl_xor_sync(0xffffffffu, c[b], o);
        int bb = -1;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (fill[b] < cap && (bb < 0 || c[b] < c[bb] || (c[b] == c[bb] && fill[b] < fill[bb]))) bb = b;
        ++fill[bb];
        if (lane == 0) col[u] = bb;
        for (int m = moff[u] + lane; m < moff[u + 1]; m += 32) {
            const int gi = mlist[m];
            for (int l = 0; l < 8; ++l) {
                const int v = member(gi, l);
                if (v >= 0 && v != u) atomicOr(&sat[v], 1 << bb);
            }
        }
        __syncwarp();
    }
    for (int u = lane; u < V; u += 32) asg[l0 + u] = col[u];
}

// per-tile descriptor (64 B): the producer loads the first 32 B; the whole record is
// bulk-copied into the stage header for the consumers
struct __align__(16) TileDesc {
    long long eb;   // first entry slot (tiles are 256-byte aligned in the slot array)
    long long l0;   // neighbour list base
    int v0, nv;     // vertices
    int ne;         // entry slots
    int nl;         // distinct neighbours
    int wr[8];      // consumer warp w: rounds | (first slot / 32) << 16
};
struct __align__(16) TileDescHead {
    long long eb, l0;
    int v0, nv, ne, nl;
};

__global__ void k_tile_desc(const int* __restrict__ tv0, const int* __restrict__ tnv,
                            const long long* __restrict__ eoff, const long long* __restrict__ lbase,
                            const long long* __restrict__ sbase, int nt, int W, TileDesc* __restrict__ out,
                            const signed char* __restrict__ tw = nullptr, const int* __restrict__ tcw = nullptr)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    if (tw) W = tw[t];
    TileDesc d;
    d.v0 = tv0[t];
    d.nv = tnv[t];
    d.eb = sbase[t];
    d.ne = (int)(sbase[t + 1] - sbase[t]);
    d.l0 = lbase[t];
    d.nl = (int)(lbase[t + 1] - d.l0);
    int pre = 0;
    for (int w = 0; w < 8; ++w) {
        const int r = tile_warp_rounds(eoff, d.v0, d.nv, w, W);
        d.wr[w] = r | (pre << 16);
        pre += r;
    }
    // class tiles (4 consumer warps of 32 vertices, so warp 7 has no rounds): wr[7] =
    // (class + 1) | (byte offset of the instance's records in the shared table) << 16
    if (tcw && tcw[t]) d.wr[7] = tcw[t];
    out[t] = d;
}

template <typename R> struct K1TArgs {
    K1Args<R> a;               // vbeg/count = the colour range; pos/xt/y/flag/peer as K1
    const uint2* tent;         // tile entries, global CSR order (+2 pad)
    const int* tnbr;           // neighbour lists
    const TileDesc* desc;      // per-tile descriptors
    const typename PlaneT<R>::T* kinds;  // KindRec table (the sweep stages the first 12 R)
    int tbeg, tcount;          // tiles of this colour
    int ent_cap, nbr_cap;      // per-stage capacity (entries incl. pad, neighbours)
    int nkinds;
    int dbg;  // timing experiments only (VBD_TILE_DBG): 1 consumers skip the entry sweep,
              // 2 the producer skips the neighbour gathers; results are wrong in both
    const float* xrows;  // K1T-X: slot-weight rows, 9 planes of xstride floats in slot order
    long long xstride;
    int early;           // producer loads its first descriptors / ids before the PDL wait
    const int* ckind;    // class tiles: kind id of every class record (after the zero record)
    int ncrec;
    int svpt;            // stage capacity for x / x_t / y (vertices; 128 with class tiles)
    int xtg;             // x_t / y read from global by the consumers, not staged (class tiles)
    int tcls;            // class tiles of this colour are [tcls, tcount) (tcount: none)
};

typedef TileDesc TileHdr;  // the stage header is a copy of the tile's descriptor



__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
template <int N> __device__ __forceinline__ void cp_async_n(void* dst, const void* src)
{
    if constexpr (N == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// dynamic smem: [kind records (12 R each)][stages]; per stage: hdr | entry slots | neighbour
// positions | x | x_t | y
template <typename R> struct TileSmem {
    typedef typename Vec4<R>::T R4;
    int ent_cap, nbr_cap, nk, vpt;  // vpt: vertices per tile
    int nxv = 3;  // vertex arrays staged: x, x_t, y (3) or x only (1: x_t / y read from global)
    // kind records (HOT R each), then for fp32 (displacement state) the kinds' rest edges
    // (3 float4 = 48 B each: the same byte offset as the fp32 record, in the second table)
    // fp32 (displacement state): one packed 80-byte SWEEP record per kind, read with 4 LDS.128 +
    // 1 LDS.32 per entry: [E0.xyz, t0] [E1.xyz, t1] [E2.xyz, t2] [t3 t4 t5 t6] [t7 t8 dsc opd]
    // (E = rest edges, t = ec_terms); fp64: the HOT part of the kind record
    static constexpr unsigned KSTRIDE = sizeof(R) == 4 ? 80u : (unsigned)(KindRec<R>::HOT * sizeof(R));
    __host__ __device__ size_t recs_bytes() const { return (size_t)(nk + 1) * KSTRIDE; }
    __host__ __device__ size_t kinds_bytes() const { return recs_bytes(); }
    __host__ __device__ size_t off_hdr() const { return 0; }
    __host__ __device__ size_t off_ent() const { return sizeof(TileDesc); }
    // neighbour positions, 16-byte units: fp32 one float4 per neighbour; fp64 the (x, y) halves of
    // all neighbours, then the (z, w) halves (off_nzw), so a quarter-warp LDS.128 of 8 placed
    // neighbours hits 8 distinct bank groups (a 32-byte double4 stride would reach only 4)
    static constexpr unsigned PU = 16;
    __host__ __device__ size_t off_npos() const { return off_ent() + (size_t)ent_cap * 8; }
    __host__ __device__ size_t off_nzw() const { return off_npos() + (size_t)(nbr_cap + 1) * PU; }
    __host__ __device__ size_t off_x() const { return off_npos() + (size_t)(nbr_cap + 1) * sizeof(R4); }
    __host__ __device__ size_t off_xt() const { return off_x() + (nxv == 3 ? vpt * sizeof(R4) : 0); }
    __host__ __device__ size_t off_y() const { return off_xt() + (nxv == 3 ? vpt * sizeof(R4) : 0); }
    __host__ __device__ size_t stage_bytes() const
    {
        return (off_x() + (size_t)nxv * vpt * sizeof(R4) + 127) & ~(size_t)127;
    }
    __host__ __device__ size_t total(int stages) const { return ((kinds_bytes() + 127) & ~(size_t)127) + stages * stage_bytes(); }
};

// 32-bit shared-window loads (one add per address instead of generic-pointer arithmetic);
// volatile keeps them after the stage's mbarrier wait
__device__ __forceinline__ void lds_v(unsigned a, float4& v)
{
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
}
__device__ __forceinline__ void lds_v(unsigned a, double4& v)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.z), "=d"(v.w) : "r"(a + 16));
}
// a staged neighbour position at byte offset a (16-byte units): fp64 reads the (z, w) half
// from the second array, zw bytes further
__device__ __forceinline__ void lds_pos(unsigned a, unsigned, float4& v) { lds_v(a, v); }
__device__ __forceinline__ void lds_pos(unsigned a, unsigned zw, double4& v)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.z), "=d"(v.w) : "r"(a + zw));
}
__device__ __forceinline__ void lds_v(unsigned a, double2& v)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
}
__device__ __forceinline__ float lds_f32(unsigned a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_u2(unsigned a)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// the vertex update after the block solve: in-place store, NVLink ghost store, finite check
template <typename R>
__device__ __forceinline__ void k1t_store(const K1Args<R>& a, int v, typename Vec4<R>::T nx)
{
    a.pos[v] = nx;
    if (a.peer_pos[0] || a.peer_pos[1]) {
        const int jj = v - a.vbeg;
        if (jj < a.nb[0]) {
            a.peer_pos[0][a.peer_off[0] + jj] = nx;  // NVLink store into the left ghost
        } else if (jj < a.nb[0] + a.nb[1]) {
            a.peer_pos[1][a.peer_off[1] + (jj - a.nb[0])] = nx;
        }
    }
    if (a.flag && !finite3(nx.x, nx.y, nx.z))
        atomicMin(a.flag, StepFlag::key((unsigned)*a.stepctr, (unsigned)a.iter, (unsigned)a.perm[v]));
}

// read-only global loads issued where they stand (volatile: not sunk to their first use)
__device__ __forceinline__ void ldg_nc(const float4* p, float4& v)
{
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
}
__device__ __forceinline__ void ldg_nc(const double4* p, double4& v)
{
    v = *p;
}
__device__ __forceinline__ float ldg_nc(const float* p)
{
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg_nc(const double* p) { return *p; }

// K1T class tile sweep (one lane per vertex of grid class C, vbd_grid_classes.cuh).  The lane's
// slots are its vertex's distinct neighbours in class order, 3 per row (bank-placed offsets);
// each position is loaded once, at its first use, and the class's entries run in position order
// q from registers with the record at recs + 80 q (the instance's block in the shared table:
// the same address on every lane, a broadcast).  Entry q goes to accumulator set q mod 4 in
// increasing q, so (s0 + s2) + (s1 + s3) is exactly the 2-lane path's lane sums + butterfly.
template <int C>
__device__ __forceinline__ void class_sweep(const unsigned char* slots, const unsigned char* npos,
                                            const unsigned char* recs, float2 nxy, float nz, AccXY (&acc)[4])
{
    using G = GridClass<C>;
    DiffXY P[G::NL];  // u_k - u_i of every neighbour, formed once (each is used ~5 times)
    uint2 row[G::R];
#pragma unroll
    for (int q = 0; q < G::NE; ++q) {
#pragma unroll
        for (int k = 0; k < G::NL; ++k) {
            if (G::first(k) != q) continue;
            if (k % 3 == 0) row[k / 3] = *reinterpret_cast<const uint2*>(slots + 256 * (k / 3));
            const unsigned off = k % 3 == 0 ? (row[k / 3].x & 0xffffu)
                                            : (k % 3 == 1 ? (row[k / 3].x >> 16) : (row[k / 3].y & 0xffffu));
            P[k] = diff_xy(*reinterpret_cast<const float4*>(npos + off), nxy, nz);
        }
        const float4* rec = reinterpret_cast<const float4*>(recs + 80 * q);
        const float4 e0 = rec[0], e1 = rec[1], e2 = rec[2], c3 = rec[3];
        const float t[8] = {e0.w, e1.w, e2.w, c3.x, c3.y, c3.z, c3.w, reinterpret_cast<const float*>(rec + 4)[0]};
        tet_contrib_ec_xy_d(P[G::nbr(q, 0)], P[G::nbr(q, 1)], P[G::nbr(q, 2)], e0, e1, e2, t, acc[q & 3]);
    }
}

// OCC = CTAs per SM the kernel is compiled for (register budget); OCC >= 3 sweeps one entry
// per lane at a time (fewer live registers), else two.
// DEF = W: deferred block solves.  After a tile's butterfly every lane of a vertex holds its
// sums; the vertex terms run on all of them and lane j = (tile count mod W) keeps (f, H, v).
// Every W tiles the warp solves and stores 32 vertices with all lanes active, instead of
// 32 / W vertices per tile with a quarter of the lanes.  Vertices of one colour do not read
// each other, so deferring their stores inside the launch changes nothing (bitwise).
// Tiles are 64 vertices: NCW = 2 W consumer warps of 32 / W vertices (W = 4: 8 warps, W = 2:
// 4 warps of 16 vertices with twice the rounds -- half the per-vertex reduction and solve
// overhead per entry).
// KG: the kind table is too large for shared memory (e.g. fp64 grids whose rest shapes differ
// in the last bits): slots carry the kind index and the records are read through L1 from global.
// XR (K1T-X, fp32, one material per vertex): explicit entries -- the slots carry no kind; each
// entry's 9 slot-weight rows stream from ta.xrows (coalesced: a warp round reads 128 B per
// plane) and its constants, volume and rest edges are derived exactly as the explicit K1 does
// (ec_terms, volume_from_rows, rest_edges_from_rows), so results stay bitwise equal to it.
// TV: vertices per tile (64; 32 for small scenes: twice the CTAs per colour pass, half the
// gather and sweep per CTA).
// CL: the colour's class tiles run in a second loop (class_sweep); instantiated only for
// contexts that have class tiles, so the plain kernel keeps its register allocation.
template <typename R, bool UM, int S, int W, int OCC, int DEF, bool KG = false, bool XR = false, int TV = 64,
          bool CL = false>
__global__ void __launch_bounds__(TV * W + 32, OCC) k1_tiles(const K1TArgs<R> ta)
{
    typedef typename Vec4<R>::T R4;
    constexpr int VPW = 32 / W;  // vertices per consumer warp
    constexpr int NCW = TV * W / 32;  // consumer warps
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long full[S], empty[S];
    const K1Args<R>& a = ta.a;
    static_assert(!XR || (sizeof(R) == 4 && UM && !KG), "K1T-X: fp32, one material per vertex");
    // CL (class tiles): x_t / y are not staged but read by the consumers (ta.xtg is then 1)
    const TileSmem<R> L{ta.ent_cap, ta.nbr_cap, (KG || XR) ? -1 : ta.nkinds + ta.ncrec, ta.svpt, CL ? 1 : 3};
    typedef typename PlaneT<R>::T PL;
    PL* skind = reinterpret_cast<PL*>(smem);
    unsigned char* stages = smem + ((L.kinds_bytes() + 127) & ~(size_t)127);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int QH = KindRec<R>::QH, Q = KindRec<R>::Q;
    // chunks the entry loop reads: with one material per vertex the sweep needs t[0..7] only
    // (t[8] = V mu |w|^2 is summed per vertex at pack time, dsc / opd are read once per vertex)
    constexpr int QS = UM ? 8 * (int)sizeof(R) / 16 : QH;
    constexpr bool DISP = sizeof(R) == 4;  // fp32: displacement state, rest edges per kind
    if (!KG && !XR) {
        if constexpr (DISP) {  // packed fp32 sweep records (TileSmem::KSTRIDE); padding: zero record
            // (class tiles: the instances' records follow the zero record, ckind[i] for record
            // nkinds + 1 + i)
            float4* sk = reinterpret_cast<float4*>(smem);
            for (int i = tid; i < (ta.nkinds + 1 + ta.ncrec) * 5; i += blockDim.x) {
                const int k0 = i / 5, q = i % 5;
                const int k = k0 < ta.nkinds ? k0 : (k0 == ta.nkinds ? -1 : ta.ckind[k0 - ta.nkinds - 1]);
                float4 v{};
                if (k >= 0) {
                    const float* t = reinterpret_cast<const float*>(ta.kinds + (size_t)k * Q);
                    if (q < 3) {
                        v = ta.a.kedge[3 * k + q];
                        v.w = t[q];
                    } else if (q == 3) {
                        v = make_float4(t[3], t[4], t[5], t[6]);
                    } else {
                        v = make_float4(t[7], t[8], t[9], t[10]);
                    }
                }
                sk[i] = v;
            }
        } else {
            for (int i = tid; i < ta.nkinds * QH; i += blockDim.x) skind[i] = ta.kinds[(i / QH) * Q + i % QH];
            for (int i = tid; i < QH; i += blockDim.x) skind[ta.nkinds * QH + i] = PL{};  // padding: zero record
        }
    }
    for (int s = 0; s < S; ++s)  // padding: zero position after the largest neighbour list
        if (tid == 0) {
            unsigned char* z = stages + s * L.stage_bytes() + L.off_npos() + (size_t)ta.nbr_cap * L.PU;
            *reinterpret_cast<float4*>(z) = float4{};
            if constexpr (sizeof(R4) == 32) *reinterpret_cast<float4*>(z + (L.off_nzw() - L.off_npos())) = float4{};
        }
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(smem_u32(&full[s]), 33);  // expect_tx arrive + 32 cp.async arrivals
            mbar_init(smem_u32(&empty[s]), NCW);  // one per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // programmatic dependent launch: everything above reads step constants only (the kind
    // table is rewritten only by refresh_kinds, which synchronises the stream before any
    // colour pass is enqueued); positions are read after the predecessor grid has finished.
    // Overlapping this prologue with the previous pass is worth ~10 % on C1 / C2.  The
    // producer also loads its first tiles' descriptors and neighbour ids (step constants)
    // before it waits; the consumers wait here.
    if (warp != NCW || !ta.early) pdl_wait();
    pdl_launch_dependents();

    if (warp == NCW) {  // ---------------- producer
        // Software-pipelined, unrolled by two with named buffers (no register copies that would
        // expose load latency): while tile t is issued, the neighbour ids of tile t + grid and
        // the descriptor of tile t + 2 grid are in flight.
        constexpr int B = 16;
        auto head = [&](int t) {
            TileDescHead h{};
            if (t < ta.tcount) h = *reinterpret_cast<const TileDescHead*>(ta.desc + ta.tbeg + t);
            return h;
        };
        auto load_ids = [&](const TileDescHead& dd, int base, int* ids) {
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int i = base + q * 32 + lane;
                ids[q] = i < dd.nl ? __ldg(ta.tnbr + dd.l0 + i) : -1;
            }
        };
        int stage = 0;
        unsigned ph = 0;
        auto issue = [&](int t, const TileDescHead& d, int* ids) {
            mbar_wait_parity(smem_u32(&empty[stage]), ph ^ 1);
            unsigned char* st = stages + stage * L.stage_bytes();
            const unsigned bar = smem_u32(&full[stage]);
            if (lane == 0) {
                const unsigned eby = (unsigned)d.ne * 8u, vby = (unsigned)(d.nv * sizeof(R4));
                mbar_expect_tx(bar, (unsigned)sizeof(TileDesc) + eby + (unsigned)L.nxv * vby);
                bulk_g2s(st + L.off_hdr(), ta.desc + ta.tbeg + t, (unsigned)sizeof(TileDesc), bar);
                if (eby) bulk_g2s(st + L.off_ent(), ta.tent + d.eb, eby, bar);
                bulk_g2s(st + L.off_x(), a.pos + d.v0, vby, bar);
                if constexpr (!CL) {
                    bulk_g2s(st + L.off_xt(), a.xt + d.v0, vby, bar);
                    bulk_g2s(st + L.off_y(), a.y + d.v0, vby, bar);
                } else {  // x_t / y (and the vertices' V mu |w|^2 sums) into L2 for the consumers
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.xt + d.v0), "r"(vby) : "memory");
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.y + d.v0), "r"(vby) : "memory");
                    if (UM && a.vsv) {  // (16-byte aligned range covering the tile's sums)
                        const size_t b0 = reinterpret_cast<size_t>(a.vsv + d.v0) & ~(size_t)15;
                        const size_t b1 = (reinterpret_cast<size_t>(a.vsv + d.v0 + d.nv) + 15) & ~(size_t)15;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"((unsigned)(b1 - b0))
                                     : "memory");
                    }
                }
                if constexpr (XR) {  // the tile's rows into L2 (the consumers stream them next)
#pragma unroll 1
                    for (int q = 0; q < 9; ++q)
                        if (eby)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                             ta.xrows + (size_t)q * ta.xstride + d.eb),
                                         "r"(eby / 2u)
                                         : "memory");
                }
            }
            unsigned char* np = st + L.off_npos();
            for (int base = 0; ta.dbg != 2;) {
#pragma unroll
                for (int q = 0; q < B; ++q) {
                    if (ids[q] < 0) continue;
                    const int i = base + q * 32 + lane;
                    const char* src = reinterpret_cast<const char*>(a.pos + ids[q]);
                    cp_async_n<16>(np + (size_t)i * L.PU, src);
                    if constexpr (sizeof(R4) == 32)  // (z, w) half into the second array
                        cp_async_n<16>(np + (L.off_nzw() - L.off_npos()) + (size_t)i * L.PU, src + 16);
                }
                base += 32 * B;
                if (base >= d.nl) break;
                load_ids(d, base, ids);  // rare: more than 32 B neighbours
            }
            cp_async_mbar_arrive(bar);
            if (++stage == S) {
                stage = 0;
                ph ^= 1;
            }
        };
        const int g = (int)gridDim.x;
        TileDescHead d0 = head(blockIdx.x), d1 = head(blockIdx.x + g);
        int i0[B], i1[B];
        load_ids(d0, 0, i0);
        if (ta.early) pdl_wait();  // positions and x / x_t / y are the predecessor's output
        for (int t = blockIdx.x; t < ta.tcount; t += 2 * g) {
            load_ids(d1, 0, i1);                       // tile t + g
            const TileDescHead d0n = head(t + 2 * g);  // tile t + 2g
            issue(t, d0, i0);
            if (t + g >= ta.tcount) break;
            load_ids(d0n, 0, i0);                      // tile t + 2g
            const TileDescHead d1n = head(t + 3 * g);  // tile t + 3g
            issue(t + g, d1, i1);
            d0 = d0n;
            d1 = d1n;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ---------------- consumers: warp w handles tile vertices VPW w .. VPW w + VPW - 1;
    // lane = VPW j + vi serves entry positions j, j + W, ... of vertex vi
    const int vi = lane % VPW, j = lane / VPW;
    const int lv = warp * VPW + vi;
    int stage = 0;
    unsigned ph = 0;
    static_assert(DEF == 1 || DEF == W, "deferral batches one tile per lane of a vertex");
    int tc = 0, qv = -1;  // DEF > 1: tiles since the last flush; the deferred vertex of this lane
    R qf[DEF > 1 ? 3 : 1], qH[DEF > 1 ? 6 : 1];
    typename Vec4<R>::T qx{};  // its x (from the stage; a reload from global stalled the flush)
    auto flush = [&]() {
        if constexpr (DEF > 1) {
            if (qv >= 0) {
                R d[3];
                block_solve<R>(qf, qH, a.eps_det, a.mode, d);
                R4 nx = qx;
                nx.x = nx.x + d[0];
                nx.y = nx.y + d[1];
                nx.z = nx.z + d[2];
                k1t_store<R>(a, qv, nx);
            }
            qv = -1;
        }
    };
    // class tiles (fp32, one material per vertex, 2-lane 64-vertex tiles): wr[7] = (class + 1) |
    // record block offset << 16; one lane per vertex, 32 vertices per consumer warp
    constexpr bool CLS = CL && sizeof(R) == 4 && UM && W == 2 && !KG && !XR && TV == 64;
    static_assert(!CL || CLS, "class tiles: fp32, one material per vertex, 2-lane 64-vertex tiles");
    // the colour's plain tiles first, then (CLS) its class tiles [tcls, tcount) in a second loop
    // over the same grid-stride sequence, so the deferral state is dead in the class sweep
    int t = blockIdx.x;
    for (; t < (CLS ? ta.tcls : ta.tcount); t += gridDim.x) {
        mbar_wait_parity(smem_u32(&full[stage]), ph);
        const unsigned char* st = stages + stage * L.stage_bytes();
        const TileHdr* hp = reinterpret_cast<const TileHdr*>(st + L.off_hdr());
        const int hv0 = hp->v0, hnv = hp->nv, wr = hp->wr[warp];
        const int rounds = ta.dbg == 1 ? 0 : wr & 0xffff, sb = wr >> 16;
        const uint2* sent = reinterpret_cast<const uint2*>(st + L.off_ent()) + 32 * sb + lane;
        const R4* np = reinterpret_cast<const R4*>(st + L.off_npos());
        const bool act = lv < hnv;
        const int lvc = act ? lv : 0;
        const R4 xi4 = reinterpret_cast<const R4*>(st + L.off_x())[lvc];
        const R4 xt4 = CL ? a.xt[hv0 + lvc] : reinterpret_cast<const R4*>(st + L.off_xt())[lvc];
        const R4 y4 = CL ? a.y[hv0 + lvc] : reinterpret_cast<const R4*>(st + L.off_y())[lvc];
        const R xi[3] = {xi4.x, xi4.y, xi4.z};
        const R dx[3] = {xi[0] - xt4.x, xi[1] - xt4.y, xi[2] - xt4.z};
        // NA = 4 / W accumulator sets: with W = 2, lane j sums entry positions j mod 4 (even
        // rounds) and j + 2 mod 4 (odd rounds) apart and adds them before the butterfly --
        // exactly the partial sums and pairing of the 4-lane variants (bitwise equal)
        constexpr int NA = 4 / W;
        R fa[NA][3], Ha[NA][6], sva[NA];
#pragma unroll
        for (int b = 0; b < NA; ++b) {
#pragma unroll
            for (int q = 0; q < 3; ++q) fa[b][q] = R(0);
#pragma unroll
            for (int q = 0; q < 6; ++q) Ha[b][q] = R(0);
            sva[b] = R(0);
        }
        const R svv = UM && act ? a.vsv[hv0 + lv] : R(0);  // added after the lane reduction
        R dsc = R(0), opd = R(1);
        constexpr int U = OCC >= 3 && W == 4 ? 1 : VBD_TILE_U;  // register budget
        static_assert(U % NA == 0, "rounds per iteration must cover the accumulator sets");
        // fp32 with one material per vertex: packed fp32x2 arithmetic (tet_contrib_ec_xy)
        constexpr bool PACK = sizeof(R) == 4 && UM;
        AccXY acc[NA];
#pragma unroll
        for (int b = 0; b < NA; ++b) acc[b].zero();
        const float2 nxy = make_float2(-(float)xi[0], -(float)xi[1]);
        const float nz = -(float)xi[2];
        const unsigned npb = smem_u32(np);
        const unsigned nzw = (unsigned)(L.off_nzw() - L.off_npos());
        const unsigned kb = smem_u32(skind);
        const unsigned sb32 = smem_u32(sent);
        const long long hxeb = XR ? hp->eb : 0;  // K1T-X: the tile's first slot (rows index)
        const unsigned padp = (unsigned)ta.nbr_cap * L.PU;
        Material<R> xmat{};
        if constexpr (XR) xmat = a.mat[a.vmat[hv0 + lvc]];
        // K1T-X: the rows of the next XPF iterations are in flight (registers), a rotating window
        constexpr int XPF = 1;  // (2 at 2 CTAs/SM spills: 3.54 vs 3.21 ms per C5j pass)
        float wn[XR ? XPF : 1][XR ? U : 1][XR ? 9 : 1];
        auto load_rows = [&](int i0n, float (&dst)[XR ? U : 1][XR ? 9 : 1]) {
            if constexpr (XR) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float* xp = ta.xrows + hxeb + 32ll * (sb + i0n + u) + lane;
#pragma unroll
                    for (int q = 0; q < 9; ++q) dst[u][q] = i0n < rounds ? __ldcs(xp + q * ta.xstride) : 0.0f;
                }
            }
        };
#pragma unroll
        for (int f = 0; f < (XR ? XPF : 0); ++f) load_rows(f * U, wn[f]);
        for (int i0 = 0; i0 < rounds; i0 += U) {  // rounds is a multiple of U
            uint2 e[U];
            R4 p[U][3];
            float wc[XR ? U : 1][XR ? 9 : 1];
            if constexpr (XR) {
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < 9; ++q) wc[u][q] = wn[0][u][q];
#pragma unroll
                for (int f = 0; f + 1 < XPF; ++f)
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < 9; ++q) wn[f][u][q] = wn[f + 1][u][q];
                load_rows(i0 + XPF * U, wn[XPF - 1]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                e[u] = lds_u2(sb32 + 256u * (unsigned)(i0 + u));
                lds_pos(npb + (e[u].x & 0xffffu), nzw, p[u][0]);
                lds_pos(npb + (e[u].x >> 16), nzw, p[u][1]);
                lds_pos(npb + (e[u].y & 0xffffu), nzw, p[u][2]);
            }
            float4 ex[U][3];  // fp32: the entries' rest edges
            R r[U][KindRec<R>::HOT];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned rp = kb + (e[u].y >> 16);
                if constexpr (XR) {  // rows streamed from global (one iteration ahead), constants here
                    const float* w = wc[u];
                    const bool valid = (e[u].x & 0xffffu) != padp;  // padding slot: contributes +0
                    const float V = valid ? volume_from_rows(w) : 0.0f;
                    ec_terms<float>(w, V, xmat.mu, xmat.lam, xmat.gamma, reinterpret_cast<float*>(r[u]));
                    rest_edges_from_rows(w, ex[u]);
                    if (!valid) ex[u][0] = ex[u][1] = ex[u][2] = float4{};
                } else if constexpr (DISP && !KG) {  // packed sweep record: 4 LDS.128 + 1 LDS.32 (UM)
                    float4 c3;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        lds_v(rp + 16u * q, ex[u][q]);
                        r[u][q] = ex[u][q].w;
                    }
                    lds_v(rp + 48u, c3);
                    r[u][3] = c3.x;
                    r[u][4] = c3.y;
                    r[u][5] = c3.z;
                    r[u][6] = c3.w;
                    if constexpr (UM) {
                        r[u][7] = lds_f32(rp + 64u);
                    } else {
                        float4 c4;
                        lds_v(rp + 64u, c4);
                        r[u][7] = c4.x;
                        r[u][8] = c4.y;
                        r[u][9] = c4.z;
                        r[u][10] = c4.w;
                    }
                } else {
                    if constexpr (DISP) {  // (KG: rest edges from the global table)
#pragma unroll
                        for (int q = 0; q < 3; ++q) ex[u][q] = __ldg(ta.a.kedge + 3 * (size_t)(e[u].y >> 16) + q);
                    }
#pragma unroll
                    for (int q = 0; q < QS; ++q) {
                        PL v;
                        if constexpr (KG) v = __ldg(ta.kinds + (size_t)(e[u].y >> 16) * Q + q);
                        else lds_v(rp + 16u * q, v);
                        const R* vr = reinterpret_cast<const R*>(&v);
#pragma unroll
                        for (int z = 0; z < 16 / (int)sizeof(R); ++z) r[u][q * (16 / (int)sizeof(R)) + z] = vr[z];
                    }
                }
            }
            if constexpr (PACK) {  // x/y of every 3-vector packed as fp32x2 (FFMA2)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    tet_contrib_ec_xy(p[u][0], p[u][1], p[u][2], nxy, nz, ex[u][0], ex[u][1], ex[u][2],
                                      reinterpret_cast<const float*>(r[u]), acc[u % NA]);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    R e0[3], e1[3], e2[3];
                    edge3<R>(p[u][0], xi, ex[u][0], DISP, e0);
                    edge3<R>(p[u][1], xi, ex[u][1], DISP, e1);
                    edge3<R>(p[u][2], xi, ex[u][2], DISP, e2);
                    const int b = u % NA;  // i0 is a multiple of U, so (i0 + u) % NA == u % NA (unrolled)
                    tet_contrib_ec<R, !UM>(e0, e1, e2, r[u], UM ? R(0) : r[u][9], UM ? R(1) : r[u][10], dx, fa[b],
                                           Ha[b], sva[b]);
                }
            }
        }
        if constexpr (XR) {  // damping from the vertex's material (explicit K1: the same)
            dsc = xmat.dsc;
            opd = xmat.opd;
        } else if (UM && rounds > 0) {  // the record of this lane's round-0 slot (position j; lane j = 0
                                 // holds the vertex's first entry), read once, not per iteration
            const uint2 e0s = lds_u2(sb32);
            PL v;
            if constexpr (KG) v = __ldg(ta.kinds + (size_t)(e0s.y >> 16) * Q + 2);
            else if constexpr (DISP) {  // packed record chunk 4 = (t7, t8, dsc, opd): as chunk 2's (., dsc, opd)
                float4 c4;
                lds_v(kb + (e0s.y >> 16) + 64u, c4);
                v = make_float4(c4.y, c4.z, c4.w, 0.0f);
            } else lds_v(kb + (e0s.y >> 16) + 32u, v);
            const R* vr = reinterpret_cast<const R*>(&v);
            if constexpr (sizeof(R) == 4) {  // r[8..11] = chunk 2
                dsc = vr[1];
                opd = vr[2];
            } else {  // double2 chunks: r[8..9] = chunk 4, r[10..11] = chunk 5
                PL v5;
                if constexpr (KG) {
                    v = __ldg(ta.kinds + (size_t)(e0s.y >> 16) * Q + 4);
                    v5 = __ldg(ta.kinds + (size_t)(e0s.y >> 16) * Q + 5);
                } else {
                    lds_v(kb + (e0s.y >> 16) + 64u, v);
                    lds_v(kb + (e0s.y >> 16) + 80u, v5);
                }
                dsc = reinterpret_cast<const R*>(&v)[1];
                opd = reinterpret_cast<const R*>(&v5)[0];
            }
        }
        if constexpr (PACK) {
#pragma unroll
            for (int b = 0; b < NA; ++b) {
                fa[b][0] = acc[b].f01.x;
                fa[b][1] = acc[b].f01.y;
                fa[b][2] = acc[b].f2;
                Ha[b][0] = acc[b].h03.x;
                Ha[b][1] = acc[b].h1;
                Ha[b][2] = acc[b].h24.x;
                Ha[b][3] = acc[b].h03.y;
                Ha[b][4] = acc[b].h24.y;
                Ha[b][5] = acc[b].h5;
            }
        }
        R f[3], H[6];
#pragma unroll
        for (int q = 0; q < 3; ++q) f[q] = NA == 2 ? fa[0][q] + fa[NA - 1][q] : fa[0][q];
#pragma unroll
        for (int q = 0; q < 6; ++q) H[q] = NA == 2 ? Ha[0][q] + Ha[NA - 1][q] : Ha[0][q];
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));  // stage's smem no longer read
        // the W lanes of a vertex are vi + VPW j: same butterfly order as the other K1
        // variants with W lanes (j ^ W/2 first, ..., j ^ 1 last)
#pragma unroll
        for (int o = 16; o >= VPW; o >>= 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q) f[q] += __shfl_xor_sync(0xffffffffu, f[q], o);
#pragma unroll
            for (int q = 0; q < 6; ++q) H[q] += __shfl_xor_sync(0xffffffffu, H[q], o);
        }
        if constexpr (DEF > 1) {
            if (UM) {  // the vertex's first entry (position 0) is on lane j = 0
                dsc = __shfl_sync(0xffffffffu, dsc, vi);
                opd = __shfl_sync(0xffffffffu, opd, vi);
            }
            if (UM) {
                H[0] = H[0] + svv;
                H[3] = H[3] + svv;
                H[5] = H[5] + svv;
            }
            vertex_terms<R>(f, H, dx, xi, y4.x, y4.y, y4.z, y4.w, UM, dsc, opd);
            if (j == tc) {
#pragma unroll
                for (int q = 0; q < 3; ++q) qf[q] = f[q];
#pragma unroll
                for (int q = 0; q < 6; ++q) qH[q] = H[q];
                qv = act ? hv0 + lv : -1;
                qx = xi4;
            }
            if (++tc == DEF) {
                tc = 0;
                flush();
            }
        } else if (act && j == 0) {  // j = 0 processed the vertex's first entry (UM: dsc/opd)
            const int v = hv0 + lv;
            if (UM) {
                H[0] = H[0] + svv;
                H[3] = H[3] + svv;
                H[5] = H[5] + svv;
            }
            vertex_terms<R>(f, H, dx, xi, y4.x, y4.y, y4.z, y4.w, UM, dsc, opd);  // no entries: dsc = opd = 0, H = 0
            R d[3];
            block_solve<R>(f, H, a.eps_det, a.mode, d);
            R4 nx = xi4;
            nx.x = xi[0] + d[0];
            nx.y = xi[1] + d[1];
            nx.z = xi[2] + d[2];
            k1t_store<R>(a, v, nx);
        }
        if (++stage == S) {
            stage = 0;
            ph ^= 1;
        }
    }
    if constexpr (DEF > 1) flush();
    if constexpr (CLS) {
        for (; t < ta.tcount; t += gridDim.x) {
            mbar_wait_parity(smem_u32(&full[stage]), ph);
            const unsigned char* st = stages + stage * L.stage_bytes();
            const TileHdr* hp = reinterpret_cast<const TileHdr*>(st + L.off_hdr());
            const int cw = hp->wr[7], hv0 = hp->v0, hnv = hp->nv, sbw = hp->wr[warp] >> 16;
            const int lq = warp * 32 + lane;
            const bool act = lq < hnv;
            const int lc = act ? lq : 0;
            if (warp * 32 < hnv) {  // (a warp without vertices has no slots)
                const R4 xi4 = reinterpret_cast<const R4*>(st + L.off_x())[lc];
                R4 xt4, y4;
                R svv = R(0);
                if constexpr (CL) {  // issued before the sweep (used after it)
                    ldg_nc(a.xt + hv0 + lc, xt4);
                    ldg_nc(a.y + hv0 + lc, y4);
                    svv = ldg_nc(a.vsv + hv0 + lc);
                } else {
                    xt4 = reinterpret_cast<const R4*>(st + L.off_xt())[lc];
                    y4 = reinterpret_cast<const R4*>(st + L.off_y())[lc];
                    svv = a.vsv[hv0 + lc];
                }
                const unsigned char* recs = smem + (cw >> 16);
                AccXY acc[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[b].zero();
                const float2 nxy = make_float2(-(float)xi4.x, -(float)xi4.y);
                const float nz = -(float)xi4.z;
                const unsigned char* slots = st + L.off_ent() + 8 * (32 * sbw + lane);
                const unsigned char* npos = st + L.off_npos();
                if (ta.dbg == 1) {  // (timing experiment: no sweep)
                } else if ((cw & 0xff) == 1) class_sweep<0>(slots, npos, recs, nxy, nz, acc);
                else class_sweep<1>(slots, npos, recs, nxy, nz, acc);
                const float4 c4 = reinterpret_cast<const float4*>(recs)[4];  // position 0: (t7, t8, dsc, opd)
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));  // stage's smem no longer read
                R f[3] = {(acc[0].f01.x + acc[2].f01.x) + (acc[1].f01.x + acc[3].f01.x),
                          (acc[0].f01.y + acc[2].f01.y) + (acc[1].f01.y + acc[3].f01.y),
                          (acc[0].f2 + acc[2].f2) + (acc[1].f2 + acc[3].f2)};
                R H[6] = {(acc[0].h03.x + acc[2].h03.x) + (acc[1].h03.x + acc[3].h03.x),
                          (acc[0].h1 + acc[2].h1) + (acc[1].h1 + acc[3].h1),
                          (acc[0].h24.x + acc[2].h24.x) + (acc[1].h24.x + acc[3].h24.x),
                          (acc[0].h03.y + acc[2].h03.y) + (acc[1].h03.y + acc[3].h03.y),
                          (acc[0].h24.y + acc[2].h24.y) + (acc[1].h24.y + acc[3].h24.y),
                          (acc[0].h5 + acc[2].h5) + (acc[1].h5 + acc[3].h5)};
                if (act) {
                    H[0] = H[0] + svv;
                    H[3] = H[3] + svv;
                    H[5] = H[5] + svv;
                    const R xi[3] = {xi4.x, xi4.y, xi4.z};
                    const R dx[3] = {xi[0] - xt4.x, xi[1] - xt4.y, xi[2] - xt4.z};
                    vertex_terms<R>(f, H, dx, xi, y4.x, y4.y, y4.z, y4.w, UM, (R)c4.z, (R)c4.w);
                    R d[3];
                    block_solve<R>(f, H, a.eps_det, a.mode, d);
                    R4 nx = xi4;
                    nx.x = xi[0] + d[0];
                    nx.y = xi[1] + d[1];
                    nx.z = xi[2] + d[2];
                    k1t_store<R>(a, hv0 + lq, nx);
                }
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
            }
            if (++stage == S) {
                stage = 0;
                ph ^= 1;
            }
        }
    }
}
