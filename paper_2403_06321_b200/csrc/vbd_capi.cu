// vbd_capi.cu -- the C ABI (include/vbd_b200.h): device context, scene packing, the
// CUDA-graph step pipeline and the protocol-compatible colour pass.
#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/vbd_b200.h"
#include "vbd_build.cuh"
#include "vbd_common.cuh"
#include "vbd_kernels.cuh"
#include "vbd_tiles.cuh"
#include "vbd_contact.cuh"
#include "vbd_resident.cuh"

// K1 launch variant (lanes per vertex W, entries per lane per iteration U, min blocks/SM);
// selected per context from VBD_K1 (e.g. "8x1", "4x2", "4x2b3"), default below.
struct K1Variant {
    int W = 4, U = 2, minb = 3, pf = 1;
};
K1Variant k1_variant_from_env()
{
    K1Variant v;
    const char* e = getenv("VBD_K1");
    if (e && *e) {
        int w = 0, u = 0, b = 0, p = 0;
        int n = sscanf(e, "%dx%db%dp%d", &w, &u, &b, &p);
        if (n >= 2) { v.W = w; v.U = u; v.minb = n >= 3 ? b : 1; v.pf = n >= 4 ? p : 0; }
    }
    return v;
}

namespace {

thread_local std::string g_err;

struct VbdError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw VbdError{code, m}; }

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            fail(VBD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + \
                                   __FILE__ + ":" + std::to_string(__LINE__) + ")");      \
    } while (0)

// NVTX ranges (header-only nvtx3; free when no tool is attached).  Host-driven paths mark
// every step / iteration / colour pass; the graph path marks each step's graph launch.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    template <typename... A> Nvtx(const char* fmt, A... a)
    {
        char buf[96];
        snprintf(buf, sizeof buf, fmt, a...);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

template <typename F> int guarded(F&& f)
{
    try {
        f();
        return VBD_OK;
    } catch (const VbdError& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return VBD_ERR_INTERNAL;
    }
}

inline unsigned blocks_for(long long n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

// owning device buffer
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;  // pooled buffers: the stream they were allocated (and are freed) on
    bool pooled = false;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void alloc(size_t b)
    {
        release();
        if (b == 0) b = 16;
        CK(cudaMalloc(&p, b));
        bytes = b;
    }
    // stream-ordered allocation from the device's memory pool (no device-wide synchronisation
    // on allocate / free; for the many short-lived scratch buffers of contact detection, sorts
    // and scans)
    void alloc_on(size_t b, cudaStream_t s)
    {
        release();
        if (b == 0) b = 16;
        CK(cudaMallocAsync(&p, b, s));
        bytes = b;
        st = s;
        pooled = true;
    }
    void release()
    {
        if (p) {
            if (pooled) cudaFreeAsync(p, st);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
        pooled = false;
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
    void swap(DBuf& o)
    {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(st, o.st);
        std::swap(pooled, o.pooled);
    }
};

inline int EntryPlanesBytes(int precision) { return precision == VBD_PREC_F64 ? 96 : 48; }

template <typename T> void upload(DBuf& b, const T* host, size_t n, cudaStream_t s)
{
    b.alloc(n * sizeof(T));
    if (n) CK(cudaMemcpyAsync(b.p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

// the same into a stream-ordered pooled buffer (per-step scratch: no cudaMalloc / cudaFree,
// whose free synchronises the whole device)
template <typename T> void upload_on(DBuf& b, const T* host, size_t n, cudaStream_t s)
{
    b.alloc_on(n * sizeof(T), s);
    if (n) CK(cudaMemcpyAsync(b.p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

struct MaterialKey {
    double mu, lam, kd, density;
    bool operator<(const MaterialKey& o) const
    {
        return std::tie(mu, lam, kd, density) < std::tie(o.mu, o.lam, o.kd, o.density);
    }
};

struct GraphKey {
    vbd_step_params p;
    bool operator==(const GraphKey& o) const { return std::memcmp(&p, &o.p, sizeof p) == 0; }
};

}  // namespace

// Pageable host arrays (ordinary numpy) cross PCIe through two pinned staging chunks: host
// threads copy chunk k + 1 into one while the DMA engine moves chunk k out of the other, so the
// copy runs near the pinned rate instead of the driver's pageable path (~11 GB/s measured).
// Page-locked caller arrays go straight to cudaMemcpyAsync.
struct HostStager {
    static constexpr size_t CHUNK = (size_t)64 << 20;
    void* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~HostStager()
    {
        for (int b = 0; b < 2; ++b) {
            if (pin[b]) cudaFreeHost(pin[b]);
            if (ev[b]) cudaEventDestroy(ev[b]);
        }
    }
    bool ready()
    {
        if (pin[0]) return true;
        for (int b = 0; b < 2; ++b) {
            if (cudaMallocHost(&pin[b], CHUNK) != cudaSuccess) {
                cudaGetLastError();
                pin[b] = nullptr;
                return false;
            }
            if (cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess) return false;
        }
        return true;
    }
};

struct vbd_ctx {
    // first member, destroyed last: pooled buffers are freed on this stream by their destructors
    struct OwnedStream {
        cudaStream_t s = nullptr;
        ~OwnedStream()
        {
            if (s) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        }
    } owned;
    int device = 0;
    int precision = VBD_PREC_F32;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    long long n = 0, nsolve = 0, nfree_all = 0, T = 0, E = 0;
    int ncolors = 0;
    std::vector<long long> cbeg, ccnt;
    // slab halo blocks: bnd_cnt[side][c] solved boundary vertices at the head of colour c's
    // range (side 0 first), ghost_beg/ghost_cnt[side][c] the ghost block of colour c
    std::vector<long long> bnd_cnt[2], ghost_beg[2], ghost_cnt[2];
    bool inplace = true;
    std::vector<MaterialKey> mats;
    double mat_h = NAN;
    HostStager hstage;  // pageable host arrays <-> the device stage buffer
    DBuf perm, inv, eoff, ent, mat, pos, xt, vt, vprev, y, ha, hb, mass, out, group, stage,
        flag, stepctr, color_orig;
    std::vector<BeamDev> beams;
    DBuf beams_dev;
    std::vector<int> hinv;  // host copy of inv (protocol colour pass)
    std::vector<int> hperm; // host copy of perm (contact sets)
    K1Variant k1 = k1_variant_from_env();
    // P2P slab halo: flags[0..1] written by the neighbours, [2] epoch, [3] error word
    DBuf p2p_flags;
    void* peer_pos[2] = {nullptr, nullptr};
    unsigned long long* peer_flag_slot[2] = {nullptr, nullptr};
    std::vector<long long> peer_ghost_beg[2];
    cudaGraphExec_t p2p_gexec = nullptr;
    GraphKey p2p_key{};
    DBuf omega_dev;
    DBuf vmat;
    bool uniform_mat = false;
    // compact layout: ent holds int4 entries, kinds the KindRec table (refreshed with the
    // materials), kind_keys the exact rest data of each kind
    bool compact = false;
    int nkinds = 0;
    int max_deg = 0;
    DBuf kinds, kind_keys;
    // fp32 displacement state: position-like vectors (x, x_t, y, Chebyshev history)
    // are stored as x - X with the rest positions X kept in double (rest, colour-major); the
    // kernels add the kinds' rest edges (kedge, 3 float4 per kind + a zero record)
    bool disp = false;
    DBuf rest, kedge;
    // non-tet terms (springs, world box, subspace): host-built systems only; global K1
    bool has_extras = false;
    DBuf soff, sp_oth, sp_par, box, sub_idx, sub;
    // contact set (vbd_set_contacts, or the device detection below; 0 = none)
    long long ncontacts = 0;
    double mu_c = 0.0, eps_v = 1e-2;
    DBuf coff, ccid, cslot, cidx, creal;
    // device contact detection for step() (vbd_set_collision): surface primitives
    // (colour-major ids, original order), per-vertex active mask, sticky colliding flags, the
    // DCD records of the step (and their codes) and the CCD records of the last pass
    bool coll_on = false;
    DBuf csv, ctri, cedge, cactive, ccoll, dcd_recs, dcd_codes, ccd_recs;
    int nsv = 0, ntri = 0, nedge = 0;
    long long ndcd = 0, nccd = 0;
    double coll_cell = 1.0, coll_kc = 1.0, coll_dcd_r = 1e-3, coll_max_depth = 0.0;
    int coll_has_max_depth = 0, coll_ncol = 4;
    // graph-mode contact step (step_contacts_graph): capacities sized from the largest counts
    // seen on the host-synchronised path (mx_*), sentinel-padded buffers, one graph per step
    long long mx_cell[3] = {0, 0, 0}, mx_join[2] = {0, 0};
    long long cap_cell[3] = {0, 0, 0}, cap_join[2] = {0, 0};
    bool cg_ready = false, cg_pending = false;
    bool cg_enabled = true;  // VBD_CONTACT_GRAPH=0 at context creation: host path only
    long long cg_steps = 0;
    int cg_fallbacks = 0;  // steps redone on the host path after a capacity overflow
    cudaGraphExec_t cg_exec = nullptr;
    GraphKey cg_key{};
    DBuf cg_cnt, cg_off, cg_key_q, cg_own_q, cg_key_t, cg_own_t, cg_jcnt, cg_joff, cg_codes, cg_codes2,
        cg_nsel, cg_recs, cg_acc, cg_aoff, cg_tmp, cg_dcd_codes, cg_vt, cg_ee, cg_all, cg_inc, cg_inc2, cg_flag,
        cg_snap;
    // K1T tile pipeline (compact layout, in-place range passes): tiles of 64 vertices per
    // colour, their neighbour lists and 8-byte entries
    bool tiles = false;
    std::vector<int> tile_beg;  // first tile of colour c (size ncolors + 1)
    int ent_cap = 0, nbr_cap = 0;
    DBuf tv0, tnv, loff, tnbr, tent, tdesc;
    DBuf vsv;  // per solved vertex: sum of V mu |w|^2 over its entries (one material per vertex)
    int tile_stages = 2, tile_w = 4, tile_occ = 2;
    bool tile_defer = true;  // K1T deferred block solves (VBD_TILE_DEFER=0 disables)
    bool tile_kg = false;    // K1T kind records read from global (table too large for shared memory)
    // K1T-X (explicit layout, fp32, one material per vertex): the tiles' slots carry no kind;
    // each slot's 9 slot-weight rows stream from xrows (9 planes of `slots` floats, slot order)
    // and the per-entry constants and rest edges are derived on the fly (as the explicit K1 does)
    bool tile_xr = false;
    int tile_vpt = 64;  // K1T vertices per tile (64, or 32 for small scenes)
    // K1T class tiles (fp32 grids, vbd_grid_classes.cuh): the solved vertices of one grid-class
    // instance (class + the kinds at every entry position) form one run per colour
    struct ClassRun {
        long long beg, cnt;
        int inst;
    };
    std::vector<ClassRun> crun;
    std::vector<int> cinst_tpl;  // class of instance i
    int tile_svpt = 64;          // stage capacity for x / x_t / y (128 with class tiles)
    bool tile_xtg = false;       // class tiles: x_t / y not staged (read by the consumers)
    int ncrec = 0;               // class records after the kind table's zero record
    DBuf ckind;                  // kind id of every class record
    long long class_vertices = 0;
    int class_tiles = 0;
    std::vector<int> tile_cls_beg;  // first class tile of colour c (after its plain tiles)
    DBuf xrows;
    // K1R resident whole-step kernel (small scenes): 0 off, 1 REPL (one cluster, position
    // replicas in shared memory), 2 GLOB (one CTA per SM, grid barrier); -1 not decided yet
    int res_mode = -1;
    std::string res_want;  // VBD_RESIDENT at context creation
    int res_ncta = 0, res_slot_cap = 0, res_grp_cap = 0;
    size_t res_smem = 0;
    DBuf res_slots, res_slot_beg, res_groups, res_grp_beg, res_col_grp, res_bar, res_push, res_prof;
    // step state for the fine-grained path
    vbd_step_params cur{};
    std::vector<double> omegas;
    bool in_step = false;
    // graph cache
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey{};
    // halo lists: [side][color] -> device ids
    std::vector<std::vector<long long>> halo_send_cnt[2], halo_recv_cnt[2];
    std::vector<std::vector<DBuf*>> halo_send[2], halo_recv[2];
    ~vbd_ctx()
    {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (p2p_gexec) cudaGraphExecDestroy(p2p_gexec);
        if (cg_exec) cudaGraphExecDestroy(cg_exec);
        for (int s = 0; s < 2; ++s) {
            for (auto& v : halo_send[s])
                for (auto* b : v) delete b;
            for (auto& v : halo_recv[s])
                for (auto* b : v) delete b;
        }
        if (stream) cudaStreamSynchronize(stream);  // own_stream is destroyed by `owned`, last
    }
    size_t r4() const { return precision == VBD_PREC_F64 ? 32 : 16; }
    size_t rs() const { return precision == VBD_PREC_F64 ? 8 : 4; }
};

namespace {

// ---------------------------------------------------------------------------------------
// CUB helpers

void sort_pairs_i32(DBuf& keys, DBuf& vals, long long n, int end_bit, cudaStream_t s)
{
    DBuf k2, v2, tmp;
    k2.alloc(n * 4);
    v2.alloc(n * 4);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<int>(), k2.as<int>(),
                                       vals.as<unsigned>(), v2.as<unsigned>(), (int64_t)n, 0,
                                       end_bit, s));
    tmp.alloc(tb);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<int>(), k2.as<int>(),
                                       vals.as<unsigned>(), v2.as<unsigned>(), (int64_t)n, 0,
                                       end_bit, s));
    CK(cudaStreamSynchronize(s));
    std::swap(keys.p, k2.p);
    std::swap(keys.bytes, k2.bytes);
    std::swap(vals.p, v2.p);
    std::swap(vals.bytes, v2.bytes);
}

void sort_pairs_u64_i32(DBuf& keys, DBuf& vals, long long n, cudaStream_t s)
{
    DBuf k2, v2, tmp;
    k2.alloc_on(n * 8, s);
    v2.alloc_on(n * 4, s);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<unsigned long long>(),
                                       k2.as<unsigned long long>(), vals.as<int>(), v2.as<int>(),
                                       (int64_t)n, 0, 64, s));
    tmp.alloc_on(tb, s);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<unsigned long long>(),
                                       k2.as<unsigned long long>(), vals.as<int>(), v2.as<int>(),
                                       (int64_t)n, 0, 64, s));
    CK(cudaStreamSynchronize(s));
    keys.swap(k2);
    vals.swap(v2);
}

void sort_keys_u64(DBuf& keys, long long n, cudaStream_t s)
{
    DBuf k2, tmp;
    k2.alloc_on(n * 8, s);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<unsigned long long>(),
                                      k2.as<unsigned long long>(), (int64_t)n, 0, 64, s));
    tmp.alloc_on(tb, s);
    CK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.as<unsigned long long>(),
                                      k2.as<unsigned long long>(), (int64_t)n, 0, 64, s));
    CK(cudaStreamSynchronize(s));
    keys.swap(k2);
}

// out[0] = 0, out[i+1] = sum(in[0..i]); in has n entries of type In
template <typename In>
void exclusive_offsets(const In* in, long long n, DBuf& out, cudaStream_t s)
{
    out.alloc_on((n + 1) * sizeof(long long), s);
    CK(cudaMemsetAsync(out.p, 0, sizeof(long long), s));
    if (n == 0) return;
    DBuf tmp;
    size_t tb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out.as<long long>() + 1, (int64_t)n, s));
    tmp.alloc_on(tb, s);
    CK(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out.as<long long>() + 1, (int64_t)n, s));
    CK(cudaStreamSynchronize(s));
}

template <typename T> T read_scalar(const void* dptr, cudaStream_t s)
{
    T v;
    CK(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
}

// ---------------------------------------------------------------------------------------
// scene intermediate (device, original numbering) consumed by the packer

struct Scene {
    long long n = 0, T = 0;
    DBuf tets;      // int32 (T,4)
    DBuf tet_w;     // f64 (T,12)
    DBuf vol;       // f64 (T)
    DBuf tmat;      // int32 (T)
    DBuf inc_off;   // int64 (n+1)
    DBuf inc;       // u32 (4T) = 4 t + s, ascending per vertex
    DBuf mass;      // f64 (n)
    DBuf kind;      // u8 (n): 0 free, 1 fixed, 3 ghost
    DBuf halo;      // u8 (n) slab role (k_order_keys), or empty
    DBuf color;     // int32 (n)
    DBuf pos;       // f64 (n,3) rest positions (drives the spatial order) or empty
    double bbox_lo[3] = {0.0, 0.0, 0.0};
    double bbox_scale = 0.0;  // 2^21 - 1 over the largest bbox extent
    void set_bbox(const double lo[3], const double hi[3])
    {
        double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
        for (int k = 0; k < 3; ++k) bbox_lo[k] = lo[k];
        bbox_scale = ext > 0 ? 2097151.0 / ext : 0.0;
    }
};

void build_incidence(Scene& sc, cudaStream_t s)
{
    long long n4 = 4 * sc.T;
    DBuf keys, vals, cnt;
    keys.alloc(n4 * 4);
    vals.alloc(n4 * 4);
    cnt.alloc(sc.n * 4);
    CK(cudaMemsetAsync(cnt.p, 0, sc.n * 4, s));
    if (n4) k_inc_keys<<<blocks_for(n4), 256, 0, s>>>(sc.tets.as<int>(), n4, keys.as<int>(),
                                                     vals.as<unsigned>(), cnt.as<int>());
    CK(cudaGetLastError());
    int bits = 1;
    while ((1LL << bits) < sc.n) ++bits;
    if (n4) sort_pairs_i32(keys, vals, n4, bits, s);
    exclusive_offsets(cnt.as<int>(), sc.n, sc.inc_off, s);
    std::swap(sc.inc.p, vals.p);
    std::swap(sc.inc.bytes, vals.bytes);
}

// K5 on a device neighbour CSR; colour (int32, n) out
int run_jp(const long long* noff, const int* nids, const long long* rank, long long n,
           int* color, cudaStream_t s)
{
    if (n == 0) return 0;
    DBuf pending, fa, fb, cnts, colored, overflow;
    pending.alloc(n * 4);
    fa.alloc(n * 4);
    fb.alloc(n * 4);
    cnts.alloc(2 * sizeof(int));
    colored.alloc(8);
    overflow.alloc(4);
    CK(cudaMemsetAsync(cnts.p, 0, 2 * sizeof(int), s));
    CK(cudaMemsetAsync(colored.p, 0, 8, s));
    CK(cudaMemsetAsync(overflow.p, 0, 4, s));
    int* cnt = cnts.as<int>();
    k_jp_init<<<blocks_for(n), 256, 0, s>>>(noff, nids, rank, n, pending.as<int>(), color,
                                            fa.as<int>(), cnt);
    CK(cudaGetLastError());
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int* fin = fa.as<int>();
    int* fout = fb.as<int>();
    int cin = 0, cout = 1;
    long long rounds = 0;
    for (;;) {
        CK(cudaMemsetAsync(cnt + cout, 0, sizeof(int), s));
        k_jp_round<<<sms * 4, 256, 0, s>>>(noff, nids, rank, fin, cnt + cin, pending.as<int>(),
                                           color, fout, cnt + cout,
                                           colored.as<unsigned long long>(), overflow.as<int>());
        std::swap(fin, fout);
        std::swap(cin, cout);
        ++rounds;
        if ((rounds & 15) == 0 || rounds < 4) {
            CK(cudaGetLastError());
            unsigned long long done = read_scalar<unsigned long long>(colored.p, s);
            if ((long long)done >= n) break;
            int next = read_scalar<int>(cnt + cin, s);
            if (next == 0) fail(VBD_ERR_INTERNAL, "colouring stalled (inconsistent CSR?)");
        }
        if (rounds > 4 * n + 64) fail(VBD_ERR_INTERNAL, "colouring did not terminate");
    }
    if (read_scalar<int>(overflow.p, s)) fail(VBD_ERR_UNSUPPORTED, "more than 256 colours");
    return 0;
}

// neighbour CSR from the incidence, then K5
void color_scene(Scene& sc, cudaStream_t s)
{
    Nvtx nv_("colouring (K5)");
    DBuf cnt, overflow, noff, nids;
    cnt.alloc(sc.n * 4);
    overflow.alloc(4);
    CK(cudaMemsetAsync(overflow.p, 0, 4, s));
    k_nbr_count<<<blocks_for(sc.n, 128), 128, 0, s>>>(sc.inc_off.as<long long>(),
                                                       sc.inc.as<unsigned>(), sc.tets.as<int>(),
                                                       sc.n, cnt.as<int>(), overflow.as<int>());
    CK(cudaGetLastError());
    if (read_scalar<int>(overflow.p, s))
        fail(VBD_ERR_UNSUPPORTED, "vertex with more than 128 incident tets");
    exclusive_offsets(cnt.as<int>(), sc.n, noff, s);
    long long nn = read_scalar<long long>(noff.as<long long>() + sc.n, s);
    nids.alloc(nn * 4);
    k_nbr_fill<<<blocks_for(sc.n, 128), 128, 0, s>>>(sc.inc_off.as<long long>(),
                                                      sc.inc.as<unsigned>(), sc.tets.as<int>(),
                                                      sc.n, noff.as<long long>(), nids.as<int>());
    CK(cudaGetLastError());
    sc.color.alloc(sc.n * 4);
    run_jp(noff.as<long long>(), nids.as<int>(), nullptr, sc.n, sc.color.as<int>(), s);
}

template <typename R> void alloc_state(vbd_ctx* c)
{
    size_t b = c->n * c->r4();
    for (DBuf* d : {&c->pos, &c->xt, &c->vt, &c->vprev, &c->y, &c->ha, &c->hb, &c->out}) {
        d->alloc(b);
        CK(cudaMemsetAsync(d->p, 0, b, c->stream));
    }
    c->stage.alloc(std::max<long long>(c->n, 1) * 3 * sizeof(double));
    c->flag.alloc(8);
    c->stepctr.alloc(4);
    CK(cudaMemsetAsync(c->stepctr.p, 0, 4, c->stream));
}

// Lossless entry dictionary (compact layout): when the explicit entries hold at
// most VBD_KIND_CAP distinct (rows, volume, material) keys, re-pack them as int4
// {n0, n1, n2, kind} and keep one record per kind.  VBD_LAYOUT=explicit disables it.
template <typename R> void compact_entries(vbd_ctx* c)
{
    cudaStream_t s = c->stream;
    c->compact = false;
    c->nkinds = 0;
    const char* lay = getenv("VBD_LAYOUT");
    if ((lay && !strcmp(lay, "explicit")) || c->E == 0) return;
    const char* capenv = getenv("VBD_KIND_CAP");
    const int cap = capenv && *capenv ? atoi(capenv) : (1 << 16);
    unsigned nslots = 1;
    while (nslots < 4u * (unsigned)cap) nslots <<= 1;
    DBuf slots, cnt;
    slots.alloc((size_t)nslots * 8);
    cnt.alloc(16);  // [0] count, [1] overflow, [2] missing
    CK(cudaMemsetAsync(slots.p, 0, (size_t)nslots * 8, s));
    CK(cudaMemsetAsync(cnt.p, 0, 16, s));
    typedef typename PlaneT<R>::T PL;
    const PL* pl = c->ent.as<PL>();
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const unsigned grid = (unsigned)std::min<long long>(blocks_for(c->E), 16LL * sms);
    k_kind_insert<R><<<grid, 256, 0, s>>>(pl, c->E, slots.as<unsigned long long>(), nslots - 1,
                                          cnt.as<int>(), cap, cnt.as<int>() + 1);
    CK(cudaGetLastError());
    int hc[3];
    CK(cudaMemcpyAsync(hc, cnt.p, 12, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hc[1] || hc[0] > cap) return;  // too many distinct kinds: keep the explicit layout
    // kind ids in slot order (deterministic given the table)
    std::vector<unsigned long long> hs(nslots);
    CK(cudaMemcpy(hs.data(), slots.p, (size_t)nslots * 8, cudaMemcpyDeviceToHost));
    std::vector<int> slot_kind(nslots, -1);
    std::vector<long long> rep;
    for (unsigned i = 0; i < nslots; ++i)
        if (hs[i]) {
            slot_kind[i] = (int)rep.size();
            rep.push_back((long long)hs[i] - 1);
        }
    const int nk = (int)rep.size();
    DBuf dsk, drep, cent;
    upload(dsk, slot_kind.data(), nslots, s);
    upload(drep, rep.data(), rep.size(), s);
    c->kind_keys.alloc((size_t)nk * KindKey<R>::KW * 4);
    k_kind_keys<R><<<blocks_for(nk), 256, 0, s>>>(pl, c->E, drep.as<long long>(), nk, c->kind_keys.as<unsigned>());
    CK(cudaGetLastError());
    cent.alloc((size_t)c->E * 16);
    k_kind_emit<R><<<grid, 256, 0, s>>>(pl, c->E, slots.as<unsigned long long>(), nslots - 1,
                                        dsk.as<int>(), cent.as<int4>(), cnt.as<int>() + 2);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hc, cnt.p, 12, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hc[2]) fail(VBD_ERR_INTERNAL, "entry dictionary lookup failed");
    c->ent.swap(cent);  // the explicit planes are released with `cent`
    // nk records + one zero record (index nk: the padding slots of K1T with global kinds)
    c->kinds.alloc((size_t)(nk + 1) * KindRec<R>::Q * 16);
    CK(cudaMemsetAsync(c->kinds.p, 0, (size_t)(nk + 1) * KindRec<R>::Q * 16, s));
    c->compact = true;
    c->nkinds = nk;
    if constexpr (sizeof(R) == 4) {  // rest edges per kind (+ the zero record at index nk)
        c->kedge.alloc((size_t)(nk + 1) * 48);
        CK(cudaMemsetAsync(c->kedge.p, 0, (size_t)(nk + 1) * 48, s));
        k_kind_edges<<<blocks_for(nk), 256, 0, s>>>(c->kind_keys.as<unsigned>(), nk, c->kedge.as<float4>());
        CK(cudaGetLastError());
    }
}

// kind records for the current material table
template <typename R> void refresh_kinds(vbd_ctx* c)
{
    if (!c->compact) return;
    k_kind_records<R><<<blocks_for(c->nkinds), 256, 0, c->stream>>>(
        c->kind_keys.as<unsigned>(), c->nkinds, c->mat.as<Material<R>>(), c->kinds.as<typename PlaneT<R>::T>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
}

// K1T tiles (vbd_tiles.cuh): 64 consecutive vertices of one colour, the sorted distinct
// neighbours they read and their entries re-encoded against that list.  Needs the compact
// layout, a valid colouring (in-place sweeps) and shared memory for two stages.
constexpr size_t VBD_TILE_SMEM_MAX = 112 * 1024;  // two CTAs per SM

template <typename R> void build_tiles(vbd_ctx* c)
{
    Nvtx nv_("tile build");
    c->tiles = false;
    const char* e = getenv("VBD_TILES");
    c->tile_xr = false;
    const char* xe = getenv("VBD_TILES_X");
    const bool xr = !c->compact && sizeof(R) == 4 && c->disp && c->uniform_mat && !(xe && *xe == '0');
    if ((e && *e == '0') || !(c->compact || xr) || !c->inplace || c->nsolve == 0 || c->nkinds >= 65535 ||
        c->has_extras)
        return;
    const char* we = getenv("VBD_TILE_W");
    const int W = we && *we ? atoi(we) : 2;  // 2 lanes x 16 vertices per warp measured fastest
    if (W != 4 && W != 2) fail(VBD_ERR_ARG, "VBD_TILE_W: 4 or 2 lanes per vertex are compiled");
    // vertices per tile: 64 (2 W consumer warps x 32 / W); 32 when the largest colour would not
    // fill the SMs twice over with 64-vertex tiles (small scenes; W = 2 only)
    long long cmax = 0;
    for (int col = 0; col < c->ncolors; ++col) cmax = std::max(cmax, c->ccnt[col]);
    int dev_ = 0, sms_ = 148;
    CK(cudaGetDevice(&dev_));
    CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_));
    const char* tve = getenv("VBD_TILE_V");
    const char* kg_e = getenv("VBD_TILE_KG");
    const char* de_e = getenv("VBD_TILE_DEFER");
    const bool small_ok = W == 2 && !xr && (long long)(c->nkinds + 1) * TileSmem<R>::KSTRIDE <= 32768 &&
                          !(kg_e && *kg_e == '1') && !(de_e && *de_e == '0');
    const int VPT = small_ok && (tve && *tve ? atoi(tve) == 32 : cmax < 64LL * 2 * sms_) ? 32 : 64;
    c->tile_vpt = VPT;
    if ((long long)VPT * c->max_deg * 3 > VBD_TILE_SORT) return;
    c->tile_w = W;
    cudaStream_t s = c->stream;
    // K1T class tiles (fp32 displacement state, one material per vertex, 2-lane 64-vertex tiles):
    // the runs of grid-class instances (pack) are cut into 128-vertex tiles of one lane per
    // vertex whose slots are the vertices' neighbour offsets in class order (k_class_pseudo)
    const char* cle = getenv("VBD_TILE_CLASS");
    const char* kge0 = getenv("VBD_TILE_KG");
    bool cls = sizeof(R) == 4 && c->disp && c->uniform_mat && !xr && W == 2 && VPT == 64 && !c->crun.empty() &&
               !(cle && *cle == '0') && !(kge0 && *kge0 == '1');
    c->ncrec = 0;
    c->class_tiles = 0;
    c->class_vertices = 0;
    if (cls) {  // worth it only when class vertices carry most of the sweep (C3: 25 %, slower)
        long long cv = 0;
        for (const auto& r : c->crun) cv += r.cnt;
        const char* me = getenv("VBD_TILE_CLASS_MIN");
        const double mn = me && *me ? atof(me) : 0.5;
        if ((double)cv < mn * (double)c->nsolve) cls = false;
    }
    std::vector<int> irec;  // first class record of instance i
    if (cls) {
        const int ninst = (int)c->cinst_tpl.size();
        std::vector<int> ck;
        for (int i = 0; i < ninst && cls; ++i) {
            irec.push_back((int)ck.size());
            const int ne = vbd_gc_ne_host[c->cinst_tpl[i]];
            long long vb = -1;
            for (const auto& r : c->crun)
                if (r.inst == i) {
                    vb = r.beg;
                    break;
                }
            if (vb < 0) {  // an instance without solved vertices (fixed only): no records needed
                for (int q = 0; q < ne; ++q) ck.push_back((int)c->nkinds);
                continue;
            }
            const long long e0 = read_scalar<long long>(c->eoff.as<long long>() + vb, s);
            std::vector<int4> ents(ne);
            CK(cudaMemcpy(ents.data(), c->ent.as<int4>() + e0, ne * sizeof(int4), cudaMemcpyDeviceToHost));
            for (int q = 0; q < ne; ++q) ck.push_back(ents[q].w);
        }
        c->ncrec = (int)ck.size();
        if ((long long)(c->nkinds + 1 + c->ncrec) * TileSmem<R>::KSTRIDE > 32768) cls = false;
        if (cls) upload(c->ckind, ck.data(), ck.size(), s);
        else c->ncrec = 0;
    }
    std::vector<int> v0, nv, tcw, tcol;
    std::vector<signed char> tw;
    int cur_col = 0;
    auto cut = [&](long long from, long long to, int per, int inst) {
        for (long long o = from; o < to; o += per) {
            v0.push_back((int)o);
            nv.push_back((int)std::min<long long>(per, to - o));
            tw.push_back((signed char)(inst >= 0 ? 1 : W));
            tcw.push_back(inst >= 0 ? (c->cinst_tpl[inst] + 1) |
                                          ((int)((c->nkinds + 1 + irec[inst]) * TileSmem<R>::KSTRIDE) << 16)
                                    : 0);
            tcol.push_back(cur_col);
        }
    };
    c->tile_beg.assign(c->ncolors + 1, 0);
    for (int col = 0; col < c->ncolors; ++col) {
        cur_col = col;
        c->tile_beg[col] = (int)v0.size();
        const long long b = c->cbeg[col], e = b + c->ccnt[col];
        long long p = b;
        for (const auto& r : c->crun) {
            if (!cls || r.beg < b || r.beg >= e) continue;
            cut(p, r.beg, VPT, -1);
            cut(r.beg, r.beg + r.cnt, 128, r.inst);
            p = r.beg + r.cnt;
        }
        cut(p, e, VPT, -1);
    }
    // (experiment) interleave the instances' class tiles of each colour in proportion (the
    // 8-entry class is gather-heavy, the 32-entry class sweep-heavy); the order of tiles is free
    // (measured: C5 0.835 -> 1.20 ms per pass -- the warps of an SM then alternate between the
    // two unrolled sweeps and miss in the instruction cache; off unless VBD_TILE_CLASS_MIX=1)
    const char* ile = getenv("VBD_TILE_CLASS_MIX");
    if (cls && ile && *ile == '1') {
        int t0 = 0;
        while (t0 < (int)v0.size()) {
            int t1 = t0;
            while (t1 < (int)v0.size() && tcol[t1] == tcol[t0]) ++t1;
            int cb = t0;
            while (cb < t1 && tcw[cb] == 0) ++cb;
            std::map<int, std::vector<int>> by;  // instance word -> tiles in order
            for (int t = cb; t < t1; ++t) by[tcw[t]].push_back(t);
            if (by.size() > 1) {
                std::vector<std::pair<const std::vector<int>*, size_t>> lists;
                for (auto& kv : by) lists.push_back({&kv.second, 0});
                std::vector<int> order;
                while ((int)order.size() < t1 - cb) {
                    int best = -1;
                    double bf = 2.0;
                    for (int k = 0; k < (int)lists.size(); ++k) {
                        const auto& L = lists[k];
                        if (L.second >= L.first->size()) continue;
                        const double f = (L.second + 0.5) / (double)L.first->size();
                        if (f < bf) {
                            bf = f;
                            best = k;
                        }
                    }
                    order.push_back((*lists[best].first)[lists[best].second++]);
                }
                std::vector<int> a0(order.size()), a1(order.size()), a2(order.size());
                std::vector<signed char> a3(order.size());
                for (size_t i = 0; i < order.size(); ++i) {
                    a0[i] = v0[order[i]];
                    a1[i] = nv[order[i]];
                    a2[i] = tcw[order[i]];
                    a3[i] = tw[order[i]];
                }
                for (size_t i = 0; i < order.size(); ++i) {
                    v0[cb + i] = a0[i];
                    nv[cb + i] = a1[i];
                    tcw[cb + i] = a2[i];
                    tw[cb + i] = a3[i];
                }
            }
            t0 = t1;
        }
    }

    int nt = 0;
    DBuf dtw, dtcw;
    // tile arrays -> device, colour ranges, the class tile split of each colour
    auto commit_tiles = [&]() {
        nt = (int)v0.size();
        c->tile_beg.assign(c->ncolors + 1, nt);
        for (int t = nt - 1; t >= 0; --t) c->tile_beg[tcol[t]] = t;
        for (int col = c->ncolors - 1; col >= 0; --col)  // (colours without tiles)
            if (c->tile_beg[col] > c->tile_beg[col + 1]) c->tile_beg[col] = c->tile_beg[col + 1];
        // per colour: its plain tiles, then its class runs (instances sort after every plain vertex)
        c->tile_cls_beg.assign(c->ncolors, 0);
        c->class_tiles = 0;
        c->class_vertices = 0;
        for (int col = 0; col < c->ncolors; ++col) {
            int t = c->tile_beg[col];
            while (t < c->tile_beg[col + 1] && tcw[t] == 0) ++t;
            c->tile_cls_beg[col] = t;
            for (int u = t; u < c->tile_beg[col + 1]; ++u) {
                if (!tcw[u]) fail(VBD_ERR_INTERNAL, "class tiles: a plain tile after a class run");
                c->class_tiles++;
                c->class_vertices += nv[u];
            }
        }
        upload(c->tv0, v0.data(), v0.size(), s);
        upload(c->tnv, nv.data(), nv.size(), s);
        if (cls) {
            upload(dtw, tw.data(), tw.size(), s);
            upload(dtcw, tcw.data(), tcw.size(), s);
        }
    };
    commit_tiles();
    c->tile_svpt = cls ? 128 : VPT;
    c->tile_xtg = cls;
    DBuf cnt, err;
    cnt.alloc((size_t)nt * 16);
    err.alloc(4);
    CK(cudaMemsetAsync(err.p, 0, 4, s));
    DBuf xids;  // XR: {n0, n1, n2, 0} of every explicit entry (the tile build's input)
    if (xr) {
        xids.alloc((size_t)std::max<long long>(c->E, 1) * 16);
        if (c->E) k_plane_ids<<<blocks_for(c->E), 256, 0, s>>>(c->ent.as<float4>(), c->E, xids.as<int4>());
        CK(cudaGetLastError());
    }
    const int4* cent = xr ? xids.as<int4>() : c->ent.as<int4>();
    const long long* eoffb = c->eoff.as<long long>();
    DBuf eoff2, cent2;  // class tiles: pseudo entries (k_class_pseudo)
    if (cls) {
        DBuf vtpl, vins, deg2, cerr;
        vtpl.alloc(c->nsolve);
        vins.alloc(c->nsolve);
        CK(cudaMemsetAsync(vtpl.p, 0xff, c->nsolve, s));
        CK(cudaMemsetAsync(vins.p, 0xff, c->nsolve, s));
        for (const auto& r : c->crun) {
            CK(cudaMemsetAsync(vtpl.as<char>() + r.beg, c->cinst_tpl[r.inst], r.cnt, s));
            CK(cudaMemsetAsync(vins.as<char>() + r.beg, r.inst, r.cnt, s));
        }
        deg2.alloc(c->nsolve * 8);
        k_class_deg<<<blocks_for(c->nsolve), 256, 0, s>>>(c->eoff.as<long long>(), vtpl.as<signed char>(), c->nsolve,
                                                          deg2.as<long long>());
        CK(cudaGetLastError());
        exclusive_offsets(deg2.as<long long>(), c->nsolve, eoff2, s);
        const long long E2 = read_scalar<long long>(eoff2.as<long long>() + c->nsolve, s);
        cent2.alloc((size_t)std::max<long long>(E2, 1) * 16);
        DBuf direc;
        upload(direc, irec.data(), irec.size(), s);
        cerr.alloc(4);
        CK(cudaMemsetAsync(cerr.p, 0, 4, s));
        k_class_pseudo<<<blocks_for(c->nsolve), 256, 0, s>>>(
            c->eoff.as<long long>(), cent, c->nsolve, vtpl.as<signed char>(), vins.as<signed char>(),
            eoff2.as<long long>(), cent2.as<int4>(), direc.as<int>(), c->ckind.as<int>(), (int)c->nkinds,
            cerr.as<int>());
        CK(cudaGetLastError());
        if (read_scalar<int>(cerr.p, s)) {  // (cannot happen for detected classes) -- plain tiles
            c->crun.clear();
            build_tiles<R>(c);
            return;
        }
        eoffb = eoff2.as<long long>();
        cent = cent2.as<int4>();
    }
    int P = 256;
    while (P < std::max(VPT * c->max_deg, cls ? 128 * VBD_GC_MAXNL : 0) * 3) P <<= 1;
    const size_t sort_smem = (size_t)P * 4;
    CK(cudaFuncSetAttribute(k_tile_nbrs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem));
    CK(cudaFuncSetAttribute(k_tile_nbrs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem));
    // bank-aware placement (k_tile_banks): lists padded by VBD_TILE_BANK_SLACK percent (default
    // 25; 0 keeps the sorted list) to a multiple of the 8 bank groups
    const char* be = getenv("VBD_TILE_BANK_SLACK");
    const int slack = be && *be ? atoi(be) : 25;
    auto padded = [&](long long n) { return slack > 0 ? (n * (100 + slack) / 100 + 8 + 7) / 8 * 8 : n; };
    std::vector<long long> hc;
    const signed char* tWp = nullptr;
    for (int round = 0;; ++round) {
        tWp = cls ? dtw.as<signed char>() : nullptr;
        cnt.alloc((size_t)nt * 16);
        k_tile_nbrs<false><<<nt, 256, sort_smem, s>>>(c->tv0.as<int>(), c->tnv.as<int>(), eoffb,
                                                     cent, cnt.as<long long>(), nullptr, nullptr, nullptr, nullptr, W,
                                                     0u, 0u, 0u, 0u, err.as<int>(), nullptr, tWp);
        CK(cudaGetLastError());
        if (read_scalar<int>(err.p, s)) return;
        hc.assign(2 * (size_t)nt, 0);
        CK(cudaMemcpy(hc.data(), cnt.p, (size_t)nt * 16, cudaMemcpyDeviceToHost));
        if (!cls || round == 4) break;
        // class tiles whose neighbour list would keep two stages from fitting 3 CTAs per SM are
        // cut in two (C4's small cubes: a class run spans several cubes)
        long long ms0 = 0;
        for (int t = 0; t < nt; ++t) ms0 = std::max(ms0, hc[2 * t + 1]);
        const long long fixed = ((long long)(c->nkinds + 1 + c->ncrec) * TileSmem<R>::KSTRIDE + 127) / 128 * 128 +
                                2 * ((long long)sizeof(TileDesc) + ms0 * 8 + 128LL * (long long)sizeof(typename Vec4<R>::T) + 256);
        const long long budget = (75 * 1024 - fixed) / 2 / (long long)TileSmem<R>::PU - 1;
        std::vector<int> v0b, nvb, tcwb, tcolb;
        std::vector<signed char> twb;
        bool any = false;
        for (int t = 0; t < nt; ++t) {
            const bool split = tcw[t] && nv[t] > 32 && padded(hc[2 * t]) > budget;
            const int h = split ? (nv[t] / 2 + 31) / 32 * 32 : nv[t];
            for (int part = 0; part < (split ? 2 : 1); ++part) {
                v0b.push_back(part ? v0[t] + h : v0[t]);
                nvb.push_back(split ? (part ? nv[t] - h : h) : nv[t]);
                tcwb.push_back(tcw[t]);
                tcolb.push_back(tcol[t]);
                twb.push_back(tw[t]);
            }
            any |= split;
        }
        if (!any) break;
        v0.swap(v0b);
        nv.swap(nvb);
        tcw.swap(tcwb);
        tcol.swap(tcolb);
        tw.swap(twb);
        commit_tiles();
    }
    std::vector<long long> nls(nt), nss(nt);
    std::vector<int> nl_real(nt);
    long long mx = 0, ms = 0;
    for (int t = 0; t < nt; ++t) {
        nl_real[t] = (int)hc[2 * t];
        nls[t] = slack > 0 ? (hc[2 * t] * (100 + slack) / 100 + 8 + 7) / 8 * 8 : hc[2 * t];
        nss[t] = hc[2 * t + 1];
        mx = std::max(mx, nls[t]);
        ms = std::max(ms, nss[t]);
    }
    // slots hold 16-bit shared-memory byte offsets (+1 zero position) and a 16-bit kind: the
    // record's byte offset in the shared-memory table, or (KG: tables over 32 KB, e.g. fp64
    // grids whose rest shapes differ in the last bits) its index in the global table
    constexpr unsigned PU = TileSmem<R>::PU;  // slot offsets address 16-byte position units
    if ((mx + 1) * (long long)PU > 65535) return;
    if (c->nkinds >= 65535) return;
    const char* kge = getenv("VBD_TILE_KG");
    c->tile_kg = !xr && ((long long)(c->nkinds + 1) * TileSmem<R>::KSTRIDE > 32768 || (kge && *kge == '1'));
    if (c->tile_kg && W != 2) return;  // compiled for the 2-lane kernel
    c->nbr_cap = (int)mx;
    c->ent_cap = (int)ms;
    TileSmem<R> L{c->ent_cap, c->nbr_cap, (c->tile_kg || xr) ? -1 : (int)c->nkinds + c->ncrec, c->tile_svpt,
                  c->tile_xtg ? 1 : 3};
    // as many stages (2..4) as fit three CTAs per SM, else two (2-lane: 2 stages)
    const char* oe = getenv("VBD_TILE_OCC");
    c->tile_occ = oe && *oe == '2' ? 2 : 3;  // 3 CTAs per SM (one entry per lane in flight) measured faster
    const bool force_occ3 = oe && *oe == '3';  // (tuning: keep 3 CTAs/SM even above 75 KB)
    const char* de = getenv("VBD_TILE_DEFER");
    c->tile_defer = !(de && *de == '0');
    int stages = 0;
    for (int st = 4; st >= 2 && !stages && c->tile_occ == 3; --st)
        if (L.total(st) <= 75 * 1024 || (force_occ3 && st == 2)) stages = st;
    if (!stages) c->tile_occ = 2;  // e.g. fp64: 32-byte positions
    for (int st = W == 2 ? 2 : 4; st >= 2 && !stages; --st)
        if (L.total(st) <= VBD_TILE_SMEM_MAX) stages = st;
    for (int st = 3; st >= 2 && !stages && W == 4; --st)  // else one CTA per SM
        if (L.total(st) <= 2 * VBD_TILE_SMEM_MAX) stages = st;
    const char* se = getenv("VBD_TILE_STAGES");
    if (se && *se) stages = std::min(stages, atoi(se));
    if (xr && (W != 2 || stages < 2)) return;
    if (VPT == 32) {  // compiled for 2 stages at 3 CTAs per SM (the stages are half as large)
        if (stages < 2) return;
        stages = 2;
        c->tile_occ = 3;
    }
    if (cls) stages = std::min(stages, 2);  // the class loop is compiled for the 2-stage ring
    if (xr) {  // K1T-X: 2 stages, 2 CTAs per SM (registers for the rows in flight; measured faster)
        stages = 2;
        if (!(oe && *oe == '3')) c->tile_occ = 2;
    }
    if (stages < 2) return;
    c->tile_stages = stages;
    DBuf dl, ds, sbase;
    upload(dl, nls.data(), nls.size(), s);
    upload(ds, nss.data(), nss.size(), s);
    exclusive_offsets(dl.as<long long>(), nt, c->loff, s);
    exclusive_offsets(ds.as<long long>(), nt, sbase, s);
    const long long total = read_scalar<long long>(c->loff.as<long long>() + nt, s);
    const long long slots = read_scalar<long long>(sbase.as<long long>() + nt, s);
    c->tnbr.alloc((size_t)std::max<long long>(total, 1) * 4);
    c->tent.alloc((size_t)std::max<long long>(slots, 1) * 8);
    DBuf slot_entry;  // XR: the explicit entry of every slot (-1: padding)
    if (xr) slot_entry.alloc((size_t)std::max<long long>(slots, 1) * 8);
    k_tile_nbrs<true><<<nt, 256, sort_smem, s>>>(c->tv0.as<int>(), c->tnv.as<int>(), eoffb,
                                                cent, nullptr, c->loff.as<long long>(), sbase.as<long long>(),
                                                c->tnbr.as<int>(), c->tent.as<uint2>(), W,
                                                PU, (unsigned)(c->nbr_cap * PU),
                                                xr ? 0u : c->tile_kg ? 1u : TileSmem<R>::KSTRIDE,
                                                xr ? 0u : c->tile_kg ? (unsigned)c->nkinds
                                                                     : (unsigned)(c->nkinds * TileSmem<R>::KSTRIDE),
                                                err.as<int>(), xr ? slot_entry.as<long long>() : nullptr, tWp);
    CK(cudaGetLastError());
    if (read_scalar<int>(err.p, s)) fail(VBD_ERR_INTERNAL, "tile build failed");
    if (slack > 0) {
        DBuf dnl, ids, asg;
        upload(dnl, nl_real.data(), nl_real.size(), s);
        ids.alloc((size_t)std::max<long long>(total, 1) * 4);
        asg.alloc((size_t)std::max<long long>(total, 1) * 4);
        // bank groups: DSATUR colouring per tile (VBD_TILE_BANKS=greedy: the sweep-order greedy)
        const char* bm = getenv("VBD_TILE_BANKS");
        const bool dsatur = !(bm && std::string(bm) == "greedy");
        const unsigned pad_pos = (unsigned)(c->nbr_cap * PU);
        if (dsatur) {
            int vmax = 1;
            for (int t = 0; t < nt; ++t) vmax = std::max(vmax, nl_real[t]);
            const int mmax = 3 * c->ent_cap;
            const size_t smem = (size_t)vmax * 12 + (size_t)(vmax + 1) * 4 + (size_t)mmax * 2 + 16;
            CK(cudaFuncSetAttribute(k_tile_banks_dsatur, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_tile_banks_dsatur<<<nt, 32, smem, s>>>(c->loff.as<long long>(), sbase.as<long long>(), dnl.as<int>(), nt,
                                                    PU, pad_pos, c->tent.as<uint2>(), asg.as<int>(), vmax, mmax);
            CK(cudaGetLastError());
        }
        k_tile_banks<<<blocks_for(nt, 64), 64, 0, s>>>(c->tv0.as<int>(), c->tnv.as<int>(), eoffb,
                                                      c->loff.as<long long>(), sbase.as<long long>(), dnl.as<int>(),
                                                      nt, W, PU, pad_pos,
                                                      c->tnbr.as<int>(), c->tent.as<uint2>(), ids.as<int>(),
                                                      asg.as<int>(), dsatur ? 1 : 0, tWp);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
    }
    if (xr) {  // the rows of every slot, 9 planes in slot order (padding: zeros)
        c->xrows.alloc((size_t)std::max<long long>(slots, 1) * 9 * 4);
        k_slot_rows<<<blocks_for(std::max<long long>(slots, 1)), 256, 0, s>>>(
            slot_entry.as<long long>(), slots, c->ent.as<float4>(), c->E, c->xrows.as<float>());
        CK(cudaGetLastError());
        c->tile_xr = true;
    }
    c->tdesc.alloc((size_t)nt * sizeof(TileDesc));
    k_tile_desc<<<blocks_for(nt), 256, 0, s>>>(c->tv0.as<int>(), c->tnv.as<int>(), eoffb,
                                              c->loff.as<long long>(), sbase.as<long long>(), nt, W,
                                              c->tdesc.as<TileDesc>(), tWp, cls ? dtcw.as<int>() : nullptr);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    c->tiles = true;
}

// per-vertex entry order: by rest-edge sign pattern (fp32 scenes large enough for class tiles,
// or VBD_ENTRY_ORDER=code) else by kind hash alone (the small scenes measured ~2 % faster with
// it on C2; fp64 has no class tiles)
template <typename R> static bool entry_order_by_code(long long n)
{
    const char* e = getenv("VBD_ENTRY_ORDER");
    if (e && std::string(e) == "code") return true;
    if (e && std::string(e) == "hash") return false;
    return sizeof(R) == 4 && n >= 200000;
}

// per-vertex entry order by kind (k_inc_kind_keys): one stable 64-bit radix sort of
// (vertex << 32 | kind hash) over the incidence
template <typename R> void sort_incidence_by_kind(Scene& sc, cudaStream_t s)
{
    const long long n4 = 4 * sc.T;
    if (n4 == 0) return;
    DBuf keys;
    keys.alloc(n4 * 8);
    k_inc_kind_keys<R><<<blocks_for(sc.n), 256, 0, s>>>(sc.inc_off.as<long long>(), sc.inc.as<unsigned>(),
                                                        sc.tet_w.as<double>(), sc.vol.as<double>(),
                                                        sc.tmat.as<int>(), sc.n, keys.as<unsigned long long>(),
                                                        entry_order_by_code<R>(sc.n) ? 1 : 0);
    CK(cudaGetLastError());
    sort_pairs_u64_i32(keys, sc.inc, n4, s);
}

// K6 + context finalisation
template <typename R> void pack(vbd_ctx* c, Scene& sc)
{
    Nvtx nv_("pack (K6)");
    cudaStream_t s = c->stream;
    c->n = sc.n;
    c->T = sc.T;
    if (sc.n >= (1LL << VBD_ID_BITS)) fail(VBD_ERR_UNSUPPORTED, "too many vertices for one context");
    if (!(getenv("VBD_KIND_ORDER") && *getenv("VBD_KIND_ORDER") == '0')) sort_incidence_by_kind<R>(sc, s);
    // colouring validity (decides in-place vs aux-buffer sweeps)
    {
        DBuf bad;
        bad.alloc(4);
        CK(cudaMemsetAsync(bad.p, 0, 4, s));
        if (sc.T)
            k_check_coloring<<<blocks_for(sc.T), 256, 0, s>>>(sc.tets.as<int>(), sc.T,
                                                             sc.color.as<int>(), bad.as<int>());
        CK(cudaGetLastError());
        c->inplace = read_scalar<int>(bad.p, s) == 0;
    }
    // order: spatial (Morton code of the rest positions) inside each (category, colour,
    // rounds) class, so the vertices of one CTA -- and their neighbours -- are compact in
    // space and share L1/L2 lines.  Two stable radix sorts: Morton first, then the class.
    DBuf order0;
    order0.alloc(sc.n * 4);
    if (sc.pos.p && sc.n) {
        DBuf mk;
        mk.alloc(sc.n * 8);
        k_morton_keys<<<blocks_for(sc.n), 256, 0, s>>>(sc.pos.as<double>(), sc.n, sc.bbox_lo[0],
                                                       sc.bbox_lo[1], sc.bbox_lo[2], sc.bbox_scale,
                                                       mk.as<unsigned long long>(), order0.as<int>());
        CK(cudaGetLastError());
        sort_pairs_u64_i32(mk, order0, sc.n, s);
    } else if (sc.n) {
        k_iota<<<blocks_for(sc.n), 256, 0, s>>>(order0.as<int>(), sc.n);
        CK(cudaGetLastError());
    }
    // grid-class instances (K1T class tiles, fp32): per original vertex its instance or -1
    DBuf vinst;
    std::vector<unsigned long long> ikeys;
    c->crun.clear();
    c->cinst_tpl.clear();
    {
        const char* ce = getenv("VBD_TILE_CLASS");
        const bool on = sizeof(R) == 4 && sc.n && sc.T && sc.tet_w.p && !(ce && *ce == '0') && entry_order_by_code<R>(sc.n) &&
                        !(getenv("VBD_KIND_ORDER") && *getenv("VBD_KIND_ORDER") == '0');
        if (on) {
            DBuf ck, table, ovf, sorted;
            ck.alloc(sc.n * 8);
            k_vertex_class<R><<<blocks_for(sc.n), 256, 0, s>>>(sc.inc_off.as<long long>(), sc.inc.as<unsigned>(),
                                                               sc.tets.as<int>(), sc.tet_w.as<double>(),
                                                               sc.vol.as<double>(), sc.tmat.as<int>(), sc.n,
                                                               ck.as<unsigned long long>());
            CK(cudaGetLastError());
            constexpr int CAP = 256;
            table.alloc(CAP * 8);
            ovf.alloc(4);
            CK(cudaMemsetAsync(table.p, 0, CAP * 8, s));
            CK(cudaMemsetAsync(ovf.p, 0, 4, s));
            k_class_keys_insert<<<blocks_for(sc.n), 256, 0, s>>>(ck.as<unsigned long long>(), sc.n,
                                                                table.as<unsigned long long>(), CAP, ovf.as<int>());
            CK(cudaGetLastError());
            std::vector<unsigned long long> ht(CAP);
            CK(cudaMemcpyAsync(ht.data(), table.p, CAP * 8, cudaMemcpyDeviceToHost, s));
            const int of = read_scalar<int>(ovf.p, s);
            for (unsigned long long k : ht)
                if (k) ikeys.push_back(k);
            std::sort(ikeys.begin(), ikeys.end());
            if (of || ikeys.size() > 64) ikeys.clear();  // too many instances: no class tiles
            if (!ikeys.empty()) {
                upload(sorted, ikeys.data(), ikeys.size(), s);
                vinst.alloc(sc.n);
                k_class_instance<<<blocks_for(sc.n), 256, 0, s>>>(ck.as<unsigned long long>(), sc.n,
                                                                 sorted.as<unsigned long long>(), (int)ikeys.size(),
                                                                 vinst.as<signed char>());
                CK(cudaGetLastError());
                CK(cudaStreamSynchronize(s));
                for (unsigned long long k : ikeys) c->cinst_tpl.push_back((int)(k >> 32) - 1);
            }
        }
    }
    DBuf keys;
    keys.alloc(sc.n * 8);
    k_order_keys<<<blocks_for(sc.n), 256, 0, s>>>(sc.inc_off.as<long long>(), sc.kind.as<unsigned char>(),
                                                  sc.halo.p ? sc.halo.as<unsigned char>() : nullptr,
                                                  sc.color.as<int>(), order0.as<int>(), sc.n, c->k1.W,
                                                  keys.as<unsigned long long>(),
                                                  vinst.p ? vinst.as<signed char>() : nullptr);
    CK(cudaGetLastError());
    sort_keys_u64(keys, sc.n, s);
    c->perm.alloc(sc.n * 4);
    c->inv.alloc(sc.n * 4);
    k_perm_from_keys<<<blocks_for(sc.n), 256, 0, s>>>(keys.as<unsigned long long>(), order0.as<int>(),
                                                      sc.n, c->perm.as<int>(), c->inv.as<int>());
    CK(cudaGetLastError());
    // category / colour ranges from the sorted keys (host scan of the boundaries)
    std::vector<unsigned long long> hk(sc.n);
    if (sc.n) CK(cudaMemcpyAsync(hk.data(), keys.p, sc.n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->nsolve = 0;
    c->nfree_all = 0;
    int maxc = -1;
    for (long long i = 0; i < sc.n; ++i) {
        unsigned cat = (unsigned)(hk[i] >> 56);
        if (cat == 0) c->nsolve = i + 1;
        if (cat <= 1) {
            c->nfree_all = i + 1;
            maxc = std::max(maxc, (int)((hk[i] >> 44) & 0xfff));
        }
    }
    c->ncolors = maxc + 1;
    c->cbeg.assign(c->ncolors, 0);
    c->ccnt.assign(c->ncolors, 0);
    for (long long i = c->nsolve - 1; i >= 0; --i) {
        int col = (int)((hk[i] >> 44) & 0xfff);
        c->cbeg[col] = i;
        c->ccnt[col]++;
    }
    // class-instance runs: (cat 0, interior class 2, rounds field 0x80 | instance)
    for (long long i = 0; i < c->nsolve && !c->cinst_tpl.empty(); ++i) {
        const unsigned cl = (unsigned)((hk[i] >> 40) & 0xf), r = (unsigned)((hk[i] >> 32) & 0xff);
        if (cl != 2 || !(r & 0x80u)) continue;
        const int col = (int)((hk[i] >> 44) & 0xfff), inst = (int)(r & 0x7fu);
        auto& v = c->crun;
        if (!v.empty() && v.back().inst == inst && v.back().beg + v.back().cnt == i &&
            (int)((hk[v.back().beg] >> 44) & 0xfff) == col)
            v.back().cnt++;
        else
            v.push_back({i, 1, inst});
    }
    // slab boundary blocks (head of each colour range) and ghost blocks per (side, colour)
    for (int sd = 0; sd < 2; ++sd) {
        c->bnd_cnt[sd].assign(c->ncolors, 0);
        c->ghost_beg[sd].assign(c->ncolors, 0);
        c->ghost_cnt[sd].assign(c->ncolors, 0);
    }
    for (long long i = 0; i < c->nfree_all; ++i) {
        const unsigned cat = (unsigned)(hk[i] >> 56), cls = (unsigned)((hk[i] >> 40) & 0xf);
        const int col = (int)((hk[i] >> 44) & 0xfff);
        if (cat == 0 && cls < 2) c->bnd_cnt[cls][col]++;
        if (cat == 1) {
            if (c->ghost_cnt[cls][col]++ == 0) c->ghost_beg[cls][col] = i;
        }
    }
    // colour ranges must be contiguous and ordered (guaranteed by the key layout)
    // entry offsets over solved vertices
    DBuf deg;
    deg.alloc(std::max<long long>(c->nsolve, 1) * 8);
    if (c->nsolve)
        k_degree_new<<<blocks_for(c->nsolve), 256, 0, s>>>(sc.inc_off.as<long long>(),
                                                           c->perm.as<int>(), c->nsolve,
                                                           deg.as<long long>());
    CK(cudaGetLastError());
    exclusive_offsets(deg.as<long long>(), c->nsolve, c->eoff, s);
    c->E = read_scalar<long long>(c->eoff.as<long long>() + c->nsolve, s);
    {
        DBuf md;
        md.alloc(4);
        CK(cudaMemsetAsync(md.p, 0, 4, s));
        if (c->nsolve)
            k_max_degree<<<blocks_for(c->nsolve), 256, 0, s>>>(c->eoff.as<long long>(), c->nsolve, md.as<int>());
        CK(cudaGetLastError());
        c->max_deg = read_scalar<int>(md.p, s);
    }
    const int P = EntryPlanes<R>::P;
    c->ent.alloc(std::max<long long>(c->E, 1) * P * 16);
    DBuf badv;
    badv.alloc(4);
    CK(cudaMemsetAsync(badv.p, 0, 4, s));
    if (c->nsolve)
        k_pack_entries<R><<<blocks_for(c->nsolve, 128), 128, 0, s>>>(
            sc.inc_off.as<long long>(), sc.inc.as<unsigned>(), sc.tets.as<int>(),
            sc.tet_w.as<double>(), sc.vol.as<double>(), sc.tmat.as<int>(), c->perm.as<int>(),
            c->inv.as<int>(), c->eoff.as<long long>(), c->nsolve,
            c->ent.as<typename PlaneT<R>::T>(), c->E, badv.as<int>());
    CK(cudaGetLastError());
    if (read_scalar<int>(badv.p, s))
        fail(VBD_ERR_UNSUPPORTED,
             "fp32 layout recomputes tet volumes from |det W|; tet_vol disagrees with tet_w "
             "(use precision=fp64)");
    compact_entries<R>(c);
    // one material per vertex? (always true for bodies built by build_system)
    {
        DBuf mixed;
        mixed.alloc(4);
        CK(cudaMemsetAsync(mixed.p, 0, 4, s));
        c->vmat.alloc(std::max<long long>(c->nsolve, 1) * 4);
        if (c->nsolve)
            k_vertex_material<<<blocks_for(c->nsolve), 256, 0, s>>>(
                sc.inc_off.as<long long>(), sc.inc.as<unsigned>(), sc.tmat.as<int>(), c->perm.as<int>(),
                c->nsolve, c->vmat.as<int>(), mixed.as<int>());
        CK(cudaGetLastError());
        c->uniform_mat = read_scalar<int>(mixed.p, s) == 0;
        const char* e = getenv("VBD_UNIFORM_MAT");
        if (e && *e == '0') c->uniform_mat = false;
    }
    // masses in colour-major order
    c->mass.alloc(sc.n * sizeof(R));
    k_mass_new<R><<<blocks_for(sc.n), 256, 0, s>>>(sc.mass.as<double>(), c->perm.as<int>(), sc.n,
                                                   c->mass.as<R>());
    CK(cudaGetLastError());
    // original-order colours (for vbd_get_colors)
    c->color_orig.alloc(sc.n * 4);
    CK(cudaMemcpyAsync(c->color_orig.p, sc.color.p, sc.n * 4, cudaMemcpyDeviceToDevice, s));
    alloc_state<R>(c);
    // rest positions (colour-major, double) and the fp32 displacement state
    if (sc.pos.p && sc.n) {
        c->rest.alloc((size_t)sc.n * sizeof(double4));
        k_rest_positions<<<blocks_for(sc.n), 256, 0, s>>>(sc.pos.as<double>(), c->perm.as<int>(), (int)sc.n,
                                                          c->rest.as<double4>());
        CK(cudaGetLastError());
        const char* de = getenv("VBD_DISP");
        c->disp = sizeof(R) == 4 && !c->has_extras && !(de && *de == '0');
    }
    if (sizeof(R) == 4 ? c->disp : true) build_tiles<R>(c);  // fp32 K1T needs the displacement state
    CK(cudaStreamSynchronize(s));
}

// material table for step size h
template <typename R> K1Args<R> k1_args(vbd_ctx* c, double eps_det, int mode, bool check, int iter);

template <typename R> void ensure_materials(vbd_ctx* c, double h)
{
    if (c->mat_h == h && c->mat.p) return;
    std::vector<Material<R>> m(c->mats.size());
    for (size_t i = 0; i < m.size(); ++i) {
        double mu = c->mats[i].mu, lam = c->mats[i].lam, kd = c->mats[i].kd;
        double g = 1.0 + mu / lam;  // _native.pyx:291
        double dsc = kd / h;        // _native.pyx:309
        m[i] = Material<R>{(R)mu, (R)lam, (R)g, (R)dsc, (R)(1.0 + dsc)};
    }
    if (!c->mat.p) c->mat.alloc(VBD_MAX_MATERIALS * sizeof(Material<R>));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(c->mat.p, m.data(), m.size() * sizeof(Material<R>), cudaMemcpyHostToDevice));
    c->mat_h = h;
    refresh_kinds<R>(c);
    if (c->uniform_mat && c->nsolve) {  // per-vertex sum of V mu |w|^2 (k_vertex_sv)
        if (c->vsv.bytes < (size_t)c->nsolve * sizeof(R)) c->vsv.alloc((size_t)c->nsolve * sizeof(R));
        K1Args<R> a = k1_args<R>(c, 1e-10, 0, false, 0);
        k_vertex_sv<R><<<blocks_for(c->nsolve), 256, 0, c->stream>>>(a, (int)c->nsolve, c->vsv.as<R>());
        CK(cudaGetLastError());
    }
}

template <typename R>
K1Args<R> k1_args(vbd_ctx* c, double eps_det, int mode, bool check, int iter)
{
    K1Args<R> a;
    a.ent = c->ent.as<typename PlaneT<R>::T>();
    a.E = c->E;
    a.kinds = c->compact ? c->kinds.as<typename PlaneT<R>::T>() : nullptr;
    a.max_deg = c->max_deg;
    typedef typename Vec4<R>::T R4;
    a.soff = c->has_extras ? c->soff.as<long long>() : nullptr;
    a.sp_oth = c->sp_oth.as<int>();
    a.sp_par = c->sp_par.as<R4>();
    a.box = c->has_extras && c->box.p ? c->box.as<R4>() : nullptr;
    a.sub_idx = c->sub_idx.as<int>();
    a.sub = c->sub.as<R4>();
    a.h = (R)c->mat_h;
    a.coff = c->ncontacts ? c->coff.as<long long>() : nullptr;
    a.ccid = c->ccid.as<int>();
    a.cslot = c->cslot.as<int>();
    a.cidx = c->cidx.as<int4>();
    a.creal = c->creal.as<R4>();
    a.mu_c = (R)c->mu_c;
    a.eps_u = (R)(c->eps_v * c->mat_h);
    a.off = c->eoff.as<long long>();
    a.pos = c->pos.as<typename Vec4<R>::T>();
    a.xt = c->xt.as<typename Vec4<R>::T>();
    a.y = c->y.as<typename Vec4<R>::T>();
    a.mat = c->mat.as<Material<R>>();
    a.group = nullptr;
    a.vbeg = 0;
    a.count = 0;
    a.nsolve = (int)c->nsolve;
    a.out = nullptr;
    a.eps_det = (R)eps_det;
    a.mode = mode;
    a.flag = check ? c->flag.as<unsigned long long>() : nullptr;
    a.perm = c->perm.as<int>();
    a.stepctr = c->stepctr.as<int>();
    a.iter = iter;
    a.pf_dist = 0;
    a.vmat = c->uniform_mat ? c->vmat.as<int>() : nullptr;
    a.vsv = c->uniform_mat ? c->vsv.as<R>() : nullptr;
    a.kedge = (c->disp && c->compact) ? c->kedge.as<float4>() : nullptr;
    a.disp = c->disp ? 1 : 0;
    a.line_search = 0;
    a.peer_pos[0] = a.peer_pos[1] = nullptr;
    a.peer_off[0] = a.peer_off[1] = 0;
    a.nb[0] = a.nb[1] = 0;
    return a;
}

// Launch with programmatic stream serialisation (PDL) for the kernels that begin with
// pdl_wait(): the next colour pass / blend is scheduled while the previous one drains, which
// hides most of the per-node launch latency of small scenes' step graphs.  VBD_PDL=0 disables.
bool pdl_enabled()
{
    static const bool on = !getenv("VBD_PDL") || atoi(getenv("VBD_PDL")) != 0;
    return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

template <typename R, int W, int U, int B> void launch_k1v(const K1Args<R>& a0, bool pf, cudaStream_t s)
{
    long long threads = (long long)a0.count * W;
    K1Args<R> a = a0;
    // prefetch distance in CTAs: 0 = each CTA prefetches its own entry range (measured best
    // on B200; a one-wave look-ahead thrashes L2)
    static const int dist = getenv("VBD_K1_PFDIST") ? atoi(getenv("VBD_K1_PFDIST")) : 0;
    a.pf_dist = dist;
    const unsigned nb = blocks_for(threads);
    const bool um = a.vmat != nullptr;
    // compact range passes: entries staged in smem by one bulk copy per CTA
    static const bool bulk_on = !getenv("VBD_K1_BULK") || atoi(getenv("VBD_K1_BULK")) != 0;
    const size_t smem = (size_t)(256 / W) * (size_t)std::max(a.max_deg, 1) * 16;
    if (a.kinds && !a.group && !a.out && bulk_on && smem <= 64 * 1024) {
        static bool attr[64][2] = {};  // per device
        int dev = 0;
        CK(cudaGetDevice(&dev));
        dev &= 63;
        auto kb = um ? k1_color_pass_bulk<R, W, U, B, true> : k1_color_pass_bulk<R, W, U, B, false>;
        if (!attr[dev][um]) {
            CK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
            attr[dev][um] = true;
        }
        launch_pdl(kb, nb, 256, smem, s, a);
        return;
    }
    if (a.kinds) {
        if (pf && um) launch_pdl(k1_color_pass<R, W, U, B, true, true, true>, nb, 256, 0, s, a);
        else if (pf) launch_pdl(k1_color_pass<R, W, U, B, true, false, true>, nb, 256, 0, s, a);
        else if (um) launch_pdl(k1_color_pass<R, W, U, B, false, true, true>, nb, 256, 0, s, a);
        else launch_pdl(k1_color_pass<R, W, U, B, false, false, true>, nb, 256, 0, s, a);
        return;
    }
    if (pf && um) launch_pdl(k1_color_pass<R, W, U, B, true, true>, nb, 256, 0, s, a);
    else if (pf) launch_pdl(k1_color_pass<R, W, U, B, true, false>, nb, 256, 0, s, a);
    else if (um) launch_pdl(k1_color_pass<R, W, U, B, false, true>, nb, 256, 0, s, a);
    else launch_pdl(k1_color_pass<R, W, U, B, false, false>, nb, 256, 0, s, a);
}

template <typename R, bool UM, int S, int W, int OCC, int DEF, bool KG = false, bool XR = false, int TV = 64,
          bool CL = false>
void launch_k1_tiles_v(const K1TArgs<R>& ta, size_t smem, cudaStream_t s)
{
    // the shared-memory opt-in and the occupancy are per device
    static size_t attr[64] = {};
    static int per_sm[64] = {}, sms[64] = {};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    dev &= 63;
    if (smem > attr[dev]) {
        CK(cudaFuncSetAttribute(k1_tiles<R, UM, S, W, OCC, DEF, KG, XR, TV, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[dev] = smem;
        CK(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k1_tiles<R, UM, S, W, OCC, DEF, KG, XR, TV, CL>, TV * W + 32, smem));
        per_sm[dev] = std::max(1, per_sm[dev]);
    }
    const int grid = std::min(ta.tcount, per_sm[dev] * sms[dev]);
    launch_pdl(k1_tiles<R, UM, S, W, OCC, DEF, KG, XR, TV, CL>, (unsigned)grid, TV * W + 32, smem, s, ta);
}

template <typename R, bool UM, int W>
void launch_k1_tiles_s(const K1TArgs<R>& ta, int stages, int occ, bool defer, bool kg, size_t smem,
                       cudaStream_t s)
{
    if constexpr (W == 2) {  // 2 stages; global kind records or 2 CTAs per SM
        if (kg && occ == 3) return launch_k1_tiles_v<R, UM, 2, W, 3, W, true>(ta, smem, s);
        if (kg) return launch_k1_tiles_v<R, UM, 2, W, 2, W, true>(ta, smem, s);
        if (occ == 2) return launch_k1_tiles_v<R, UM, 2, W, 2, W>(ta, smem, s);
    }
    if (kg) fail(VBD_ERR_INTERNAL, "global kind records are compiled for 2 lanes per vertex");
    if (occ == 3) {
        if (stages >= 3) launch_k1_tiles_v<R, UM, 3, W, 3, 1>(ta, smem, s);
        else if (defer) launch_k1_tiles_v<R, UM, 2, W, 3, W>(ta, smem, s);
        else launch_k1_tiles_v<R, UM, 2, W, 3, 1>(ta, smem, s);
        return;
    }
    if constexpr (W == 4) {
        if (stages >= 4) launch_k1_tiles_v<R, UM, 4, W, 2, 1>(ta, smem, s);
        else if (stages == 3) launch_k1_tiles_v<R, UM, 3, W, 2, 1>(ta, smem, s);
        else launch_k1_tiles_v<R, UM, 2, W, 2, 1>(ta, smem, s);
    }
}

template <typename R, bool UM>
void launch_k1_tiles_w(const K1TArgs<R>& ta, int W, int stages, int occ, bool defer, bool kg, size_t smem,
                       cudaStream_t s)
{
    // W lanes per vertex in 2 W consumer warps (64-vertex tiles); 1 lane was measured slower
    if (W == 2) launch_k1_tiles_s<R, UM, 2>(ta, stages, occ, defer, kg, smem, s);
    else launch_k1_tiles_s<R, UM, 4>(ta, stages, occ, defer, kg, smem, s);
}

template <typename R> bool launch_k1_tiles(const vbd_ctx* c, const K1Args<R>& a, cudaStream_t s)
{
    if (!c->tiles || a.group || a.out || a.line_search || (!a.kinds && !c->tile_xr) || a.coff) return false;
    int col = -1;
    for (int k = 0; k < c->ncolors; ++k)
        if (c->cbeg[k] == a.vbeg && c->ccnt[k] == a.count) col = k;
    if (col < 0) return false;
    K1TArgs<R> ta;
    ta.a = a;
    ta.tent = c->tent.as<uint2>();
    ta.tnbr = c->tnbr.as<int>();
    ta.desc = c->tdesc.as<TileDesc>();
    ta.kinds = c->kinds.as<typename PlaneT<R>::T>();
    ta.tbeg = c->tile_beg[col];
    ta.tcount = c->tile_beg[col + 1] - c->tile_beg[col];
    ta.ent_cap = c->ent_cap;
    ta.nbr_cap = c->nbr_cap;
    ta.nkinds = c->nkinds;
    const char* dbg = getenv("VBD_TILE_DBG");
    ta.dbg = dbg && *dbg ? atoi(dbg) : 0;
    if (ta.dbg) ta.a.flag = nullptr;  // garbage positions in the timing experiments
    static const bool early = !(getenv("VBD_PDL_EARLY") && *getenv("VBD_PDL_EARLY") == '0');
    ta.early = early ? 1 : 0;
    ta.ckind = c->ncrec ? c->ckind.as<int>() : nullptr;
    ta.ncrec = c->ncrec;
    ta.svpt = c->tile_svpt;
    ta.xrows = c->tile_xr ? c->xrows.as<float>() : nullptr;
    ta.xstride = c->tile_xr ? (long long)(c->tent.bytes / 8) : 0;
    ta.xtg = c->tile_xtg ? 1 : 0;
    ta.tcls = c->class_tiles ? c->tile_cls_beg[col] - ta.tbeg : ta.tcount;
    const TileSmem<R> L{ta.ent_cap, ta.nbr_cap, (c->tile_kg || c->tile_xr) ? -1 : ta.nkinds + ta.ncrec,
                        c->tile_svpt, c->tile_xtg ? 1 : 3};
    const int S = c->tile_stages;
    if (c->tile_vpt == 32) {  // small scenes: 32-vertex tiles (2 lanes, 2 stages, deferred solves)
        if (c->tile_w != 2 || S != 2 || c->tile_kg || c->tile_xr || c->tile_occ != 3 || !c->tile_defer)
            fail(VBD_ERR_INTERNAL, "32-vertex tiles: configuration");
        if (a.vmat) launch_k1_tiles_v<R, true, 2, 2, 3, 2, false, false, 32>(ta, L.total(S), s);
        else launch_k1_tiles_v<R, false, 2, 2, 3, 2, false, false, 32>(ta, L.total(S), s);
        return true;
    }
    if (c->tile_xr) {  // K1T-X: fp32, one material per vertex, 2 lanes, deferred solves
        if constexpr (sizeof(R) == 4) {
            if (!a.vmat || c->tile_w != 2 || S != 2) fail(VBD_ERR_INTERNAL, "K1T-X configuration");
            if (c->tile_occ == 3) launch_k1_tiles_v<R, true, 2, 2, 3, 2, false, true>(ta, L.total(S), s);
            else launch_k1_tiles_v<R, true, 2, 2, 2, 2, false, true>(ta, L.total(S), s);
        }
        return true;
    }
    if (c->class_tiles) {  // (build_tiles: fp32, one material per vertex, 2 lanes, 2 stages)
        if constexpr (sizeof(R) == 4) {
            if (!a.vmat || c->tile_w != 2 || c->tile_kg || S != 2) fail(VBD_ERR_INTERNAL, "class tiles: configuration");
            const size_t sm = L.total(S);
            if (c->tile_occ == 2) launch_k1_tiles_v<R, true, 2, 2, 2, 2, false, false, 64, true>(ta, sm, s);
            else if (c->tile_defer) launch_k1_tiles_v<R, true, 2, 2, 3, 2, false, false, 64, true>(ta, sm, s);
            else launch_k1_tiles_v<R, true, 2, 2, 3, 1, false, false, 64, true>(ta, sm, s);
            return true;
        }
    }
    if (a.vmat) launch_k1_tiles_w<R, true>(ta, c->tile_w, S, c->tile_occ, c->tile_defer, c->tile_kg, L.total(S), s);
    else launch_k1_tiles_w<R, false>(ta, c->tile_w, S, c->tile_occ, c->tile_defer, c->tile_kg, L.total(S), s);
    return true;
}

template <typename R> void launch_k1(const vbd_ctx* c, const K1Args<R>& a, cudaStream_t s)
{
    if (a.count <= 0) return;
    if (launch_k1_tiles<R>(c, a, s)) return;
    if (a.line_search && a.mode == 0) {
        k1_color_pass_ls<R><<<blocks_for((long long)a.count * 4), 256, 0, s>>>(a);
        return;
    }
    const K1Variant& v = c->k1;
    if (v.W == 4 && v.U == 2 && v.minb == 3) launch_k1v<R, 4, 2, 3>(a, v.pf != 0, s);
    else if (v.W == 4 && v.U == 1) launch_k1v<R, 4, 1, 1>(a, v.pf != 0, s);
    else if (v.W == 8 && v.U == 1) launch_k1v<R, 8, 1, 1>(a, v.pf != 0, s);
    else fail(VBD_ERR_ARG, "unknown VBD_K1 variant (4x2b3, 4x1, 8x1)");
}

// one colour pass of the step (in place when the colouring is valid, else aux buffer)
template <typename R> void color_sweep(vbd_ctx* c, int color, int iter, bool check)
{
    cudaStream_t s = c->stream;
    K1Args<R> a = k1_args<R>(c, c->cur.eps_det, 0, check, iter);
    a.line_search = c->cur.line_search ? 1 : 0;
    a.vbeg = (int)c->cbeg[color];
    a.count = (int)c->ccnt[color];
    if (!c->inplace || c->ncontacts) {
        // aux-buffer semantics over the contiguous colour range (invalid colouring, or contacts
        // coupling vertices of one colour): compute into `out`, then copy
        a.out = c->out.as<typename Vec4<R>::T>();
        launch_k1<R>(c, a, s);
        CK(cudaMemcpyAsync(c->pos.as<char>() + c->cbeg[color] * c->r4(), c->out.p,
                           c->ccnt[color] * c->r4(), cudaMemcpyDeviceToDevice, s));
    } else {
        launch_k1<R>(c, a, s);
    }
}

std::vector<double> omega_table(double rho, int n_max)
{
    // solver.py:167-177, evaluated exactly as the reference does (recurrence from scratch)
    std::vector<double> w(n_max + 1, 1.0);
    for (int n = 1; n <= n_max; ++n) {
        if (rho == 0.0 || n == 1) { w[n] = 1.0; continue; }
        double omega = 2.0 / (2.0 - rho * rho);
        for (int k = 3; k <= n; ++k) omega = 4.0 / (4.0 - rho * rho * omega);
        w[n] = omega;
    }
    return w;
}

template <typename R> StepArgs<R> step_args(vbd_ctx* c)
{
    typedef typename Vec4<R>::T R4;
    const vbd_step_params& p = c->cur;
    StepArgs<R> a;
    a.n = (int)c->n;
    a.nsolve = (int)c->nsolve;
    a.nfree_all = (int)c->nfree_all;
    a.pos = c->pos.as<R4>();
    a.xt = c->xt.as<R4>();
    a.vt = c->vt.as<R4>();
    a.vprev = c->vprev.as<R4>();
    a.y = c->y.as<R4>();
    a.ha = c->ha.as<R4>();
    a.hb = c->hb.as<R4>();
    a.mass = c->mass.as<R>();
    a.h = p.h;
    a.hh = p.h * p.h;
    double nrm = std::sqrt(p.a_ext[0] * p.a_ext[0] + p.a_ext[1] * p.a_ext[1] + p.a_ext[2] * p.a_ext[2]);
    for (int k = 0; k < 3; ++k) {
        a.a[k] = p.a_ext[k];
        a.an[k] = nrm > 0 ? p.a_ext[k] / nrm : 0.0;
    }
    a.anorm = nrm;
    a.init_mode = p.init_mode;
    a.hist = p.rho != 0.0;
    a.flag = c->flag.as<unsigned long long>();
    a.perm = c->perm.as<int>();
    a.stepctr = c->stepctr.as<int>();
    a.sub_idx = c->has_extras ? c->sub_idx.as<int>() : nullptr;
    a.sub = c->sub.as<R4>();
    return a;
}

template <typename R> void enqueue_begin(vbd_ctx* c)
{
    StepArgs<R> a = step_args<R>(c);
    k2_step_init<R><<<blocks_for(c->n), 256, 0, c->stream>>>(a);
}

template <typename R> void enqueue_iter_end(vbd_ctx* c, int n)
{
    typedef typename Vec4<R>::T R4;
    if (c->cur.rho == 0.0) return;  // omega == 1 throughout: no blend, no history
    R4* hist = (n % 2 == 1) ? c->hb.as<R4>() : c->ha.as<R4>();
    double w = c->omegas[n];
    int blend = (n >= 2 && w != 1.0) ? 1 : 0;
    launch_pdl(k3_chebyshev<R>, blocks_for(c->n), 256, 0, c->stream, c->pos.as<R4>(), hist, (int)c->n, w,
               blend, c->flag.as<unsigned long long>(), c->perm.as<int>(), c->stepctr.as<int>(), n,
               c->coll_on ? (const unsigned char*)c->ccoll.as<unsigned char>() : nullptr);
}

template <typename R> void enqueue_end(vbd_ctx* c)
{
    typedef typename Vec4<R>::T R4;
    k4_commit<R><<<blocks_for(std::max<long long>(c->n, 1)), 256, 0, c->stream>>>(
        c->pos.as<R4>(), c->xt.as<R4>(), c->vt.as<R4>(), c->vprev.as<R4>(), (int)c->n, c->cur.h,
        c->flag.as<unsigned long long>(), c->stepctr.as<int>());
}

template <typename R> void launch_resident(vbd_ctx* c);

template <typename R> void enqueue_step(vbd_ctx* c)
{
    if (c->res_mode > 0 && !c->cur.line_search) {  // the whole step in one resident launch
        launch_resident<R>(c);
        return;
    }
    enqueue_begin<R>(c);
    bool check_in_k1 = c->cur.rho == 0.0;  // otherwise K3 checks every vertex
    for (int n = 1; n <= c->cur.n_max; ++n) {
        for (int col = 0; col < c->ncolors; ++col) color_sweep<R>(c, col, n, check_in_k1);
        enqueue_iter_end<R>(c, n);
    }
    enqueue_end<R>(c);
}

// ---- P2P slab halo: one graph per step with neighbour phase barriers ------------------

template <typename R> void enqueue_step_p2p(vbd_ctx* c)
{
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    unsigned long long* fl = c->p2p_flags.as<unsigned long long>();
    const unsigned long long* epoch = fl + 2;
    int* err = reinterpret_cast<int*>(fl + 3);
    const int nl = c->peer_pos[0] != nullptr, nr = c->peer_pos[1] != nullptr;
    const bool cheb = c->cur.rho != 0.0;
    const unsigned long long pps = 2ull + (unsigned long long)c->cur.n_max * (c->ncolors + (cheb ? 1 : 0));
    int phase = 0;
    auto wait = [&]() { k_phase_wait<<<1, 32, 0, s>>>(fl, nl, nr, epoch, pps, phase, err); };
    auto signal = [&]() { k_phase_signal<<<1, 32, 0, s>>>(c->peer_flag_slot[0], c->peer_flag_slot[1], epoch, pps, phase); };
    ++phase;
    wait();
    enqueue_begin<R>(c);
    signal();
    const bool check_in_k1 = !cheb;
    for (int n = 1; n <= c->cur.n_max; ++n) {
        for (int col = 0; col < c->ncolors; ++col) {
            ++phase;
            wait();
            K1Args<R> a = k1_args<R>(c, c->cur.eps_det, 0, check_in_k1, n);
            a.line_search = c->cur.line_search ? 1 : 0;
            a.vbeg = (int)c->cbeg[col];
            a.count = (int)c->ccnt[col];
            for (int sd = 0; sd < 2; ++sd) {
                a.peer_pos[sd] = static_cast<R4*>(c->peer_pos[sd]);
                a.nb[sd] = (int)c->bnd_cnt[sd][col];
                a.peer_off[sd] = c->peer_pos[sd] ? (int)c->peer_ghost_beg[sd][col] : 0;
            }
            launch_k1<R>(c, a, s);
            signal();
        }
        if (cheb) {
            ++phase;
            wait();
            enqueue_iter_end<R>(c, n);
            signal();
        }
    }
    ++phase;
    wait();
    enqueue_end<R>(c);
    signal();
    k_epoch_advance<<<1, 32, 0, s>>>(fl + 2, pps);
}

// Contacts (DCD / CCD and the K1 contact terms) work on absolute positions: leave the fp32
// displacement state for good -- x = fl32(X + u) for every position-like vector -- and drop
// the paths compiled for it (K1T tiles, K1R) and the cached step graph.
void to_absolute(vbd_ctx* c)
{
    if (!c->disp) return;
    cudaStream_t s = c->stream;
    for (DBuf* d : {&c->pos, &c->xt, &c->y, &c->ha, &c->hb})
        if (d->p) k_disp_to_abs<<<blocks_for(std::max<long long>(c->n, 1)), 256, 0, s>>>(d->as<float4>(),
                                                                                     c->rest.as<double4>(), (int)c->n);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    c->disp = false;
    c->tiles = false;
    c->res_mode = 0;
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
}

// ---- K1R: resident whole-step kernel for small scenes (vbd_resident.cuh) ----------------

// Decide (once per context, at its first step) whether the step runs as one resident launch,
// and build its per-CTA layout on the host from the compact entries: per colour, 8-vertex
// groups (4 lanes per vertex, rounds = max ceil(d / 4), even) are cut into contiguous runs of
// equal slot work, one run per CTA; each group's slots are [round][lane] int4 {n0, n1, n2,
// kind}, padding = {n, n, n, nkinds} (zero position, zero record).
// VBD_RESIDENT: unset = REPL when the replica fits one cluster, else GLOB for fp32 scenes of at
// most VBD_RES_GLOB_MAX (18000) vertices per colour; "0" off, "repl" / "glob" force.
template <typename R> void ensure_resident(vbd_ctx* c)
{
    if (c->res_mode >= 0) return;
    c->res_mode = 0;
    const std::string want = c->res_want;
    if (want == "0" || !c->compact || !c->inplace || c->has_extras || c->ncontacts || c->coll_on || c->nsolve == 0 ||
        c->ncolors > VBD_RES_MAX_COLORS || c->nkinds >= 65535 || c->n >= (1LL << 30))
        return;
    Nvtx nv_("resident layout");
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    std::vector<long long> eoff(c->nsolve + 1);
    std::vector<int4> ent((size_t)c->E);
    CK(cudaMemcpyAsync(eoff.data(), c->eoff.p, eoff.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ent.data(), c->ent.p, ent.size() * 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int dev = 0, sms = 148, smem_max = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    struct G { int v0, nv, rounds; };
    std::vector<std::vector<G>> cg(c->ncolors);
    for (int col = 0; col < c->ncolors; ++col)
        for (long long o = 0; o < c->ccnt[col]; o += 8) {
            G g{(int)(c->cbeg[col] + o), (int)std::min<long long>(8, c->ccnt[col] - o), 0};
            for (int k = 0; k < g.nv; ++k) {
                const long long d = eoff[g.v0 + k + 1] - eoff[g.v0 + k];
                g.rounds = std::max(g.rounds, (int)((d + 3) / 4));
            }
            g.rounds = (g.rounds + VBD_RES_U - 1) / VBD_RES_U * VBD_RES_U;
            cg[col].push_back(g);
        }
    // runs of equal work per CTA and colour
    auto plan = [&](int ncta, std::vector<std::vector<int>>& cut, int& slot_cap, int& grp_cap) {
        cut.assign(c->ncolors, std::vector<int>(ncta + 1, 0));
        std::vector<long long> slots(ncta, 0), grps(ncta, 0);
        const char* pe = getenv("VBD_RES_PLAN");  // "count": equal group counts (tuning)
        const bool by_count = pe && std::string(pe) == "count";
        auto cost = [&](const G& g) { return by_count ? 1LL : (long long)g.rounds + 2; };
        for (int col = 0; col < c->ncolors; ++col) {
            const auto& gs = cg[col];
            long long tot = 0;
            for (const G& g : gs) tot += cost(g);
            long long acc = 0;
            int k = 0;
            for (int i = 0; i < (int)gs.size(); ++i) {
                while (k < ncta - 1 && acc * ncta >= tot * (k + 1)) cut[col][++k] = i;
                acc += cost(gs[i]);
                slots[k] += 32LL * gs[i].rounds;
                grps[k] += 1;
            }
            while (k < ncta - 1) cut[col][++k] = (int)gs.size();
            cut[col][ncta] = (int)gs.size();
        }
        slot_cap = (int)*std::max_element(slots.begin(), slots.end());
        grp_cap = (int)std::max<long long>(1, *std::max_element(grps.begin(), grps.end()));
    };
    auto smem_of = [&](bool repl, int slot_cap, int grp_cap) {
        ResSmem<R> L{(int)c->nkinds, (int)c->n, slot_cap, grp_cap, c->ncolors, repl};
        return L.total();
    };
    std::vector<std::vector<int>> cut;
    int slot_cap = 0, grp_cap = 0, mode = 0, ncta = 0;
    const size_t budget = (size_t)smem_max - 2048;
    const char* cle = getenv("VBD_RES_CL");  // cluster size (16 or 8; tuning)
    const int cl_first = cle && atoi(cle) == 8 ? 8 : 16;
    if (want != "glob") {
        for (int cl : {cl_first, 8}) {
            plan(cl, cut, slot_cap, grp_cap);
            if (smem_of(true, slot_cap, grp_cap) > budget) continue;
            auto k = (c->vmat.p && c->uniform_mat) ? k_step_resident<R, true, true> : k_step_resident<R, false, true>;
            const size_t sm = smem_of(true, slot_cap, grp_cap);
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            if (cl > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(VBD_RES_THREADS);
            cfg.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg) != cudaSuccess || nclusters < 1) {
                cudaGetLastError();
                continue;
            }
            mode = 1;
            ncta = cl;
            break;
        }
    }
    // GLOB by default for fp32 scenes whose colours are small enough for the per-colour graph to
    // be launch-bound (C2, 12.7k vertices per colour: 2.13 -> 1.91 ms/step) but too large for
    // one cluster's replica; C3 (24k per colour) is faster on the graph (2.61 vs 2.90)
    long long cmax = 0;
    for (int col = 0; col < c->ncolors; ++col) cmax = std::max(cmax, c->ccnt[col]);
    const char* gme = getenv("VBD_RES_GLOB_MAX");
    const long long glob_max = gme && *gme ? atoll(gme) : 18000;
    const bool glob_auto = want.empty() && sizeof(R) == 4 && cmax <= glob_max;
    if (!mode && (want == "glob" || glob_auto)) {
        ncta = sms;
        plan(ncta, cut, slot_cap, grp_cap);
        const size_t sm = smem_of(false, slot_cap, grp_cap);
        if (sm <= budget) {
            auto k = (c->vmat.p && c->uniform_mat) ? k_step_resident<R, true, false> : k_step_resident<R, false, false>;
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            int per = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, VBD_RES_THREADS, sm));
            if (per >= 1) mode = 2;
        }
    }
    if (!mode) return;
    // per-CTA arrays
    std::vector<int4> slots;
    std::vector<long long> slot_beg(ncta + 1, 0);
    std::vector<ResGroup> groups;
    std::vector<int> grp_beg(ncta + 1, 0), col_grp((size_t)ncta * (c->ncolors + 1), 0);
    const int nk = (int)c->nkinds, npad = (int)c->n;
    for (int k = 0; k < ncta; ++k) {
        slot_beg[k] = (long long)slots.size();
        grp_beg[k] = (int)groups.size();
        int sb = 0;
        for (int col = 0; col < c->ncolors; ++col) {
            col_grp[(size_t)k * (c->ncolors + 1) + col] = (int)groups.size() - grp_beg[k];
            for (int i = cut[col][k]; i < cut[col][k + 1]; ++i) {
                const G& g = cg[col][i];
                groups.push_back(ResGroup{g.v0, g.nv, sb, g.rounds});
                for (int r = 0; r < g.rounds; ++r)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int vi = lane & 7, j = lane >> 3, pos = 4 * r + j;
                        int4 sl = make_int4(npad, npad, npad, nk);
                        if (vi < g.nv) {
                            const long long e0 = eoff[g.v0 + vi], d = eoff[g.v0 + vi + 1] - e0;
                            if (pos < d) sl = ent[(size_t)(e0 + pos)];
                        }
                        slots.push_back(sl);
                    }
                sb += 32 * g.rounds;
            }
        }
        col_grp[(size_t)k * (c->ncolors + 1) + c->ncolors] = (int)groups.size() - grp_beg[k];
    }
    slot_beg[ncta] = (long long)slots.size();
    grp_beg[ncta] = (int)groups.size();
    // REPL push sets: CTA k reads v if v is one of its vertices, a neighbour of one of them, or
    // in its K3 / K4 chunk [n k / ncta, n (k + 1) / ncta)  (VBD_RES_PUSH=all: every CTA)
    std::vector<unsigned short> push((size_t)c->n, 0);
    const char* pe = getenv("VBD_RES_PUSH");
    const bool push_all = pe && std::string(pe) == "all";
    for (int k = 0; k < ncta; ++k) {
        const unsigned short bit = (unsigned short)(1u << k);
        const long long lo = c->n * k / ncta, hi = c->n * (k + 1) / ncta;
        for (long long v = lo; v < hi; ++v) push[v] |= bit;
        for (int gi = grp_beg[k]; gi < grp_beg[k + 1]; ++gi) {
            const ResGroup& g = groups[gi];
            for (int vi = 0; vi < g.nv; ++vi) push[g.v0 + vi] |= bit;
        }
        for (long long q = slot_beg[k]; q < slot_beg[k + 1]; ++q) {
            const int4 sl = slots[q];
            for (int id : {sl.x, sl.y, sl.z})
                if (id < npad) push[id] |= bit;
        }
    }
    if (push_all || ncta > 16)
        for (auto& m : push) m = (unsigned short)((1u << std::min(ncta, 16)) - 1);
    if (slots.empty()) slots.push_back(make_int4(npad, npad, npad, nk));
    upload(c->res_slots, slots.data(), slots.size(), s);
    upload(c->res_slot_beg, slot_beg.data(), slot_beg.size(), s);
    upload(c->res_groups, groups.data(), std::max<size_t>(groups.size(), 1), s);
    upload(c->res_grp_beg, grp_beg.data(), grp_beg.size(), s);
    upload(c->res_col_grp, col_grp.data(), col_grp.size(), s);
    upload(c->res_push, push.data(), std::max<size_t>(push.size(), 1), s);
    if (getenv("VBD_RES_DBG") && (atoi(getenv("VBD_RES_DBG")) & 8))  // diagnostics: pass timeline
        c->res_prof.alloc((size_t)40 * (4096 * (c->ncolors + 1) + 1));
    c->res_bar.alloc(16);
    CK(cudaMemsetAsync(c->res_bar.p, 0, 16, s));
    CK(cudaStreamSynchronize(s));
    c->res_mode = mode;
    c->res_ncta = ncta;
    c->res_slot_cap = slot_cap;
    c->res_grp_cap = grp_cap;
    c->res_smem = smem_of(mode == 1, slot_cap, grp_cap);
}

template <typename R> void launch_resident(vbd_ctx* c)
{
    ResArgs<R> ra;
    ra.a = k1_args<R>(c, c->cur.eps_det, 0, c->cur.rho == 0.0, 0);
    ra.s = step_args<R>(c);
    ra.slots = c->res_slots.as<int4>();
    ra.slot_beg = c->res_slot_beg.as<long long>();
    ra.groups = c->res_groups.as<ResGroup>();
    ra.grp_beg = c->res_grp_beg.as<int>();
    ra.col_grp = c->res_col_grp.as<int>();
    ra.ncolors = c->ncolors;
    ra.n_max = c->cur.n_max;
    ra.cheb = c->cur.rho != 0.0;
    ra.omegas = c->omega_dev.as<double>();
    ra.nkinds = (int)c->nkinds;
    ra.slot_cap = c->res_slot_cap;
    ra.grp_cap = c->res_grp_cap;
    ra.bar = c->res_bar.as<unsigned>();
    ra.ncta = c->res_ncta;
    ra.push = c->res_push.as<unsigned short>();
    ra.dbg = getenv("VBD_RES_DBG") ? atoi(getenv("VBD_RES_DBG")) : 0;
    if (ra.dbg & 3) ra.a.flag = ra.s.flag = nullptr;  // (garbage positions in the timing experiments)
    ra.prof = nullptr;
    if ((ra.dbg & 8) && c->res_prof.bytes >= (size_t)40 * (c->cur.n_max * (c->ncolors + 1) + 1))
        ra.prof = c->res_prof.as<long long>();  // CTA 0's pass timeline (vbd_resident_timeline)
    const bool um = c->vmat.p && c->uniform_mat;
    const bool repl = c->res_mode == 1;
    void (*k)(const ResArgs<R>) = repl ? (um ? k_step_resident<R, true, true> : k_step_resident<R, false, true>)
                                       : (um ? k_step_resident<R, true, false> : k_step_resident<R, false, false>);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->res_ncta);
    cfg.blockDim = dim3(VBD_RES_THREADS);
    cfg.dynamicSmemBytes = c->res_smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    if (repl) {
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c->res_ncta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
    } else {
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, ra));
}

// one cooperative launch per step (small scenes); see k_step_persistent
bool use_persistent(const vbd_ctx* c)
{
    const char* e = getenv("VBD_PERSIST");
    if (c->has_extras || c->ncontacts) return false;
    if (e && *e) return atoi(e) != 0 && c->inplace && c->ncolors <= VBD_PERSIST_MAX_COLORS;
    // measured on B200: grid.sync() costs more than a graph-node launch (C1 0.36 vs 0.25
    // ms/step), so the per-colour graph is the default everywhere
    return false;
}

template <typename R> void launch_step_persistent(vbd_ctx* c)
{
    PersistArgs<R> pa;
    pa.k1 = k1_args<R>(c, c->cur.eps_det, 0, c->cur.rho == 0.0, 0);
    pa.s = step_args<R>(c);
    pa.ncolors = c->ncolors;
    for (int k = 0; k < c->ncolors; ++k) {
        pa.cbeg[k] = (int)c->cbeg[k];
        pa.ccnt[k] = (int)c->ccnt[k];
    }
    pa.n_max = c->cur.n_max;
    pa.chebyshev = c->cur.rho != 0.0;
    pa.omegas = c->omega_dev.as<double>();
    static int grid_cache[2] = {0, 0};
    int& grid = grid_cache[sizeof(R) == 8 ? 1 : 0];
    if (!grid) {
        int dev = 0, sms = 148, per = 1;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_step_persistent<R, 4, 2>, 256, 0));
        grid = std::max(1, per) * sms;
    }
    void* args[] = {&pa};
    CK(cudaLaunchCooperativeKernel((const void*)k_step_persistent<R, 4, 2>, dim3(grid), dim3(256),
                                   args, 0, c->stream));
}

void validate_params(const vbd_step_params* p)
{
    if (!p) fail(VBD_ERR_ARG, "params is NULL");
    if (!(p->h > 0.0)) fail(VBD_ERR_ARG, "h must be positive");
    if (p->n_max < 1 || p->n_max > 65535) fail(VBD_ERR_ARG, "n_max must be in [1, 65535]");
    if (!(p->rho >= 0.0 && p->rho < 1.0)) fail(VBD_ERR_ARG, "rho must be in [0, 1)");
    if (!(p->eps_det >= 0.0)) fail(VBD_ERR_ARG, "eps_det must be >= 0");
    if (p->init_mode < 0 || p->init_mode > 3) fail(VBD_ERR_ARG, "bad init_mode");
}

void read_result(vbd_ctx* c, vbd_step_result* res)
{
    unsigned long long f = read_scalar<unsigned long long>(c->flag.p, c->stream);
    if (!res) return;
    std::memset(res, 0, sizeof *res);
    res->vertex = -1;
    if (f != StepFlag::NONE) {
        res->nonfinite = 1;
        res->step = (int)((f >> 48) & 0xffff);
        res->iteration = (int)((f >> 32) & 0xffff);
        res->vertex = (long long)(f & 0xffffffffull);
    }
}

// ---------------------------------------------------------------------------------------
// device contact detection (vbd_contact.cuh) and the contact step

template <typename R> CollArgs<R> coll_args(vbd_ctx* c, const DBuf& xs, const DBuf& xe, double margin)
{
    CollArgs<R> a;
    a.sv = c->csv.as<int>();
    a.tri = c->ctri.as<int4>();
    a.edge = c->cedge.as<int2>();
    a.nsv = c->nsv;
    a.ntri = c->ntri;
    a.nedge = c->nedge;
    a.active = c->cactive.as<unsigned char>();
    a.xs = xs.as<typename Vec4<R>::T>();
    a.xe = xe.as<typename Vec4<R>::T>();
    a.cell = c->coll_cell;
    a.pad = margin + 1e-12 * c->coll_cell;
    return a;
}

// cells of primitives `what` (0 vertex, 1 triangle, 2 edge), sorted by key
template <typename R> long long grid_cells(vbd_ctx* c, const CollArgs<R>& a, int what, int n, DBuf& key, DBuf& own)
{
    cudaStream_t s = c->stream;
    DBuf cnt, off;
    cnt.alloc_on((size_t)std::max(n, 1) * 8, s);
    if (n) k_cell_count<R><<<blocks_for(n), 256, 0, s>>>(a, what, n, cnt.as<long long>());
    CK(cudaGetLastError());
    exclusive_offsets(cnt.as<long long>(), n, off, s);
    const long long m = read_scalar<long long>(off.as<long long>() + n, s);
    key.alloc_on((size_t)std::max<long long>(m, 1) * 8, s);
    own.alloc_on((size_t)std::max<long long>(m, 1) * 4, s);
    if (n) k_cell_emit<R><<<blocks_for(n), 256, 0, s>>>(a, what, n, off.as<long long>(), key.as<unsigned long long>(),
                                                        own.as<int>());
    CK(cudaGetLastError());
    if (m) sort_pairs_u64_i32(key, own, m, s);
    c->mx_cell[what] = std::max(c->mx_cell[what], m);
    return m;
}

void unique_u64(DBuf& keys, long long& n, cudaStream_t s)
{
    if (n == 0) return;
    DBuf out, nsel, tmp;
    out.alloc_on((size_t)n * 8, s);
    nsel.alloc_on(8, s);
    size_t tb = 0;
    CK(cub::DeviceSelect::Unique(nullptr, tb, keys.as<unsigned long long>(), out.as<unsigned long long>(),
                                 nsel.as<long long>(), (int64_t)n, s));
    tmp.alloc_on(tb, s);
    CK(cub::DeviceSelect::Unique(tmp.p, tb, keys.as<unsigned long long>(), out.as<unsigned long long>(),
                                 nsel.as<long long>(), (int64_t)n, s));
    n = read_scalar<long long>(nsel.p, s);
    keys.swap(out);
}

// candidate codes (ascending, unique): vertex-triangle k * ntri + t, or edge-edge e * nedge + o
template <typename R> long long broad_phase(vbd_ctx* c, const CollArgs<R>& a, bool ee, DBuf& codes)
{
    cudaStream_t s = c->stream;
    DBuf qk, qo, tk, to;
    long long nq, nt;
    if (ee) {
        nt = grid_cells<R>(c, a, 2, a.nedge, tk, to);
        nq = nt;
    } else {
        nt = grid_cells<R>(c, a, 1, a.ntri, tk, to);
        nq = grid_cells<R>(c, a, 0, a.nsv, qk, qo);
    }
    const unsigned long long* qkey = ee ? tk.as<unsigned long long>() : qk.as<unsigned long long>();
    const int* qown = ee ? to.as<int>() : qo.as<int>();
    const long long width = ee ? a.nedge : a.ntri;
    DBuf cnt, off;
    cnt.alloc_on((size_t)std::max<long long>(nq, 1) * 8, s);
    if (nq) {
        if (ee) k_cell_join<false, true><<<blocks_for(nq), 256, 0, s>>>(qkey, qown, nq, tk.as<unsigned long long>(), to.as<int>(), nt, width, cnt.as<long long>(), nullptr, nullptr);
        else k_cell_join<false, false><<<blocks_for(nq), 256, 0, s>>>(qkey, qown, nq, tk.as<unsigned long long>(), to.as<int>(), nt, width, cnt.as<long long>(), nullptr, nullptr);
    }
    CK(cudaGetLastError());
    exclusive_offsets(cnt.as<long long>(), nq, off, s);
    long long m = read_scalar<long long>(off.as<long long>() + nq, s);
    c->mx_join[ee ? 1 : 0] = std::max(c->mx_join[ee ? 1 : 0], m);
    codes.alloc_on((size_t)std::max<long long>(m, 1) * 8, s);
    if (nq && m) {
        if (ee) k_cell_join<true, true><<<blocks_for(nq), 256, 0, s>>>(qkey, qown, nq, tk.as<unsigned long long>(), to.as<int>(), nt, width, nullptr, off.as<long long>(), codes.as<unsigned long long>());
        else k_cell_join<true, false><<<blocks_for(nq), 256, 0, s>>>(qkey, qown, nq, tk.as<unsigned long long>(), to.as<int>(), nt, width, nullptr, off.as<long long>(), codes.as<unsigned long long>());
    }
    CK(cudaGetLastError());
    if (m) {
        sort_keys_u64(codes, m, s);
        unique_u64(codes, m, s);
    }
    return m;
}

__global__ void k_drop_known(const unsigned long long* __restrict__ codes, long long n,
                             const unsigned long long* __restrict__ known, long long nk, int* acc)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n || !acc[i] || nk == 0) return;
    const long long j = lower_key(known, nk, codes[i]);
    if (j < nk && known[j] == codes[i]) acc[i] = 0;  // already tracked by DCD (update_ccd)
}

template <typename T>
__global__ void k_compact(const T* __restrict__ in, const int* __restrict__ acc, const long long* __restrict__ off,
                          long long n, T* __restrict__ out)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n && acc[i]) out[off[i]] = in[i];
}

// keep the accepted records (and codes) in candidate order
long long compact_recs(vbd_ctx* c, const DBuf& recs, const DBuf& codes, const DBuf& acc, long long n, DBuf& out_recs,
                       DBuf* out_codes)
{
    cudaStream_t s = c->stream;
    DBuf off;
    exclusive_offsets(acc.as<int>(), n, off, s);
    const long long m = read_scalar<long long>(off.as<long long>() + n, s);
    out_recs.alloc_on((size_t)std::max<long long>(m, 1) * sizeof(ContactRec), s);
    if (n) k_compact<ContactRec><<<blocks_for(n), 256, 0, s>>>(recs.as<ContactRec>(), acc.as<int>(), off.as<long long>(), n, out_recs.as<ContactRec>());
    if (out_codes) {
        out_codes->alloc((size_t)std::max<long long>(m, 1) * 8);
        if (n) k_compact<unsigned long long><<<blocks_for(n), 256, 0, s>>>(codes.as<unsigned long long>(), acc.as<int>(), off.as<long long>(), n, out_codes->as<unsigned long long>());
    }
    CK(cudaGetLastError());
    return m;
}

// DCD at x_t (solver.py:241-260): the step's DCD records; clears the colliding flags
template <typename R> void detect_dcd(vbd_ctx* c)
{
    cudaStream_t s = c->stream;
    const CollArgs<R> a = coll_args<R>(c, c->xt, c->xt, c->coll_dcd_r);
    DBuf codes, recs, acc;
    const long long n = broad_phase<R>(c, a, false, codes);
    recs.alloc_on((size_t)std::max<long long>(n, 1) * sizeof(ContactRec), s);
    acc.alloc_on((size_t)std::max<long long>(n, 1) * 4, s);
    if (n) k_dcd_vt<R><<<blocks_for(n, 128), 128, 0, s>>>(a, codes.as<unsigned long long>(), n, c->coll_dcd_r, c->coll_kc,
                                                     c->coll_has_max_depth, c->coll_max_depth, recs.as<ContactRec>(),
                                                     acc.as<int>());
    CK(cudaGetLastError());
    c->ndcd = compact_recs(c, recs, codes, acc, n, c->dcd_recs, &c->dcd_codes);
    c->nccd = 0;
    CK(cudaMemsetAsync(c->ccoll.p, 0, c->n, s));
}

// CCD between x_t and the current iterate (solver.py:263-279): vertex-triangle then edge-edge
template <typename R> void detect_ccd(vbd_ctx* c)
{
    cudaStream_t s = c->stream;
    const CollArgs<R> a = coll_args<R>(c, c->xt, c->pos, 0.0);
    DBuf vcodes, vrecs, vacc, ecodes, erecs, eacc, vt_out, ee_out;
    const long long nv = broad_phase<R>(c, a, false, vcodes);
    vrecs.alloc_on((size_t)std::max<long long>(nv, 1) * sizeof(ContactRec), s);
    vacc.alloc_on((size_t)std::max<long long>(nv, 1) * 4, s);
    if (nv) {
        k_ccd_vt<R><<<blocks_for(nv, 128), 128, 0, s>>>(a, vcodes.as<unsigned long long>(), nv, c->coll_kc, vrecs.as<ContactRec>(), vacc.as<int>());
        k_drop_known<<<blocks_for(nv), 256, 0, s>>>(vcodes.as<unsigned long long>(), nv, c->dcd_codes.as<unsigned long long>(), c->ndcd, vacc.as<int>());
    }
    CK(cudaGetLastError());
    const long long mv = compact_recs(c, vrecs, vcodes, vacc, nv, vt_out, nullptr);
    const long long ne = a.nedge ? broad_phase<R>(c, a, true, ecodes) : 0;
    erecs.alloc_on((size_t)std::max<long long>(ne, 1) * sizeof(ContactRec), s);
    eacc.alloc_on((size_t)std::max<long long>(ne, 1) * 4, s);
    if (ne) k_ccd_ee<R><<<blocks_for(ne, 128), 128, 0, s>>>(a, ecodes.as<unsigned long long>(), ne, c->coll_kc, erecs.as<ContactRec>(), eacc.as<int>());
    CK(cudaGetLastError());
    const long long me = compact_recs(c, erecs, ecodes, eacc, ne, ee_out, nullptr);
    c->nccd = mv + me;
    c->ccd_recs.alloc_on((size_t)std::max<long long>(c->nccd, 1) * sizeof(ContactRec), s);
    if (mv) CK(cudaMemcpyAsync(c->ccd_recs.p, vt_out.p, mv * sizeof(ContactRec), cudaMemcpyDeviceToDevice, s));
    if (me) CK(cudaMemcpyAsync(c->ccd_recs.as<ContactRec>() + mv, ee_out.p, me * sizeof(ContactRec), cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
}

// mark_flags at `x` and compile the DCD + CCD records into the K1 contact arrays
template <typename R> void compile_contact_set(vbd_ctx* c, const DBuf& x)
{
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    const long long n = c->ndcd + c->nccd;
    DBuf all;
    all.alloc_on((size_t)std::max<long long>(n, 1) * sizeof(ContactRec), s);
    if (c->ndcd) CK(cudaMemcpyAsync(all.p, c->dcd_recs.p, c->ndcd * sizeof(ContactRec), cudaMemcpyDeviceToDevice, s));
    if (c->nccd) CK(cudaMemcpyAsync(all.as<ContactRec>() + c->ndcd, c->ccd_recs.p, c->nccd * sizeof(ContactRec), cudaMemcpyDeviceToDevice, s));
    c->ncontacts = n;
    if (n == 0) return;
    k_mark_flags<R><<<blocks_for(n), 256, 0, s>>>(all.as<ContactRec>(), (int)n, x.as<R4>(), c->ccoll.as<unsigned char>());
    c->cidx.alloc_on((size_t)n * sizeof(int4), s);
    c->creal.alloc_on((size_t)n * 4 * sizeof(R4), s);
    DBuf inc, dummy;
    inc.alloc_on((size_t)n * 4 * 8, s);
    k_pack_contacts<R><<<blocks_for(n), 256, 0, s>>>(all.as<ContactRec>(), (int)n, c->cidx.as<int4>(), c->creal.as<R4>(),
                                                     inc.as<unsigned long long>());
    CK(cudaGetLastError());
    sort_keys_u64(inc, 4 * n, s);
    // incidence of solved vertices only (keys of fixed / ghost vertices sort last)
    c->coff.alloc_on((size_t)(c->nsolve + 1) * 8, s);
    c->ccid.alloc_on((size_t)4 * n * 4, s);
    c->cslot.alloc_on((size_t)4 * n * 4, s);
    k_contact_csr<<<blocks_for(4 * n), 256, 0, s>>>(inc.as<unsigned long long>(), 4 * n, c->nsolve, c->coff.as<long long>(),
                                                   c->ccid.as<int>(), c->cslot.as<int>());
    CK(cudaGetLastError());
    c->mu_c = c->mu_c;
}

// ---- graph-mode contact step ----------------------------------------------------------------
// The host path above reads every data-dependent size back (about 8 synchronisations per
// detection).  Graph mode runs the same kernels at fixed capacities with sentinel-padded
// tails (vbd_contact.cuh), so DCD, every CCD, the contact-set compile, the colour passes, K3
// and K4 of a step are ONE captured CUDA graph and the step costs one synchronisation (the
// result read).  Capacities come from the largest counts the host path has seen (2x + 1024);
// a step whose counts exceed them raises a device flag, is rolled back (x_t, v_t, v_prev,
// the step counter) and redone on the host path, which then grows the capacities.
// Records keep the host path's relative order (DCD, CCD vertex-triangle, CCD edge-edge, each
// compacted in candidate order), so the per-vertex contact sums -- and the results -- are
// bitwise those of the host path.  VBD_CONTACT_GRAPH=0 keeps the host path.

struct CgLayout {
    long long capQ, capT, capJ0, capJ1, capAll;  // sv cells, tri / edge cells, vt / ee candidates
};
inline CgLayout cg_layout(const vbd_ctx* c)
{
    CgLayout L;
    L.capQ = std::max<long long>(c->cap_cell[0], 1);
    L.capT = std::max<long long>(std::max(c->cap_cell[1], c->cap_cell[2]), 1);
    L.capJ0 = std::max<long long>(c->cap_join[0], 1);
    L.capJ1 = c->nedge ? std::max<long long>(c->cap_join[1], 1) : 0;
    L.capAll = 2 * L.capJ0 + L.capJ1;
    return L;
}

template <typename R> void cg_setup(vbd_ctx* c)
{
    for (int w = 0; w < 3; ++w) c->cap_cell[w] = 2 * c->mx_cell[w] + 1024;
    for (int w = 0; w < 2; ++w) c->cap_join[w] = 2 * c->mx_join[w] + 1024;
    const CgLayout L = cg_layout(c);
    const long long capJ = std::max(L.capJ0, L.capJ1);
    const long long nprim = std::max<long long>(std::max(c->nsv, c->ntri), std::max(c->nedge, 1));
    c->cg_cnt.alloc((size_t)nprim * 8);
    c->cg_off.alloc((size_t)(nprim + 1) * 8);
    c->cg_key_q.alloc((size_t)L.capQ * 8);
    c->cg_own_q.alloc((size_t)L.capQ * 4);
    c->cg_key_t.alloc((size_t)L.capT * 8);
    c->cg_own_t.alloc((size_t)L.capT * 4);
    const long long capK = std::max(L.capQ, L.capT);
    c->cg_jcnt.alloc((size_t)capK * 8);
    c->cg_joff.alloc((size_t)(capK + 1) * 8);
    c->cg_codes.alloc((size_t)capJ * 8);
    c->cg_codes2.alloc((size_t)std::max(capJ, capK) * 8);  // unsorted codes / unsorted cell keys
    c->cg_nsel.alloc(8);
    c->cg_recs.alloc((size_t)capJ * sizeof(ContactRec));
    c->cg_acc.alloc((size_t)std::max(capJ, capK) * 4);     // narrow-phase accept / unsorted owners
    c->cg_aoff.alloc((size_t)(capJ + 1) * 8);
    c->cg_dcd_codes.alloc((size_t)L.capJ0 * 8);
    c->cg_all.alloc((size_t)L.capAll * sizeof(ContactRec));  // [DCD | CCD vt | CCD ee]
    c->cg_inc.alloc((size_t)4 * L.capAll * 8);
    c->cg_inc2.alloc((size_t)4 * L.capAll * 8);
    c->cg_flag.alloc(16);
    c->cidx.alloc((size_t)L.capAll * sizeof(int4));
    c->creal.alloc((size_t)L.capAll * 4 * sizeof(typename Vec4<R>::T));
    c->coff.alloc((size_t)(c->nsolve + 1) * 8);
    c->ccid.alloc((size_t)4 * L.capAll * 4);
    c->cslot.alloc((size_t)4 * L.capAll * 4);
    c->cg_snap.alloc((size_t)3 * c->n * c->r4() + 16);
    // CUB temporary storage: the largest of every scan / sort / unique of a step
    size_t mx = 0, tb = 0;
    const long long nscan = std::max(std::max(nprim, capK), capJ);
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, (const long long*)nullptr, (long long*)nullptr, (int64_t)nscan));
    mx = std::max(mx, tb);
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, (const int*)nullptr, (long long*)nullptr, (int64_t)nscan));
    mx = std::max(mx, tb);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                       (const int*)nullptr, (int*)nullptr, (int64_t)capK, 0, 64));
    mx = std::max(mx, tb);
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                      (int64_t)std::max(capJ, 4 * L.capAll), 0, 64));
    mx = std::max(mx, tb);
    CK(cub::DeviceSelect::Unique(nullptr, tb, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                 (long long*)nullptr, (int64_t)capJ));
    mx = std::max(mx, tb);
    c->cg_tmp.alloc(mx);
    if (c->cg_exec) {
        cudaGraphExecDestroy(c->cg_exec);
        c->cg_exec = nullptr;
    }
    c->cg_ready = true;
}

// out[0] = 0, out[1..n] = inclusive sum (capture-safe: preallocated temp, no synchronisation)
template <typename In> void cg_scan(vbd_ctx* c, const In* in, long long n, long long* out)
{
    CK(cudaMemsetAsync(out, 0, 8, c->stream));
    if (n <= 0) return;
    size_t tb = c->cg_tmp.bytes;
    CK(cub::DeviceScan::InclusiveSum(c->cg_tmp.p, tb, in, out + 1, (int64_t)n, c->stream));
}

// sorted, sentinel-padded cells of primitives `what` (capacity cap) into key / own
template <typename R>
void cg_cells(vbd_ctx* c, const CollArgs<R>& a, int what, int n, long long cap, DBuf& key, DBuf& own)
{
    cudaStream_t s = c->stream;
    unsigned long long* kt = c->cg_codes2.as<unsigned long long>();
    int* ot = c->cg_acc.as<int>();
    long long* off = c->cg_off.as<long long>();
    if (n) k_cell_count<R><<<blocks_for(n), 256, 0, s>>>(a, what, n, c->cg_cnt.as<long long>());
    cg_scan(c, c->cg_cnt.as<long long>(), n, off);
    if (n) k_cell_emit<R><<<blocks_for(n), 256, 0, s>>>(a, what, n, off, kt, ot, cap);
    k_sent_tail<<<blocks_for(cap), 256, 0, s>>>(kt, ot, off + n, cap, c->cg_flag.as<int>());
    size_t tb = c->cg_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(c->cg_tmp.p, tb, kt, key.as<unsigned long long>(), ot, own.as<int>(),
                                       (int64_t)cap, 0, 64, s));
}

// candidate codes (sorted, unique, sentinel tail) of capacity capJ into c->cg_codes
template <typename R> void cg_broad(vbd_ctx* c, const CollArgs<R>& a, bool ee, long long capJ, const CgLayout& L)
{
    cudaStream_t s = c->stream;
    long long nq, nt;
    if (ee) {
        cg_cells<R>(c, a, 2, a.nedge, L.capT, c->cg_key_t, c->cg_own_t);
        nq = nt = L.capT;
    } else {
        cg_cells<R>(c, a, 1, a.ntri, L.capT, c->cg_key_t, c->cg_own_t);
        cg_cells<R>(c, a, 0, a.nsv, L.capQ, c->cg_key_q, c->cg_own_q);
        nq = L.capQ;
        nt = L.capT;
    }
    const unsigned long long* qk = (ee ? c->cg_key_t : c->cg_key_q).as<unsigned long long>();
    const int* qo = (ee ? c->cg_own_t : c->cg_own_q).as<int>();
    const unsigned long long* tk = c->cg_key_t.as<unsigned long long>();
    const int* to = c->cg_own_t.as<int>();
    const long long width = ee ? a.nedge : a.ntri;
    long long* jc = c->cg_jcnt.as<long long>();
    long long* jo = c->cg_joff.as<long long>();
    unsigned long long* raw = c->cg_codes2.as<unsigned long long>();
    if (ee) k_cell_join<false, true><<<blocks_for(nq), 256, 0, s>>>(qk, qo, nq, tk, to, nt, width, jc, nullptr, nullptr);
    else k_cell_join<false, false><<<blocks_for(nq), 256, 0, s>>>(qk, qo, nq, tk, to, nt, width, jc, nullptr, nullptr);
    cg_scan(c, jc, nq, jo);
    if (ee) k_cell_join<true, true><<<blocks_for(nq), 256, 0, s>>>(qk, qo, nq, tk, to, nt, width, nullptr, jo, raw, capJ);
    else k_cell_join<true, false><<<blocks_for(nq), 256, 0, s>>>(qk, qo, nq, tk, to, nt, width, nullptr, jo, raw, capJ);
    k_sent_tail<<<blocks_for(capJ), 256, 0, s>>>(raw, nullptr, jo + nq, capJ, c->cg_flag.as<int>());
    size_t tb = c->cg_tmp.bytes;
    unsigned long long* sorted = c->cg_inc2.as<unsigned long long>();  // free until the compile
    CK(cub::DeviceRadixSort::SortKeys(c->cg_tmp.p, tb, raw, sorted, (int64_t)capJ, 0, 64, s));
    tb = c->cg_tmp.bytes;
    CK(cub::DeviceSelect::Unique(c->cg_tmp.p, tb, sorted, c->cg_codes.as<unsigned long long>(),
                                 c->cg_nsel.as<long long>(), (int64_t)capJ, s));
    k_sent_tail<<<blocks_for(capJ), 256, 0, s>>>(c->cg_codes.as<unsigned long long>(), nullptr,
                                                 c->cg_nsel.as<long long>(), capJ, nullptr);
}

// accepted records (and codes) in candidate order into out (capacity capJ, idx.x = -1 tail)
inline void cg_compact(vbd_ctx* c, long long capJ, ContactRec* out, unsigned long long* out_codes)
{
    cudaStream_t s = c->stream;
    CK(cudaMemsetAsync(out, 0xff, (size_t)capJ * sizeof(ContactRec), s));
    cg_scan(c, c->cg_acc.as<int>(), capJ, c->cg_aoff.as<long long>());
    k_compact<ContactRec><<<blocks_for(capJ), 256, 0, s>>>(c->cg_recs.as<ContactRec>(), c->cg_acc.as<int>(),
                                                        c->cg_aoff.as<long long>(), capJ, out);
    if (out_codes) {
        CK(cudaMemsetAsync(out_codes, 0xff, (size_t)capJ * 8, s));
        k_compact<unsigned long long><<<blocks_for(capJ), 256, 0, s>>>(c->cg_codes.as<unsigned long long>(),
                                                                       c->cg_acc.as<int>(), c->cg_aoff.as<long long>(),
                                                                       capJ, out_codes);
    }
}

template <typename R> void cg_detect_dcd(vbd_ctx* c, const CgLayout& L)
{
    cudaStream_t s = c->stream;
    const CollArgs<R> a = coll_args<R>(c, c->xt, c->xt, c->coll_dcd_r);
    cg_broad<R>(c, a, false, L.capJ0, L);
    CK(cudaMemsetAsync(c->cg_acc.p, 0, (size_t)L.capJ0 * 4, s));
    k_dcd_vt<R><<<blocks_for(L.capJ0, 128), 128, 0, s>>>(a, c->cg_codes.as<unsigned long long>(), L.capJ0, c->coll_dcd_r,
                                                       c->coll_kc, c->coll_has_max_depth, c->coll_max_depth,
                                                       c->cg_recs.as<ContactRec>(), c->cg_acc.as<int>());
    ContactRec* all = c->cg_all.as<ContactRec>();
    cg_compact(c, L.capJ0, all, c->cg_dcd_codes.as<unsigned long long>());
    CK(cudaMemsetAsync(all + L.capJ0, 0xff, (size_t)(L.capJ0 + L.capJ1) * sizeof(ContactRec), s));  // no CCD yet
    CK(cudaMemsetAsync(c->ccoll.p, 0, c->n, s));
}

template <typename R> void cg_detect_ccd(vbd_ctx* c, const CgLayout& L)
{
    cudaStream_t s = c->stream;
    const CollArgs<R> a = coll_args<R>(c, c->xt, c->pos, 0.0);
    ContactRec* all = c->cg_all.as<ContactRec>();
    cg_broad<R>(c, a, false, L.capJ0, L);
    CK(cudaMemsetAsync(c->cg_acc.p, 0, (size_t)L.capJ0 * 4, s));
    k_ccd_vt<R><<<blocks_for(L.capJ0, 128), 128, 0, s>>>(a, c->cg_codes.as<unsigned long long>(), L.capJ0, c->coll_kc,
                                                       c->cg_recs.as<ContactRec>(), c->cg_acc.as<int>());
    k_drop_known<<<blocks_for(L.capJ0), 256, 0, s>>>(c->cg_codes.as<unsigned long long>(), L.capJ0,
                                                    c->cg_dcd_codes.as<unsigned long long>(), L.capJ0, c->cg_acc.as<int>());
    cg_compact(c, L.capJ0, all + L.capJ0, nullptr);
    if (L.capJ1) {
        cg_broad<R>(c, a, true, L.capJ1, L);
        CK(cudaMemsetAsync(c->cg_acc.p, 0, (size_t)L.capJ1 * 4, s));
        k_ccd_ee<R><<<blocks_for(L.capJ1, 128), 128, 0, s>>>(a, c->cg_codes.as<unsigned long long>(), L.capJ1, c->coll_kc,
                                                           c->cg_recs.as<ContactRec>(), c->cg_acc.as<int>());
        cg_compact(c, L.capJ1, all + 2 * L.capJ0, nullptr);
    }
}

// mark_flags at x and the K1 contact arrays of [DCD | CCD vt | CCD ee] (sentinel records skip)
template <typename R> void cg_compile(vbd_ctx* c, const DBuf& x, const CgLayout& L)
{
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    const long long n = L.capAll;
    const ContactRec* all = c->cg_all.as<ContactRec>();
    k_mark_flags<R><<<blocks_for(n), 256, 0, s>>>(all, (int)n, x.as<R4>(), c->ccoll.as<unsigned char>());
    CK(cudaMemsetAsync(c->cidx.p, 0xff, (size_t)n * sizeof(int4), s));
    k_pack_contacts<R><<<blocks_for(n), 256, 0, s>>>(all, (int)n, c->cidx.as<int4>(), c->creal.as<R4>(),
                                                     c->cg_inc.as<unsigned long long>());
    size_t tb = c->cg_tmp.bytes;
    CK(cub::DeviceRadixSort::SortKeys(c->cg_tmp.p, tb, c->cg_inc.as<unsigned long long>(),
                                      c->cg_inc2.as<unsigned long long>(), (int64_t)(4 * n), 0, 64, s));
    k_contact_csr<<<blocks_for(4 * n), 256, 0, s>>>(c->cg_inc2.as<unsigned long long>(), 4 * n, c->nsolve,
                                                   c->coff.as<long long>(), c->ccid.as<int>(), c->cslot.as<int>());
}

template <typename R> void enqueue_step_contacts_graph(vbd_ctx* c)
{
    const CgLayout L = cg_layout(c);
    c->ncontacts = L.capAll;  // padded arrays: K1 aux passes with the contact epilogue
    cg_detect_dcd<R>(c, L);
    cg_compile<R>(c, c->xt, L);
    enqueue_begin<R>(c);
    for (int n = 1; n <= c->cur.n_max; ++n) {
        if ((n - 1) % c->coll_ncol == 0) {
            cg_detect_ccd<R>(c, L);
            cg_compile<R>(c, c->pos, L);
        }
        for (int col = 0; col < c->ncolors; ++col) color_sweep<R>(c, col, n, c->cur.rho == 0.0);
        enqueue_iter_end<R>(c, n);
    }
    enqueue_end<R>(c);
}

template <typename R> void do_step_contacts(vbd_ctx* c, vbd_step_result* res);

// one contact step as one graph launch; false = the capacities overflowed (state rolled back)
template <typename R> bool step_contacts_graph(vbd_ctx* c, vbd_step_result* res)
{
    cudaStream_t s = c->stream;
    const size_t vb = (size_t)c->n * c->r4();
    char* snap = c->cg_snap.as<char>();
    CK(cudaMemcpyAsync(snap, c->xt.p, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(snap + vb, c->vt.p, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(snap + 2 * vb, c->vprev.p, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(snap + 3 * vb, c->stepctr.p, 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(c->cg_flag.p, 0, 16, s));
    GraphKey key{c->cur};
    if (!c->cg_exec || !(key == c->cg_key)) {
        if (c->cg_exec) {
            cudaGraphExecDestroy(c->cg_exec);
            c->cg_exec = nullptr;
        }
        Nvtx r("contact step capture");
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        enqueue_step_contacts_graph<R>(c);
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&c->cg_exec, g, 0));
        cudaGraphDestroy(g);
        c->cg_key = key;
    }
    {
        Nvtx r("vbd_step contact graph");
        CK(cudaGraphLaunch(c->cg_exec, s));
    }
    const int overflow = read_scalar<int>(c->cg_flag.p, s);
    if (!overflow) {
        read_result(c, res);
        return true;
    }
    CK(cudaMemcpyAsync(c->xt.p, snap, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->vt.p, snap + vb, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->vprev.p, snap + 2 * vb, vb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->stepctr.p, snap + 3 * vb, 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(c->flag.p, 0xff, 8, s));
    return false;
}

// one step with contacts: DCD at x_t, CCD every n_col iterations, aux-buffer colour passes
// (contacts couple vertices of one colour), K3 keeping colliding vertices unblended
template <typename R> void do_step_contacts(vbd_ctx* c, vbd_step_result* res)
{
    Nvtx r0("vbd_step (contacts)");
    {
        Nvtx r1("dcd");
        detect_dcd<R>(c);
        compile_contact_set<R>(c, c->xt);
    }
    enqueue_begin<R>(c);
    for (int n = 1; n <= c->cur.n_max; ++n) {
        Nvtx r1("iteration %d", n);
        if ((n - 1) % c->coll_ncol == 0) {
            Nvtx r2("ccd");
            detect_ccd<R>(c);
            compile_contact_set<R>(c, c->pos);
        }
        for (int col = 0; col < c->ncolors; ++col) {
            Nvtx r2("colour %d", col);
            color_sweep<R>(c, col, n, c->cur.rho == 0.0);
        }
        enqueue_iter_end<R>(c, n);
    }
    enqueue_end<R>(c);
    read_result(c, res);
}

template <typename R> void do_step(vbd_ctx* c, const vbd_step_params* p, int n_steps, vbd_step_result* res)
{
    validate_params(p);
    if (n_steps < 1 || n_steps > 65535) fail(VBD_ERR_ARG, "n_steps must be in [1, 65535]");
    c->cur = *p;
    c->omegas = omega_table(p->rho, p->n_max);
    ensure_materials<R>(c, p->h);
    cudaStream_t s = c->stream;
    CK(cudaMemsetAsync(c->flag.p, 0xff, 8, s));
    CK(cudaMemsetAsync(c->stepctr.p, 0, 4, s));
    if (c->coll_on) {
        const bool graph_on = c->cg_enabled;
        for (int k = 0; k < n_steps; ++k) {
            if (graph_on && c->cg_pending) {  // (not right after the host step: its contact set
                cg_setup<R>(c);               //  stays readable by the metrics until the next step)
                c->cg_pending = false;
            }
            if (graph_on && c->cg_ready && step_contacts_graph<R>(c, res)) {
                ++c->cg_steps;
                continue;
            }
            if (graph_on && c->cg_ready) ++c->cg_fallbacks;
            do_step_contacts<R>(c, res);  // host path; records the counts the capacities need
            c->cg_pending = graph_on;
        }
        return;
    }
    if (use_persistent(c) && !p->line_search) {
        c->omega_dev.alloc((p->n_max + 1) * sizeof(double));
        CK(cudaMemcpyAsync(c->omega_dev.p, c->omegas.data(), (p->n_max + 1) * sizeof(double),
                           cudaMemcpyHostToDevice, s));
        for (int k = 0; k < n_steps; ++k) launch_step_persistent<R>(c);
        read_result(c, res);
        return;
    }
    ensure_resident<R>(c);
    if (c->res_mode > 0 && !p->line_search) {  // K1R reads the omega table from the device
        if (c->omega_dev.bytes < (p->n_max + 1) * sizeof(double)) c->omega_dev.alloc((p->n_max + 1) * sizeof(double));
        CK(cudaMemcpyAsync(c->omega_dev.p, c->omegas.data(), (p->n_max + 1) * sizeof(double),
                           cudaMemcpyHostToDevice, s));
    }
    GraphKey key{*p};
    if (!c->gexec || !(key == c->gkey)) {
        if (c->gexec) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        Nvtx r("vbd_step capture");
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        enqueue_step<R>(c);
        cudaError_t e = cudaStreamEndCapture(s, &g);
        CK(e);
        CK(cudaGraphInstantiate(&c->gexec, g, 0));
        cudaGraphDestroy(g);
        c->gkey = key;
    }
    for (int k = 0; k < n_steps; ++k) {
        Nvtx r("vbd_step graph (n_max %d, %d colours)", p->n_max, c->ncolors);
        CK(cudaGraphLaunch(c->gexec, s));
    }
    read_result(c, res);
}

// ---------------------------------------------------------------------------------------
// state transfer

// rest positions to subtract / add for a position-like vector (fp32 displacement state)
inline const double4* rest_for(const vbd_ctx* c, bool position)
{
    return c->disp && position ? const_cast<DBuf&>(c->rest).as<double4>() : nullptr;
}

bool host_pinned(const void* p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// memcpy split across host threads (the host side of the staged pageable path)
void par_memcpy(void* dst, const void* src, size_t n)
{
    static const int T = [] {
        const char* e = getenv("VBD_STAGE_THREADS");
        const int hw = (int)std::thread::hardware_concurrency();
        return std::max(1, e && *e ? atoi(e) : std::min(16, hw));
    }();
    if (n < ((size_t)4 << 20) || T == 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const size_t o = (size_t)t * part;
        if (o >= n) break;
        th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(part, n - o)); });
    }
    for (auto& x : th) x.join();
}

// host -> device (stream-ordered; a pageable source is staged chunk by chunk)
void h2d(vbd_ctx* c, void* dev, const void* host, size_t bytes)
{
    cudaStream_t s = c->stream;
    if (bytes < ((size_t)8 << 20) || host_pinned(host) || !c->hstage.ready()) {
        CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    HostStager& st = c->hstage;
    for (size_t off = 0, k = 0; off < bytes; off += HostStager::CHUNK, ++k) {
        const int b = (int)(k & 1);
        const size_t sz = std::min(HostStager::CHUNK, bytes - off);
        CK(cudaEventSynchronize(st.ev[b]));  // the DMA out of this chunk two rounds ago is done
        par_memcpy(st.pin[b], (const char*)host + off, sz);
        CK(cudaMemcpyAsync((char*)dev + off, st.pin[b], sz, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(st.ev[b], s));
    }
}

// device -> host, synchronous (a pageable destination is staged chunk by chunk)
void d2h(vbd_ctx* c, void* host, const void* dev, size_t bytes)
{
    cudaStream_t s = c->stream;
    if (bytes < ((size_t)8 << 20) || host_pinned(host) || !c->hstage.ready()) {
        CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    HostStager& st = c->hstage;
    const size_t nch = (bytes + HostStager::CHUNK - 1) / HostStager::CHUNK;
    auto issue = [&](size_t k) {
        const size_t off = k * HostStager::CHUNK, sz = std::min(HostStager::CHUNK, bytes - off);
        CK(cudaMemcpyAsync(st.pin[k & 1], (const char*)dev + off, sz, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(st.ev[k & 1], s));
    };
    issue(0);
    for (size_t k = 0; k < nch; ++k) {
        if (k + 1 < nch) issue(k + 1);  // the other chunk's host copy (k - 1) is already done
        CK(cudaEventSynchronize(st.ev[k & 1]));
        const size_t off = k * HostStager::CHUNK, sz = std::min(HostStager::CHUNK, bytes - off);
        par_memcpy((char*)host + off, st.pin[k & 1], sz);
    }
}

template <typename R> void load_vec(vbd_ctx* c, const double* host, DBuf& dst, bool position)
{
    cudaStream_t s = c->stream;
    h2d(c, c->stage.p, host, c->n * 3 * sizeof(double));
    k_load_vec<R><<<blocks_for(c->n), 256, 0, s>>>(c->stage.as<double>(),
                                                   dst.as<typename Vec4<R>::T>(),
                                                   c->perm.as<int>(), (int)c->n, rest_for(c, position));
    CK(cudaGetLastError());
}

template <typename R> void store_vec(vbd_ctx* c, const DBuf& src, double* host, bool position)
{
    cudaStream_t s = c->stream;
    k_store_vec<R><<<blocks_for(c->n), 256, 0, s>>>(src.as<typename Vec4<R>::T>(),
                                                    c->stage.as<double>(), c->inv.as<int>(),
                                                    (int)c->n, rest_for(c, position));
    CK(cudaGetLastError());
    d2h(c, host, c->stage.p, c->n * 3 * sizeof(double));
}

template <typename R>
void do_color_pass(vbd_ctx* c, double* x, const double* x_t, const double* y, double h,
                   const int64_t* group, int64_t ng, int mode, int line_search, double eps_det)
{
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    if (ng <= 0) return;  // _native.pyx:520-521
    Nvtx r("vbd_color_pass (%lld vertices)", (long long)ng);
    ensure_materials<R>(c, h);
    load_vec<R>(c, x, c->pos, true);
    load_vec<R>(c, x_t, c->xt, true);
    load_vec<R>(c, y, c->y, true);
    k_fill_mih2<R><<<blocks_for(c->n), 256, 0, s>>>(c->y.as<R4>(), c->mass.as<R>(), (int)c->n, h * h);
    // group (original ids) -> colour-major ids
    std::vector<int> gi(ng);
    std::vector<int>& hinv = c->hinv;
    {
        if ((long long)hinv.size() != c->n) {
            hinv.resize(c->n);
            CK(cudaMemcpyAsync(hinv.data(), c->inv.p, c->n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        for (int64_t k = 0; k < ng; ++k) {
            if (group[k] < 0 || group[k] >= c->n) fail(VBD_ERR_ARG, "group vertex out of range");
            gi[k] = hinv[group[k]];
        }
    }
    DBuf gdev, odev;
    upload(gdev, gi.data(), ng, s);
    odev.alloc(ng * c->r4());
    K1Args<R> a = k1_args<R>(c, eps_det, mode, false, 0);
    a.group = gdev.as<int>();
    a.count = (int)ng;
    a.line_search = line_search ? 1 : 0;
    a.out = odev.as<R4>();
    launch_k1<R>(c, a, s);
    CK(cudaGetLastError());
    // the group's new rows in double (+ the rest positions in the displacement state)
    DBuf o64;
    o64.alloc((size_t)ng * 24);
    k_group_abs<R><<<blocks_for(ng), 256, 0, s>>>(odev.as<R4>(), gdev.as<int>(), rest_for(c, true), (int)ng,
                                                  o64.as<double>());
    CK(cudaGetLastError());
    std::vector<double> ho(3 * ng);
    CK(cudaMemcpyAsync(ho.data(), o64.p, ng * 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // merge (_native.pyx:585-589): only the group's rows change
    for (int64_t k = 0; k < ng; ++k) {
        int64_t v = group[k];
        x[3 * v] = ho[3 * k];
        x[3 * v + 1] = ho[3 * k + 1];
        x[3 * v + 2] = ho[3 * k + 2];
    }
}

// Springs, world boxes and subspace constraints of a host-built system, in colour-major order
// over the solved vertices (the global K1 adds them in its per-vertex epilogue).
template <typename R> void attach_extras(vbd_ctx* c, const vbd_system_desc* d, const std::vector<int>& color)
{
    typedef typename Vec4<R>::T R4;
    cudaStream_t s = c->stream;
    const long long N = d->num_vertices, S = d->springs ? d->num_springs : 0;
    std::vector<int> perm(N), inv(N);
    CK(cudaMemcpy(perm.data(), c->perm.p, N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(inv.data(), c->inv.p, N * 4, cudaMemcpyDeviceToHost));
    const long long ns = c->nsolve;
    // vertex -> spring CSR, ascending spring id per vertex (incidence_from_elements order)
    std::vector<long long> deg(N + 1, 0);
    for (long long k = 0; k < S; ++k)
        for (int e = 0; e < 2; ++e) {
            const int64_t v = d->springs[2 * k + e];
            if (v < 0 || v >= N) fail(VBD_ERR_ARG, "spring index out of range");
            deg[v + 1]++;
        }
    for (long long v = 0; v < N; ++v) deg[v + 1] += deg[v];
    std::vector<long long> fill(deg.begin(), deg.end() - 1);
    std::vector<long long> vsp(2 * S);
    std::vector<int> vslot(2 * S);
    for (long long k = 0; k < S; ++k)
        for (int e = 0; e < 2; ++e) {
            const int64_t v = d->springs[2 * k + e];
            vsp[fill[v]] = k;
            vslot[fill[v]++] = e;
        }
    std::vector<long long> soff(ns + 1, 0);
    for (long long i = 0; i < ns; ++i) soff[i + 1] = soff[i] + (deg[perm[i] + 1] - deg[perm[i]]);
    std::vector<int> oth(std::max<long long>(soff[ns], 1));
    std::vector<R4> par(std::max<long long>(soff[ns], 1));
    for (long long i = 0; i < ns; ++i) {
        const int o = perm[i];
        long long w = soff[i];
        for (long long k = deg[o]; k < deg[o + 1]; ++k, ++w) {
            const long long sp = vsp[k];
            oth[w] = inv[d->springs[2 * sp + (1 - vslot[k])]];
            R4 q;
            q.x = (R)d->sp_l0[sp];
            q.y = (R)d->sp_k[sp];
            q.z = (R)d->sp_kd[sp];
            q.w = R(0);
            par[w] = q;
        }
    }
    upload(c->soff, soff.data(), soff.size(), s);
    upload(c->sp_oth, oth.data(), oth.size(), s);
    upload(c->sp_par, par.data(), par.size(), s);
    // springs join vertices of different colours (the in-place sweep relies on it)
    for (long long k = 0; k < S; ++k) {
        const int64_t a = d->springs[2 * k], b = d->springs[2 * k + 1];
        if (color[a] >= 0 && color[a] == color[b]) c->inplace = false;
    }
    // world boxes
    bool any_box = false;
    if (d->box_k)
        for (long long v = 0; v < N; ++v) any_box |= d->box_k[v] > 0.0;
    if (any_box) {  // over all vertices (the energy counts fixed vertices' boxes too)
        std::vector<R4> bx(2 * std::max<long long>(N, 1));
        for (long long i = 0; i < N; ++i) {
            const int o = perm[i];
            R4 lo, hi;
            lo.x = (R)d->box_lo[3 * o]; lo.y = (R)d->box_lo[3 * o + 1]; lo.z = (R)d->box_lo[3 * o + 2];
            lo.w = (R)(d->box_k[o] > 0.0 ? d->box_k[o] : 0.0);
            hi.x = (R)d->box_hi[3 * o]; hi.y = (R)d->box_hi[3 * o + 1]; hi.z = (R)d->box_hi[3 * o + 2];
            hi.w = R(0);
            bx[2 * i] = lo;
            bx[2 * i + 1] = hi;
        }
        upload(c->box, bx.data(), bx.size(), s);
    } else {
        c->box.release();
    }
    // subspace constraints
    std::vector<int> sidx(std::max<long long>(ns, 1), -1);
    std::vector<R4> sub;
    if (d->kind)
        for (long long i = 0; i < ns; ++i) {
            const int o = perm[i];
            if (d->kind[o] != VBD_KIND_SUBSPACE) continue;
            if (!d->sub_dim || !d->sub_basis || !d->sub_anchor) fail(VBD_ERR_ARG, "subspace arrays missing");
            const int dim = (int)d->sub_dim[o];
            if (dim != 1 && dim != 2) fail(VBD_ERR_ARG, "subspace dimension must be 1 or 2");
            const double* B = d->sub_basis + 6 * o;
            const double* an = d->sub_anchor + 3 * o;
            sidx[i] = (int)(sub.size() / 3);
            R4 a, b, e;
            a.x = (R)B[0]; a.y = (R)B[1]; a.z = (R)B[2]; a.w = (R)B[3];
            b.x = (R)B[4]; b.y = (R)B[5]; b.z = (R)an[0]; b.w = (R)an[1];
            e.x = (R)an[2]; e.y = (R)dim; e.z = R(0); e.w = R(0);
            sub.push_back(a);
            sub.push_back(b);
            sub.push_back(e);
        }
    if (sub.empty()) sub.resize(3);
    upload(c->sub_idx, sidx.data(), sidx.size(), s);
    upload(c->sub, sub.data(), sub.size(), s);
    CK(cudaStreamSynchronize(s));
}

int material_id(vbd_ctx* c, std::map<MaterialKey, int>& ids, const MaterialKey& k)
{
    auto it = ids.find(k);
    if (it != ids.end()) return it->second;
    int id = (int)c->mats.size();
    if (id >= VBD_MAX_MATERIALS) fail(VBD_ERR_UNSUPPORTED, "more than 512 distinct materials");
    ids[k] = id;
    c->mats.push_back(k);
    return id;
}

void init_ctx(vbd_ctx* c, int device, int precision)
{
    if (const char* e = getenv("VBD_RESIDENT")) c->res_want = e;
    if (const char* e = getenv("VBD_CONTACT_GRAPH")) c->cg_enabled = *e != '0';
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        fail(VBD_ERR_NODEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= count) fail(VBD_ERR_ARG, "bad device index");
    if (precision != VBD_PREC_F32 && precision != VBD_PREC_F64) fail(VBD_ERR_ARG, "bad precision");
    c->device = device;
    c->precision = precision;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        fail(VBD_ERR_NODEVICE, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->owned.s = c->own_stream;
    c->stream = c->own_stream;
    {  // keep up to 1 GB of freed pool memory cached (stream-ordered scratch allocations)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
            unsigned long long thr = 1ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
}

void finish_pack(vbd_ctx* c, Scene& sc)
{
    if (c->precision == VBD_PREC_F64)
        pack<double>(c, sc);
    else
        pack<float>(c, sc);
}

template <typename R> void set_rest_state(vbd_ctx* c, const Scene& sc)
{
    // x = x_t = y = rest positions, v = v_prev = 0 (make_state, solver.py:111-117)
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(c->stage.p, sc.pos.p, c->n * 3 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    for (DBuf* d : {&c->pos, &c->xt, &c->y})
        k_load_vec<R><<<blocks_for(c->n), 256, 0, s>>>(c->stage.as<double>(),
                                                       d->as<typename Vec4<R>::T>(),
                                                       c->perm.as<int>(), (int)c->n, rest_for(c, true));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
}

__global__ void k_beam_velocity(const BeamDev* __restrict__ beams, int nb, const double* __restrict__ la,
                                const double* __restrict__ pos, long long n, double* __restrict__ v)
{
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int b = find_beam(beams, nb, i, false);
    const BeamDev& B = beams[b];
    double cx = B.origin[0] + 0.5 * B.spacing * (B.nx - 1);
    double cy = B.origin[1] + 0.5 * B.spacing * (B.ny - 1);
    double cz = B.origin[2] + 0.5 * B.spacing * (B.nz - 1);
    double rx = pos[3 * i] - cx, ry = pos[3 * i + 1] - cy, rz = pos[3 * i + 2] - cz;
    const double* q = la + 6 * b;
    v[3 * i] = q[0] + (q[4] * rz - q[5] * ry);
    v[3 * i + 1] = q[1] + (q[5] * rx - q[3] * rz);
    v[3 * i + 2] = q[2] + (q[3] * ry - q[4] * rx);
}

// FMA-pipe peak microbenchmark (vbd_fma_peak): 8 independent FMA chains per thread (enough
// to cover the 4-cycle pipe latency at full occupancy); the sum is stored only under an
// impossible condition so the chains stay live.
template <int MODE>  // 0 FFMA, 1 FFMA2 (fp32x2), 2 DFMA
__global__ void __launch_bounds__(256) k_fma_peak(float* sink, int iters, float a, float b)
{
    constexpr int CH = 8;
    if constexpr (MODE == 1) {
        float2 acc[CH];
        for (int j = 0; j < CH; ++j) acc[j] = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f);
        const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll 16
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = __ffma2_rn(acc[j], A, B);
        float t = 0.f;
        for (int j = 0; j < CH; ++j) t += acc[j].x + acc[j].y;
        if (t == 1234.5f) sink[threadIdx.x] = t;
    } else if constexpr (MODE == 0) {
        float acc[CH];
        for (int j = 0; j < CH; ++j) acc[j] = threadIdx.x * 1e-3f + j;
#pragma unroll 16
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = __fmaf_rn(acc[j], a, b);
        float t = 0.f;
        for (int j = 0; j < CH; ++j) t += acc[j];
        if (t == 1234.5f) sink[threadIdx.x] = t;
    } else {
        double acc[CH];
        for (int j = 0; j < CH; ++j) acc[j] = threadIdx.x * 1e-3 + j;
#pragma unroll 16
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = __fma_rn(acc[j], (double)a, (double)b);
        double t = 0.0;
        for (int j = 0; j < CH; ++j) t += acc[j];
        if (t == 1234.5) sink[threadIdx.x] = (float)t;
    }
}

}  // namespace

// =========================================================================================
// C ABI

extern "C" {

const char* vbd_last_error(void) { return g_err.c_str(); }
const char* vbd_version(void) { return "vbd_b200 0.1 (sm_100a)"; }

int vbd_device_count(int* count)
{
    return guarded([&] {
        if (!count) fail(VBD_ERR_ARG, "count is NULL");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
        *count = n;
    });
}

int vbd_ctx_create(const vbd_system_desc* d, int device, int precision, vbd_ctx** out)
{
    vbd_ctx* c = nullptr;
    int rc = guarded([&] {
        if (!d || !out) fail(VBD_ERR_ARG, "NULL argument");
        if (d->num_vertices < 0 || d->num_tets < 0) fail(VBD_ERR_ARG, "negative sizes");
        if (!d->masses || !d->color_off || !d->color_verts || !d->t_off)
            fail(VBD_ERR_ARG, "missing System arrays");
        if (d->num_tets && (!d->tets || !d->tet_w || !d->tet_vol || !d->tet_mu || !d->tet_lam ||
                            !d->tet_kd || !d->t_id || !d->t_slot))
            fail(VBD_ERR_ARG, "missing tet arrays");
        c = new vbd_ctx();
        init_ctx(c, device, precision);
        cudaStream_t s = c->stream;
        const long long N = d->num_vertices, T = d->num_tets;
        if (4 * T >= (1LL << 32)) fail(VBD_ERR_UNSUPPORTED, "too many tets for one context");
        Scene sc;
        sc.n = N;
        sc.T = T;
        // tets (int64 -> int32) and materials
        std::vector<int> tets32(4 * T), tmat(T);
        std::map<MaterialKey, int> ids;
        for (long long t = 0; t < T; ++t) {
            for (int k = 0; k < 4; ++k) {
                int64_t v = d->tets[4 * t + k];
                if (v < 0 || v >= N) fail(VBD_ERR_ARG, "tet index out of range");
                tets32[4 * t + k] = (int)v;
            }
            if (!(d->tet_lam[t] != 0.0)) fail(VBD_ERR_ARG, "tet_lam must be non-zero");
            tmat[t] = material_id(c, ids, MaterialKey{d->tet_mu[t], d->tet_lam[t], d->tet_kd[t], 0.0});
        }
        upload(sc.tets, tets32.data(), tets32.size(), s);
        upload(sc.tmat, tmat.data(), tmat.size(), s);
        upload(sc.tet_w, d->tet_w, 12 * T, s);
        upload(sc.vol, d->tet_vol, T, s);
        upload(sc.mass, d->masses, N, s);
        std::vector<unsigned char> kind(N, 0);
        bool extras = d->springs && d->num_springs > 0;
        if (d->kind)
            for (long long v = 0; v < N; ++v) {
                if (d->kind[v] == VBD_KIND_SUBSPACE) extras = true;  // solved, in its subspace
                kind[v] = d->kind[v] == VBD_KIND_FIXED ? 1 : 0;
            }
        if (d->box_k)
            for (long long v = 0; v < N && !extras; ++v) extras = d->box_k[v] > 0.0;
        c->has_extras = extras;
        upload(sc.kind, kind.data(), N, s);
        // incidence exactly as given (ascending tet id per vertex, mesh.py:243-250)
        if (d->t_off[0] != 0 || d->t_off[N] != 4 * T) fail(VBD_ERR_ARG, "t_off inconsistent with tets");
        std::vector<unsigned> inc(4 * T);
        for (long long k = 0; k < 4 * T; ++k) {
            if (d->t_slot[k] < 0 || d->t_slot[k] > 3 || d->t_id[k] < 0 || d->t_id[k] >= T)
                fail(VBD_ERR_ARG, "bad t_id/t_slot");
            inc[k] = (unsigned)(4 * d->t_id[k] + d->t_slot[k]);
        }
        upload(sc.inc_off, d->t_off, N + 1, s);
        upload(sc.inc, inc.data(), inc.size(), s);
        // colours from the groups
        std::vector<int> color(N, -1);
        for (long long g = 0; g < d->num_colors; ++g)
            for (long long k = d->color_off[g]; k < d->color_off[g + 1]; ++k) {
                int64_t v = d->color_verts[k];
                if (v < 0 || v >= N) fail(VBD_ERR_ARG, "colour vertex out of range");
                color[v] = (int)g;
            }
        for (long long v = 0; v < N; ++v)
            if (color[v] < 0 && kind[v] != 1) fail(VBD_ERR_ARG, "vertex without colour");
        if (d->num_colors > 4095) fail(VBD_ERR_UNSUPPORTED, "too many colours");
        upload(sc.color, color.data(), N, s);
        if (d->rest_positions && N) {
            double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (long long v = 0; v < N; ++v)
                for (int k = 0; k < 3; ++k) {
                    lo[k] = std::min(lo[k], d->rest_positions[3 * v + k]);
                    hi[k] = std::max(hi[k], d->rest_positions[3 * v + k]);
                }
            sc.set_bbox(lo, hi);
            upload(sc.pos, d->rest_positions, 3 * N, s);
        }
        CK(cudaStreamSynchronize(s));
        finish_pack(c, sc);
        if (c->has_extras) {
            if (c->precision == VBD_PREC_F64) attach_extras<double>(c, d, color);
            else attach_extras<float>(c, d, color);
        }
        *out = c;
    });
    if (rc != VBD_OK) delete c;
    return rc;
}

int vbd_ctx_create_beams(const vbd_beam_desc* beams, int64_t nb, int64_t slab_lo, int64_t slab_hi,
                         int device, int precision, vbd_ctx** out)
{
    vbd_ctx* c = nullptr;
    int rc = guarded([&] {
        if (!beams || nb < 1 || !out) fail(VBD_ERR_ARG, "bad beam list");
        bool slab = slab_hi > slab_lo;
        if (slab && nb != 1) fail(VBD_ERR_ARG, "slab decomposition needs exactly one beam");
        c = new vbd_ctx();
        init_ctx(c, device, precision);
        cudaStream_t s = c->stream;
        std::map<MaterialKey, int> ids;
        std::vector<double> dens;
        // full beams (for colouring and non-slab scenes)
        auto make_table = [&](bool full) {
            std::vector<BeamDev> tb(nb);
            long long vb = 0, tbase = 0;
            for (int64_t i = 0; i < nb; ++i) {
                const vbd_beam_desc& d = beams[i];
                if (d.nx < 2 || d.ny < 2 || d.nz < 2) fail(VBD_ERR_ARG, "beam needs >= 2 vertices per axis");
                if (!(d.spacing > 0) || !(d.density > 0) || !(d.mu > 0) || !(d.lam > 0) || d.kd < 0)
                    fail(VBD_ERR_ARG, "bad beam parameters");
                BeamDev& B = tb[i];
                B.nx = d.nx; B.ny = d.ny; B.nz = d.nz;
                B.spacing = d.spacing; B.density = d.density;
                for (int k = 0; k < 3; ++k) B.origin[k] = d.origin[k];
                B.fix_min_x = d.fix_min_x;
                B.fix_max_x = d.fix_max_x;
                if (!(d.jitter >= 0.0 && d.jitter < 0.25)) fail(VBD_ERR_ARG, "beam jitter must be in [0, 0.25)");
                B.jitter = d.jitter;
                B.mat = material_id(c, ids, MaterialKey{d.mu, d.lam, d.kd, d.density});
                if ((int)dens.size() <= B.mat) dens.resize(B.mat + 1, d.density);
                if (full || !slab) {
                    B.ax0 = 0; B.ax1 = d.nx - 1; B.gcell0 = 0;
                } else {
                    if (slab_lo < 0 || slab_hi > d.nx) fail(VBD_ERR_ARG, "slab outside the beam");
                    B.ax0 = std::max<long long>(slab_lo - 1, 0);
                    B.ax1 = std::min<long long>(slab_hi, d.nx - 1);
                    B.gcell0 = B.ax0;
                }
                B.vbase = vb;
                B.tbase = tbase;
                vb += (B.ax1 - B.ax0 + 1) * B.ny * B.nz;
                tbase += (B.ax1 - B.ax0) * (B.ny - 1) * (B.nz - 1) * 5;
            }
            return std::make_tuple(tb, vb, tbase);
        };
        auto generate = [&](Scene& sc, const std::vector<BeamDev>& tb, long long n, long long T, DBuf& bdev) {
            upload(bdev, tb.data(), tb.size(), s);
            sc.n = n;
            sc.T = T;
            if (n >= (1LL << 31) || 4 * T >= (1LL << 32)) fail(VBD_ERR_UNSUPPORTED, "scene too large for one context");
            sc.pos.alloc(n * 3 * 8);
            sc.kind.alloc(n);
            k_gen_vertices<<<blocks_for(n), 256, 0, s>>>(bdev.as<BeamDev>(), (int)nb, n,
                                                          sc.pos.as<double>(), sc.kind.as<unsigned char>());
            sc.tets.alloc(T * 16);
            sc.tet_w.alloc(T * 96);
            sc.vol.alloc(T * 8);
            sc.tmat.alloc(T * 4);
            k_gen_tets<<<blocks_for(T), 256, 0, s>>>(bdev.as<BeamDev>(), (int)nb, T, sc.pos.as<double>(),
                                                      sc.tets.as<int>(), sc.tet_w.as<double>(),
                                                      sc.vol.as<double>(), sc.tmat.as<int>());
            CK(cudaGetLastError());
            build_incidence(sc, s);
        };
        std::vector<int> color_keep;
        long long keep_off = 0;
        if (slab) {
            // colour the whole beam once (bit-exact global colouring), keep the slab's part
            auto [tb, n, T] = make_table(true);
            Scene full;
            DBuf bdev;
            generate(full, tb, n, T, bdev);
            color_scene(full, s);
            auto [tl, nl, Tl] = make_table(false);
            keep_off = tl[0].ax0 * tl[0].ny * tl[0].nz;
            color_keep.resize(nl);
            CK(cudaMemcpyAsync(color_keep.data(), full.color.as<int>() + keep_off, nl * 4,
                               cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        auto [tb, n, T] = make_table(false);
        c->beams = tb;
        Scene sc;
        generate(sc, tb, n, T, c->beams_dev);
        {
            // bbox of the (whole) beams: the spatial order must not depend on the slab
            double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int64_t i = 0; i < nb; ++i) {
                const vbd_beam_desc& d = beams[i];
                const long long ext[3] = {d.nx - 1, d.ny - 1, d.nz - 1};
                for (int k = 0; k < 3; ++k) {
                    lo[k] = std::min(lo[k], d.origin[k]);
                    hi[k] = std::max(hi[k], d.origin[k] + d.spacing * (double)ext[k]);
                }
            }
            sc.set_bbox(lo, hi);
        }
        DBuf dm;
        upload(dm, dens.data(), dens.size(), s);
        sc.mass.alloc(n * 8);
        k_mass_gather<<<blocks_for(n), 256, 0, s>>>(sc.inc_off.as<long long>(), sc.inc.as<unsigned>(),
                                                     sc.vol.as<double>(), sc.tmat.as<int>(),
                                                     dm.as<double>(), n, sc.mass.as<double>());
        CK(cudaGetLastError());
        if (slab) {
            sc.color.alloc(n * 4);
            CK(cudaMemcpyAsync(sc.color.p, color_keep.data(), n * 4, cudaMemcpyHostToDevice, s));
            // ghost planes: ax0 (if < slab_lo) and ax1 (if >= slab_hi)
            const BeamDev& B = tb[0];
            long long plane = B.ny * B.nz;
            std::vector<unsigned char> kind(n);
            CK(cudaMemcpyAsync(kind.data(), sc.kind.p, n, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<unsigned char> halo(n, 0);
            for (long long v = 0; v < n; ++v) {
                long long ax = B.ax0 + v / plane;
                if ((ax < slab_lo || ax >= slab_hi) && kind[v] != 1) kind[v] = 3;
                if (ax == slab_lo - 1) halo[v] = 3;
                else if (ax == slab_hi) halo[v] = 4;
                else if (ax == slab_lo && slab_lo > 0) halo[v] = 1;
                else if (ax == slab_hi - 1 && slab_hi < B.nx) halo[v] = 2;
            }
            if (slab_hi - slab_lo < 2) fail(VBD_ERR_ARG, "slabs must own at least 2 vertex planes");
            CK(cudaMemcpyAsync(sc.kind.p, kind.data(), n, cudaMemcpyHostToDevice, s));
            upload(sc.halo, halo.data(), n, s);
            CK(cudaStreamSynchronize(s));
        } else {
            color_scene(sc, s);
        }
        finish_pack(c, sc);
        if (c->precision == VBD_PREC_F64) set_rest_state<double>(c, sc);
        else set_rest_state<float>(c, sc);
        if (slab) {
            // halo lists: side 0 = towards slab_lo (rank - 1), side 1 = towards slab_hi (rank + 1)
            const BeamDev& B = tb[0];
            long long plane = B.ny * B.nz;
            std::vector<int> hinv(n), col(n);
            CK(cudaMemcpyAsync(hinv.data(), c->inv.p, n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(col.data(), sc.color.p, n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            long long planes_send[2] = {slab_lo, slab_hi - 1}, planes_recv[2] = {slab_lo - 1, slab_hi};
            for (int side = 0; side < 2; ++side) {
                c->halo_send[side].assign(c->ncolors, {});
                c->halo_recv[side].assign(c->ncolors, {});
                c->halo_send_cnt[side].assign(c->ncolors, {});
                c->halo_recv_cnt[side].assign(c->ncolors, {});
                bool exists = side == 0 ? slab_lo > 0 : slab_hi < B.nx;
                for (int col_i = 0; col_i < c->ncolors; ++col_i) {
                    std::vector<int> sl, rl;
                    if (exists) {
                        long long ps = planes_send[side] - B.ax0, pr = planes_recv[side] - B.ax0;
                        for (long long k = 0; k < plane; ++k) {
                            long long vs = ps * plane + k, vr = pr * plane + k;
                            if (col[vs] == col_i) sl.push_back(hinv[vs]);
                            if (col[vr] == col_i) rl.push_back(hinv[vr]);
                        }
                    }
                    DBuf* bs = new DBuf();
                    DBuf* br = new DBuf();
                    upload(*bs, sl.data(), sl.size(), s);
                    upload(*br, rl.data(), rl.size(), s);
                    c->halo_send[side][col_i].push_back(bs);
                    c->halo_recv[side][col_i].push_back(br);
                    c->halo_send_cnt[side][col_i].push_back((long long)sl.size());
                    c->halo_recv_cnt[side][col_i].push_back((long long)rl.size());
                }
            }
            CK(cudaStreamSynchronize(s));
        }
        *out = c;
    });
    if (rc != VBD_OK) delete c;
    return rc;
}

int vbd_ctx_destroy(vbd_ctx* c)
{
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        delete c;
    });
}

int vbd_ctx_get_info(vbd_ctx* c, vbd_ctx_info* info)
{
    return guarded([&] {
        if (!c || !info) fail(VBD_ERR_ARG, "NULL argument");
        std::memset(info, 0, sizeof *info);
        info->num_vertices = c->n;
        info->num_solved = c->nsolve;
        info->num_ghost = c->nfree_all - c->nsolve;
        info->num_fixed = c->n - c->nfree_all;
        info->num_tets = c->T;
        info->num_entries = c->E;
        info->num_colors = c->ncolors;
        for (int k = 0; k < c->ncolors && k < 64; ++k) info->color_count[k] = c->ccnt[k];
        long long b = 0;
        for (DBuf* d : {&c->soff, &c->sp_oth, &c->sp_par, &c->box, &c->sub_idx, &c->sub,
                        &c->perm, &c->inv, &c->eoff, &c->ent, &c->mat, &c->pos, &c->xt, &c->vt, &c->vprev,
                        &c->y, &c->ha, &c->hb, &c->mass, &c->out, &c->stage, &c->color_orig, &c->kinds,
                        &c->kind_keys, &c->vmat, &c->tv0, &c->tnv, &c->loff, &c->tnbr, &c->tent,
                        &c->tdesc})
            b += (long long)d->bytes;
        info->device_bytes = b;
        info->precision = c->precision;
        info->inplace = c->inplace ? 1 : 0;
        info->lanes_per_vertex = c->k1.W;
        info->num_materials = (int)c->mats.size();
        info->layout = c->compact ? 1 : 0;
        info->num_entry_kinds = c->nkinds;
        info->tiles = c->tiles ? (int)(c->tile_beg.back()) : 0;
        info->tile_nbr_cap = c->nbr_cap;
        info->tile_slots = c->tiles ? c->tent.bytes / 8 : 0;
        info->tile_nbr_refs = c->tiles ? c->tnbr.bytes / 4 : 0;
        info->tile_lanes = c->tiles ? c->tile_w : 0;
        info->tile_stages = c->tiles ? c->tile_stages : 0;
        info->tile_ent_cap = c->tiles ? c->ent_cap : 0;
        if (c->tiles) {
            const int kn = (c->tile_kg || c->tile_xr) ? -1 : (int)c->nkinds + c->ncrec;
            const TileSmem<float> L32{c->ent_cap, c->nbr_cap, kn, c->tile_svpt, c->tile_xtg ? 1 : 3};
            const TileSmem<double> L64{c->ent_cap, c->nbr_cap, kn, c->tile_svpt, c->tile_xtg ? 1 : 3};
            info->tile_smem_bytes = (int)(c->precision == VBD_PREC_F64 ? L64.total(c->tile_stages)
                                                                       : L32.total(c->tile_stages));
        }
        info->entry_bytes = c->compact ? 16 : EntryPlanesBytes(c->precision);
        info->resident = c->res_mode > 0 ? c->res_mode : 0;
        info->resident_ctas = c->res_mode > 0 ? c->res_ncta : 0;
        info->contact_graph_steps = c->cg_steps;
        info->contact_graph_fallbacks = c->cg_fallbacks;
        info->class_vertices = c->tiles ? c->class_vertices : 0;
        info->class_tiles = c->tiles ? c->class_tiles : 0;
        info->class_records = c->tiles ? c->ncrec : 0;
    });
}

int vbd_set_stream(vbd_ctx* c, void* stream)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        c->stream = stream ? (cudaStream_t)stream : c->own_stream;
        if (c->gexec) {  // graphs are stream-agnostic, but keep things simple
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
    });
}

int vbd_get_stream(vbd_ctx* c, void** stream)
{
    return guarded([&] {
        if (!c || !stream) fail(VBD_ERR_ARG, "NULL argument");
        *stream = (void*)c->stream;
    });
}

int vbd_get_colors(vbd_ctx* c, int64_t* color_of)
{
    return guarded([&] {
        if (!c || !color_of) fail(VBD_ERR_ARG, "NULL argument");
        CK(cudaSetDevice(c->device));
        std::vector<int> h(c->n);
        CK(cudaMemcpyAsync(h.data(), c->color_orig.p, c->n * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (long long v = 0; v < c->n; ++v) color_of[v] = h[v];
    });
}

int vbd_set_state(vbd_ctx* c, const double* x, const double* x_t, const double* v_t,
                  const double* v_prev, const double* y)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        CK(cudaSetDevice(c->device));
        if (c->precision == VBD_PREC_F64) {
            if (x) load_vec<double>(c, x, c->pos, true);
            if (x_t) load_vec<double>(c, x_t, c->xt, true);
            if (v_t) load_vec<double>(c, v_t, c->vt, false);
            if (v_prev) load_vec<double>(c, v_prev, c->vprev, false);
            if (y) load_vec<double>(c, y, c->y, true);
        } else {
            if (x) load_vec<float>(c, x, c->pos, true);
            if (x_t) load_vec<float>(c, x_t, c->xt, true);
            if (v_t) load_vec<float>(c, v_t, c->vt, false);
            if (v_prev) load_vec<float>(c, v_prev, c->vprev, false);
            if (y) load_vec<float>(c, y, c->y, true);
        }
        CK(cudaStreamSynchronize(c->stream));
    });
}

int vbd_get_state(vbd_ctx* c, double* x, double* x_t, double* v_t, double* v_prev, double* y)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        CK(cudaSetDevice(c->device));
        if (c->precision == VBD_PREC_F64) {
            if (x) store_vec<double>(c, c->pos, x, true);
            if (x_t) store_vec<double>(c, c->xt, x_t, true);
            if (v_t) store_vec<double>(c, c->vt, v_t, false);
            if (v_prev) store_vec<double>(c, c->vprev, v_prev, false);
            if (y) store_vec<double>(c, c->y, y, true);
        } else {
            if (x) store_vec<float>(c, c->pos, x, true);
            if (x_t) store_vec<float>(c, c->xt, x_t, true);
            if (v_t) store_vec<float>(c, c->vt, v_t, false);
            if (v_prev) store_vec<float>(c, c->vprev, v_prev, false);
            if (y) store_vec<float>(c, c->y, y, true);
        }
    });
}

int vbd_set_beam_velocities(vbd_ctx* c, const double* la)
{
    return guarded([&] {
        if (!c || !la) fail(VBD_ERR_ARG, "NULL argument");
        if (c->beams.empty()) fail(VBD_ERR_ARG, "context was not built from beams");
        CK(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        DBuf dla, posd, vd;
        upload(dla, la, 6 * c->beams.size(), s);
        posd.alloc(c->n * 24);
        vd.alloc(c->n * 24);
        // rest positions in original order from x_t
        if (c->precision == VBD_PREC_F64)
            k_store_vec<double><<<blocks_for(c->n), 256, 0, s>>>(c->xt.as<double4>(), posd.as<double>(),
                                                                 c->inv.as<int>(), (int)c->n);
        else
            k_store_vec<float><<<blocks_for(c->n), 256, 0, s>>>(c->xt.as<float4>(), posd.as<double>(),
                                                                c->inv.as<int>(), (int)c->n, rest_for(c, true));
        k_beam_velocity<<<blocks_for(c->n), 256, 0, s>>>(c->beams_dev.as<BeamDev>(), (int)c->beams.size(),
                                                         dla.as<double>(), posd.as<double>(), c->n,
                                                         vd.as<double>());
        CK(cudaGetLastError());
        for (DBuf* d : {&c->vt, &c->vprev}) {
            if (c->precision == VBD_PREC_F64)
                k_load_vec<double><<<blocks_for(c->n), 256, 0, s>>>(vd.as<double>(), d->as<double4>(),
                                                                    c->perm.as<int>(), (int)c->n);
            else
                k_load_vec<float><<<blocks_for(c->n), 256, 0, s>>>(vd.as<double>(), d->as<float4>(),
                                                                   c->perm.as<int>(), (int)c->n);
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
    });
}

int vbd_set_fixed_targets(vbd_ctx* c, int64_t n, const int64_t* idx, const double* xyz)
{
    return guarded([&] {
        if (!c || (n > 0 && (!idx || !xyz))) fail(VBD_ERR_ARG, "NULL argument");
        if (n <= 0) return;
        CK(cudaSetDevice(c->device));
        std::vector<int>& hinv = c->hinv;
        if ((long long)hinv.size() != c->n) {
            hinv.resize(c->n);
            CK(cudaMemcpyAsync(hinv.data(), c->inv.p, c->n * 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        std::vector<int> ids(n);
        for (int64_t k = 0; k < n; ++k) {
            if (idx[k] < 0 || idx[k] >= c->n) fail(VBD_ERR_ARG, "vertex out of range");
            ids[k] = hinv[idx[k]];
            if (ids[k] < c->nfree_all) fail(VBD_ERR_ARG, "kinematic targets apply to fixed vertices only");
        }
        DBuf did, dxyz;
        upload_on(did, ids.data(), n, c->stream);
        upload_on(dxyz, xyz, 3 * n, c->stream);
        if (c->precision == VBD_PREC_F64)
            k_set_targets<double><<<blocks_for(n), 256, 0, c->stream>>>(did.as<int>(), dxyz.as<double>(), (int)n,
                                                                       c->xt.as<double4>(), c->pos.as<double4>());
        else
            k_set_targets<float><<<blocks_for(n), 256, 0, c->stream>>>(did.as<int>(), dxyz.as<double>(), (int)n,
                                                                      c->xt.as<float4>(), c->pos.as<float4>(),
                                                                      rest_for(c, true));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
    });
}

int vbd_step(vbd_ctx* c, const vbd_step_params* p, int32_t n_steps, vbd_step_result* res)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        if (c->in_step) fail(VBD_ERR_ARG, "a fine-grained step is in progress");
        CK(cudaSetDevice(c->device));
        if (c->precision == VBD_PREC_F64) do_step<double>(c, p, n_steps, res);
        else do_step<float>(c, p, n_steps, res);
    });
}

int vbd_color_pass(vbd_ctx* c, double* x, const double* x_t, const double* y, double h,
                   const int64_t* group, int64_t ng, int32_t mode, int32_t line_search, double eps_det)
{
    return guarded([&] {
        if (!c || !x || !x_t || !y) fail(VBD_ERR_ARG, "NULL argument");
        if (ng > 0 && !group) fail(VBD_ERR_ARG, "NULL group");
        if (mode != 0 && mode != 1) fail(VBD_ERR_ARG, "mode must be 0 or 1");
        if (!(h > 0.0)) fail(VBD_ERR_ARG, "h must be positive");
        CK(cudaSetDevice(c->device));
        if (c->precision == VBD_PREC_F64) do_color_pass<double>(c, x, x_t, y, h, group, ng, mode, line_search, eps_det);
        else do_color_pass<float>(c, x, x_t, y, h, group, ng, mode, line_search, eps_det);
    });
}

int vbd_initialize(vbd_ctx* c, const vbd_step_params* p)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        if (c->in_step) fail(VBD_ERR_ARG, "a fine-grained step is in progress");
        validate_params(p);
        CK(cudaSetDevice(c->device));
        c->cur = *p;
        CK(cudaMemsetAsync(c->flag.p, 0xff, 8, c->stream));
        if (c->precision == VBD_PREC_F64) enqueue_begin<double>(c);
        else enqueue_begin<float>(c);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
    });
}

int vbd_step_begin(vbd_ctx* c, const vbd_step_params* p)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        validate_params(p);
        CK(cudaSetDevice(c->device));
        c->cur = *p;
        c->omegas = omega_table(p->rho, p->n_max);
        c->in_step = true;
        CK(cudaMemsetAsync(c->flag.p, 0xff, 8, c->stream));
        CK(cudaMemsetAsync(c->stepctr.p, 0, 4, c->stream));
        auto begin = [&](auto tag) {
            typedef decltype(tag) R;
            ensure_materials<R>(c, p->h);
            if (c->coll_on) {  // DCD at x_t (solver.py:298-300)
                detect_dcd<R>(c);
                compile_contact_set<R>(c, c->xt);
            }
            enqueue_begin<R>(c);
        };
        if (c->precision == VBD_PREC_F64) begin(double{});
        else begin(float{});
        CK(cudaGetLastError());
    });
}

int vbd_step_color(vbd_ctx* c, int32_t color, int32_t iter)
{
    return guarded([&] {
        Nvtx nv_("colour %d (iteration %d)", (int)color, (int)iter);
        if (!c || !c->in_step) fail(VBD_ERR_ARG, "no step in progress");
        if (color < 0 || color >= c->ncolors) fail(VBD_ERR_ARG, "bad colour");
        if (c->coll_on && color == 0 && (iter - 1) % c->coll_ncol == 0) {  // CCD (solver.py:308-309)
            if (c->precision == VBD_PREC_F64) {
                detect_ccd<double>(c);
                compile_contact_set<double>(c, c->pos);
            } else {
                detect_ccd<float>(c);
                compile_contact_set<float>(c, c->pos);
            }
        }
        bool check = c->cur.rho == 0.0;
        if (c->precision == VBD_PREC_F64) color_sweep<double>(c, color, iter, check);
        else color_sweep<float>(c, color, iter, check);
        CK(cudaGetLastError());
    });
}

int vbd_step_iter_end(vbd_ctx* c, int32_t iter)
{
    return guarded([&] {
        if (!c || !c->in_step) fail(VBD_ERR_ARG, "no step in progress");
        if (iter < 1 || iter > c->cur.n_max) fail(VBD_ERR_ARG, "bad iteration");
        if (c->precision == VBD_PREC_F64) enqueue_iter_end<double>(c, iter);
        else enqueue_iter_end<float>(c, iter);
        CK(cudaGetLastError());
    });
}

int vbd_step_end(vbd_ctx* c, vbd_step_result* res)
{
    return guarded([&] {
        if (!c || !c->in_step) fail(VBD_ERR_ARG, "no step in progress");
        if (c->precision == VBD_PREC_F64) enqueue_end<double>(c);
        else enqueue_end<float>(c);
        CK(cudaGetLastError());
        c->in_step = false;
        read_result(c, res);
    });
}

int vbd_halo_count(vbd_ctx* c, int32_t side, int32_t color, int64_t* ns, int64_t* nr)
{
    return guarded([&] {
        if (!c || side < 0 || side > 1) fail(VBD_ERR_ARG, "bad argument");
        if (c->halo_send[side].empty()) {
            if (ns) *ns = 0;
            if (nr) *nr = 0;
            return;
        }
        if (color < 0 || color >= c->ncolors) fail(VBD_ERR_ARG, "bad colour");
        if (ns) *ns = c->halo_send_cnt[side][color][0];
        if (nr) *nr = c->halo_recv_cnt[side][color][0];
    });
}

int vbd_halo_pack(vbd_ctx* c, int32_t side, int32_t color, void* buf)
{
    return guarded([&] {
        if (!c || side < 0 || side > 1 || c->halo_send[side].empty()) fail(VBD_ERR_ARG, "no halo");
        long long n = c->halo_send_cnt[side][color][0];
        if (!n) return;
        const int* ids = c->halo_send[side][color][0]->as<int>();
        if (c->precision == VBD_PREC_F64)
            k_halo_pack<double><<<blocks_for(n), 256, 0, c->stream>>>(c->pos.as<double4>(), ids, (int)n,
                                                                      (double4*)buf);
        else
            k_halo_pack<float><<<blocks_for(n), 256, 0, c->stream>>>(c->pos.as<float4>(), ids, (int)n,
                                                                     (float4*)buf);
        CK(cudaGetLastError());
    });
}

int vbd_halo_unpack(vbd_ctx* c, int32_t side, int32_t color, const void* buf)
{
    return guarded([&] {
        if (!c || side < 0 || side > 1 || c->halo_recv[side].empty()) fail(VBD_ERR_ARG, "no halo");
        long long n = c->halo_recv_cnt[side][color][0];
        if (!n) return;
        const int* ids = c->halo_recv[side][color][0]->as<int>();
        if (c->precision == VBD_PREC_F64)
            k_halo_unpack<double><<<blocks_for(n), 256, 0, c->stream>>>(c->pos.as<double4>(), ids, (int)n,
                                                                        (const double4*)buf);
        else
            k_halo_unpack<float><<<blocks_for(n), 256, 0, c->stream>>>(c->pos.as<float4>(), ids, (int)n,
                                                                       (const float4*)buf);
        CK(cudaGetLastError());
    });
}

int vbd_halo_ghost_blocks(vbd_ctx* c, int32_t side, int64_t* begin, int64_t* count, int64_t* boundary)
{
    return guarded([&] {
        if (!c || side < 0 || side > 1) fail(VBD_ERR_ARG, "bad argument");
        for (int k = 0; k < c->ncolors; ++k) {
            if (begin) begin[k] = c->ghost_beg[side].empty() ? 0 : c->ghost_beg[side][k];
            if (count) count[k] = c->ghost_cnt[side].empty() ? 0 : c->ghost_cnt[side][k];
            if (boundary) boundary[k] = c->bnd_cnt[side].empty() ? 0 : c->bnd_cnt[side][k];
        }
    });
}

static void ensure_p2p_flags(vbd_ctx* c)
{
    if (c->p2p_flags.p) return;
    c->p2p_flags.alloc(64);
    CK(cudaMemset(c->p2p_flags.p, 0, 64));
}

int vbd_halo_p2p_local(vbd_ctx* c, void** pos, void** flags)
{
    return guarded([&] {
        if (!c || !pos || !flags) fail(VBD_ERR_ARG, "NULL argument");
        CK(cudaSetDevice(c->device));
        ensure_p2p_flags(c);
        *pos = c->pos.p;
        *flags = c->p2p_flags.p;
    });
}

int vbd_halo_p2p_export(vbd_ctx* c, void* pos_handle, void* flags_handle)
{
    return guarded([&] {
        if (!c || !pos_handle || !flags_handle) fail(VBD_ERR_ARG, "NULL argument");
        CK(cudaSetDevice(c->device));
        ensure_p2p_flags(c);
        cudaIpcMemHandle_t h1, h2;
        CK(cudaIpcGetMemHandle(&h1, c->pos.p));
        CK(cudaIpcGetMemHandle(&h2, c->p2p_flags.p));
        std::memcpy(pos_handle, &h1, sizeof h1);
        std::memcpy(flags_handle, &h2, sizeof h2);
    });
}

int vbd_ipc_open(int device, const void* handle, void** ptr)
{
    return guarded([&] {
        if (!handle || !ptr) fail(VBD_ERR_ARG, "NULL argument");
        CK(cudaSetDevice(device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int vbd_ipc_close(void* ptr)
{
    return guarded([&] { CK(cudaIpcCloseMemHandle(ptr)); });
}

int vbd_halo_p2p_connect(vbd_ctx* c, int32_t side, void* peer_pos, void* peer_flags,
                         const int64_t* peer_ghost_begin, const int64_t* peer_ghost_count)
{
    return guarded([&] {
        if (!c || side < 0 || side > 1) fail(VBD_ERR_ARG, "NULL argument");
        if (!peer_pos) {  // disconnect this side (e.g. falling back to the NCCL halo)
            c->peer_pos[side] = nullptr;
            c->peer_flag_slot[side] = nullptr;
            if (c->p2p_gexec) {
                cudaGraphExecDestroy(c->p2p_gexec);
                c->p2p_gexec = nullptr;
            }
            return;
        }
        if (!peer_flags || !peer_ghost_begin || !peer_ghost_count) fail(VBD_ERR_ARG, "NULL argument");
        if (c->bnd_cnt[side].empty()) fail(VBD_ERR_ARG, "context is not a slab");
        CK(cudaSetDevice(c->device));
        ensure_p2p_flags(c);
        for (int k = 0; k < c->ncolors; ++k)
            if (peer_ghost_count[k] != c->bnd_cnt[side][k])
                fail(VBD_ERR_ARG, "neighbour ghost block does not match this slab's boundary block");
        c->peer_pos[side] = peer_pos;
        // my signal lands in the neighbour's slot that faces me
        c->peer_flag_slot[side] = static_cast<unsigned long long*>(peer_flags) + (side == 0 ? 1 : 0);
        c->peer_ghost_beg[side].assign(peer_ghost_begin, peer_ghost_begin + c->ncolors);
        if (c->p2p_gexec) {
            cudaGraphExecDestroy(c->p2p_gexec);
            c->p2p_gexec = nullptr;
        }
    });
}

int vbd_step_p2p_launch(vbd_ctx* c, const vbd_step_params* p)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        validate_params(p);
        CK(cudaSetDevice(c->device));
        ensure_p2p_flags(c);
        c->cur = *p;
        c->omegas = omega_table(p->rho, p->n_max);
        cudaStream_t s = c->stream;
        if (c->precision == VBD_PREC_F64) ensure_materials<double>(c, p->h);
        else ensure_materials<float>(c, p->h);
        CK(cudaMemsetAsync(c->flag.p, 0xff, 8, s));
        CK(cudaMemsetAsync(c->stepctr.p, 0, 4, s));
        GraphKey key{*p};
        if (!c->p2p_gexec || !(key == c->p2p_key)) {
            if (c->p2p_gexec) {
                cudaGraphExecDestroy(c->p2p_gexec);
                c->p2p_gexec = nullptr;
            }
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            if (c->precision == VBD_PREC_F64) enqueue_step_p2p<double>(c);
            else enqueue_step_p2p<float>(c);
            CK(cudaStreamEndCapture(s, &g));
            CK(cudaGraphInstantiate(&c->p2p_gexec, g, 0));
            cudaGraphDestroy(g);
            c->p2p_key = key;
        }
        CK(cudaGraphLaunch(c->p2p_gexec, s));
    });
}

int vbd_step_p2p_finish(vbd_ctx* c, vbd_step_result* res)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL ctx");
        CK(cudaSetDevice(c->device));
        read_result(c, res);
        int err = read_scalar<int>(c->p2p_flags.as<unsigned long long>() + 3, c->stream);
        if (err) fail(VBD_ERR_INTERNAL, "P2P halo barrier timed out (neighbour not progressing)");
    });
}

int vbd_greedy_color(int64_t n, const int64_t* noff, const int64_t* nids, const int64_t* order,
                     int device, int64_t* color_of, int64_t* num_colors)
{
    return guarded([&] {
        if (n < 0 || !noff || !color_of || (n > 0 && noff[n] > 0 && !nids)) fail(VBD_ERR_ARG, "bad CSR");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            fail(VBD_ERR_NODEVICE, "no CUDA device available (no CPU fallback)");
        CK(cudaSetDevice(device));
        if (n == 0) {
            if (num_colors) *num_colors = 0;
            return;
        }
        if (n >= (1LL << 31)) fail(VBD_ERR_UNSUPPORTED, "graph too large");
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
        long long m = noff[n];
        std::vector<int> ids(m);
        for (long long k = 0; k < m; ++k) {
            if (nids[k] < 0 || nids[k] >= n) fail(VBD_ERR_ARG, "neighbour id out of range");
            ids[k] = (int)nids[k];
        }
        DBuf doff, dids, drank, dcol;
        upload(doff, noff, n + 1, s);
        upload(dids, ids.data(), m, s);
        const long long* rank = nullptr;
        if (order) {
            std::vector<long long> r(n, -1);
            for (long long k = 0; k < n; ++k) {
                if (order[k] < 0 || order[k] >= n || r[order[k]] >= 0)
                    fail(VBD_ERR_ARG, "order must be a permutation of all vertices");
                r[order[k]] = k;
            }
            upload(drank, r.data(), n, s);
            rank = drank.as<long long>();
        }
        dcol.alloc(n * 4);
        run_jp(doff.as<long long>(), dids.as<int>(), rank, n, dcol.as<int>(), s);
        std::vector<int> hc(n);
        CK(cudaMemcpyAsync(hc.data(), dcol.p, n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        long long mx = -1;
        for (long long v = 0; v < n; ++v) {
            color_of[v] = hc[v];
            mx = std::max<long long>(mx, hc[v]);
        }
        if (num_colors) *num_colors = mx + 1;
    });
}

int vbd_set_contacts(vbd_ctx* c, int64_t count, const int64_t* idx, const double* gamma,
                     const uint8_t* refresh, const double* normal, const double* tangent,
                     const double* k_c, const int64_t* cv_off, const int64_t* cv_cid,
                     const int64_t* cv_slot, double mu_c, double eps_v)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL context");
        if (count < 0) fail(VBD_ERR_ARG, "negative contact count");
        c->ncontacts = 0;
        if (count == 0) return;
        to_absolute(c);
        if (!idx || !gamma || !refresh || !normal || !tangent || !k_c || !cv_off || !cv_cid || !cv_slot)
            fail(VBD_ERR_ARG, "missing contact arrays");
        if (!(eps_v > 0.0) || mu_c < 0.0) fail(VBD_ERR_ARG, "bad friction parameters");
        if (c->hinv.empty()) {
            c->hinv.resize(c->n);
            CK(cudaMemcpy(c->hinv.data(), c->inv.p, c->n * 4, cudaMemcpyDeviceToHost));
        }
        const long long N = c->n;
        if ((long long)c->hperm.size() != N) {
            c->hperm.resize(N);
            for (long long o = 0; o < N; ++o) c->hperm[c->hinv[o]] = (int)o;
        }
        const std::vector<int>& perm = c->hperm;
        const bool f64p = c->precision == VBD_PREC_F64;
        std::vector<int4> ci(count);
        std::vector<double> cr(16 * count);
        for (long long k = 0; k < count; ++k) {
            int ids[4];
            for (int q = 0; q < 4; ++q) {
                const int64_t v = idx[4 * k + q];
                if (v < 0 || v >= N) fail(VBD_ERR_ARG, "contact index out of range");
                ids[q] = c->hinv[v];
            }
            ci[k] = make_int4(ids[0], ids[1], ids[2], ids[3]);
            double* r = &cr[16 * k];
            for (int q = 0; q < 4; ++q) r[q] = gamma[4 * k + q];
            r[4] = normal[3 * k]; r[5] = normal[3 * k + 1]; r[6] = normal[3 * k + 2]; r[7] = k_c[k];
            for (int q = 0; q < 4; ++q) r[8 + q] = tangent[6 * k + q];
            r[12] = tangent[6 * k + 4]; r[13] = tangent[6 * k + 5];
            r[14] = refresh[k] ? 1.0 : 0.0; r[15] = 0.0;
        }
        const long long ns = c->nsolve;
        std::vector<long long> off(ns + 1, 0);
        for (long long i = 0; i < ns; ++i) {
            const int o = perm[i];
            off[i + 1] = off[i] + (cv_off[o + 1] - cv_off[o]);
        }
        std::vector<int> cc(std::max<long long>(off[ns], 1)), cs(std::max<long long>(off[ns], 1));
        for (long long i = 0; i < ns; ++i) {
            const int o = perm[i];
            long long w = off[i];
            for (long long kk = cv_off[o]; kk < cv_off[o + 1]; ++kk, ++w) {
                if (cv_cid[kk] < 0 || cv_cid[kk] >= count || cv_slot[kk] < 0 || cv_slot[kk] > 3)
                    fail(VBD_ERR_ARG, "bad contact incidence");
                cc[w] = (int)cv_cid[kk];
                cs[w] = (int)cv_slot[kk];
            }
        }
        cudaStream_t s = c->stream;
        upload(c->coff, off.data(), off.size(), s);
        upload(c->ccid, cc.data(), cc.size(), s);
        upload(c->cslot, cs.data(), cs.size(), s);
        upload(c->cidx, ci.data(), ci.size(), s);
        if (f64p) {
            upload(c->creal, cr.data(), cr.size(), s);
        } else {
            std::vector<float> crf(cr.begin(), cr.end());
            upload(c->creal, crf.data(), crf.size(), s);
        }
        CK(cudaStreamSynchronize(s));
        c->mu_c = mu_c;
        c->eps_v = eps_v;
        c->ncontacts = count;
        if (c->gexec) {  // captured step graphs hold the old contact pointers
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
    });
}

int vbd_set_collision(vbd_ctx* c, int64_t ntri, const int64_t* tris, int64_t nedge, const int64_t* edges,
                      double cell, double k_c, double mu_c, double eps_v, double dcd_radius,
                      int32_t has_max_depth, double max_depth, int32_t n_col)
{
    return guarded([&] {
        if (!c) fail(VBD_ERR_ARG, "NULL context");
        c->coll_on = false;
        c->ncontacts = 0;
        if (c->gexec) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        c->cg_ready = c->cg_pending = false;
        for (long long& m : c->mx_cell) m = 0;
        for (long long& m : c->mx_join) m = 0;
        if (c->cg_exec) {
            cudaGraphExecDestroy(c->cg_exec);
            c->cg_exec = nullptr;
        }
        if (ntri <= 0) return;
        to_absolute(c);
        if (!tris || (nedge > 0 && !edges)) fail(VBD_ERR_ARG, "missing surface arrays");
        if (!(cell > 0.0) || !(k_c > 0.0) || mu_c < 0.0 || !(eps_v > 0.0) || dcd_radius < 0.0 || n_col < 1)
            fail(VBD_ERR_ARG, "bad contact parameters");
        if (c->hinv.empty()) {
            c->hinv.resize(c->n);
            CK(cudaMemcpy(c->hinv.data(), c->inv.p, c->n * 4, cudaMemcpyDeviceToHost));
        }
        const long long N = c->n;
        auto map = [&](int64_t v) {
            if (v < 0 || v >= N) fail(VBD_ERR_ARG, "surface index out of range");
            return c->hinv[v];
        };
        std::vector<int64_t> sv(tris, tris + 3 * ntri);
        std::sort(sv.begin(), sv.end());
        sv.erase(std::unique(sv.begin(), sv.end()), sv.end());
        std::vector<int> svm(sv.size());
        for (size_t k = 0; k < sv.size(); ++k) svm[k] = map(sv[k]);
        std::vector<int4> tr(ntri);
        for (long long k = 0; k < ntri; ++k) tr[k] = make_int4(map(tris[3 * k]), map(tris[3 * k + 1]), map(tris[3 * k + 2]), 0);
        std::vector<int2> ed(std::max<int64_t>(nedge, 1));
        for (long long k = 0; k < nedge; ++k) ed[k] = make_int2(map(edges[2 * k]), map(edges[2 * k + 1]));
        std::vector<unsigned char> act(N);
        for (long long v = 0; v < N; ++v) act[v] = v < c->nfree_all ? 1 : 0;
        cudaStream_t s = c->stream;
        upload(c->csv, svm.data(), svm.size(), s);
        upload(c->ctri, tr.data(), tr.size(), s);
        upload(c->cedge, ed.data(), ed.size(), s);
        upload(c->cactive, act.data(), act.size(), s);
        c->ccoll.alloc((size_t)std::max<long long>(N, 1));
        CK(cudaMemsetAsync(c->ccoll.p, 0, N, s));
        CK(cudaStreamSynchronize(s));
        c->nsv = (int)sv.size();
        c->ntri = (int)ntri;
        c->nedge = (int)std::max<int64_t>(nedge, 0);
        c->coll_cell = cell;
        c->coll_kc = k_c;
        c->mu_c = mu_c;
        c->eps_v = eps_v;
        c->coll_dcd_r = dcd_radius;
        c->coll_has_max_depth = has_max_depth;
        c->coll_max_depth = max_depth;
        c->coll_ncol = n_col;
        c->coll_on = true;
    });
}

int vbd_detect_contacts(vbd_ctx* c, int32_t which, int64_t cap, int64_t* count, int64_t* idx, double* gamma,
                        double* normal, int32_t* ccd)
{
    return guarded([&] {
        if (!c || !count) fail(VBD_ERR_ARG, "NULL argument");
        if (!c->coll_on) fail(VBD_ERR_ARG, "no collision surface (vbd_set_collision)");
        auto run = [&](auto tag) {
            typedef decltype(tag) R;
            if (which == 0) {
                detect_dcd<R>(c);
                compile_contact_set<R>(c, c->xt);
            } else {
                detect_ccd<R>(c);
                compile_contact_set<R>(c, c->pos);
            }
        };
        if (c->precision == VBD_PREC_F64) run(double{});
        else run(float{});
        const long long n = which == 0 ? c->ndcd : c->nccd;
        *count = n;
        if (!idx || cap <= 0) return;
        std::vector<ContactRec> h((size_t)n);
        if (n) CK(cudaMemcpy(h.data(), (which == 0 ? c->dcd_recs : c->ccd_recs).p, n * sizeof(ContactRec),
                             cudaMemcpyDeviceToHost));
        if (c->hperm.size() != (size_t)c->n) {
            c->hperm.resize(c->n);
            for (long long o = 0; o < c->n; ++o) c->hperm[c->hinv[o]] = (int)o;
        }
        for (long long k = 0; k < std::min<long long>(n, cap); ++k) {
            const int ids[4] = {h[k].idx.x, h[k].idx.y, h[k].idx.z, h[k].idx.w};
            for (int q = 0; q < 4; ++q) {
                idx[4 * k + q] = c->hperm[ids[q]];
                if (gamma) gamma[4 * k + q] = h[k].g[q];
            }
            if (normal)
                for (int q = 0; q < 3; ++q) normal[3 * k + q] = h[k].n[q];
            if (ccd) ccd[k] = h[k].ccd;
        }
    });
}

int vbd_get_colliding(vbd_ctx* c, uint8_t* flags)
{
    return guarded([&] {
        if (!c || !flags) fail(VBD_ERR_ARG, "NULL argument");
        std::vector<unsigned char> h(c->n, 0);
        if (c->coll_on) CK(cudaMemcpy(h.data(), c->ccoll.p, c->n, cudaMemcpyDeviceToHost));
        for (long long o = 0; o < c->n; ++o) flags[o] = h[c->hinv.empty() ? o : c->hinv[o]];
    });
}

}  // extern "C"

// G(x) partial sums of the current iterate: b1 + b2 + b3 block partials to add (ascending) and
// b3 contact-gap maxima after them.  Enqueued only; the caller reduces on the host.
struct EnergyLayout {
    unsigned b1, b2, b3;
    unsigned sums() const { return b1 + b2 + b3; }
    unsigned total() const { return b1 + b2 + 2 * b3; }
};

EnergyLayout energy_layout(const vbd_ctx* c)
{
    return {blocks_for(std::max<long long>(c->nsolve, 1) * 4), blocks_for(std::max<long long>(c->n, 1)),
            c->ncontacts ? blocks_for(c->ncontacts) : 0u};
}

void enqueue_energy(vbd_ctx* c, double h, const EnergyLayout& L, double* part)
{
    cudaStream_t s = c->stream;
    auto run = [&](auto tag) {
        typedef decltype(tag) R;
        if (std::isnan(c->mat_h)) ensure_materials<R>(c, 1.0);  // rest data only
        K1Args<R> a = k1_args<R>(c, 1e-10, 0, false, 0);
        k_energy_elastic<R, 4><<<L.b1, 256, 0, s>>>(a, (int)c->nsolve, part);
        k_energy_vertex<R><<<L.b2, 256, 0, s>>>(a, c->mass.as<R>(), (int)c->n, 1.0 / (h * h), part + L.b1);
        if (c->ncontacts)
            k_energy_contact<R><<<L.b3, 256, 0, s>>>(c->cidx.as<int4>(), c->creal.as<typename Vec4<R>::T>(),
                                                     (int)c->ncontacts, a.pos, part + L.b1 + L.b2,
                                                     part + L.b1 + L.b2 + L.b3);
    };
    if (c->precision == VBD_PREC_F64) run(double{});
    else run(float{});
    CK(cudaGetLastError());
}

double reduce_energy(const EnergyLayout& L, const double* h, double* max_gap = nullptr)
{
    double acc = 0.0, mx = 0.0;
    for (unsigned i = 0; i < L.sums(); ++i) acc += h[i];
    for (unsigned i = L.sums(); i < L.total(); ++i) mx = std::max(mx, h[i]);
    if (max_gap) *max_gap = mx;
    return acc;
}

double energy_now(vbd_ctx* c, double h, double* max_gap = nullptr)
{
    const EnergyLayout L = energy_layout(c);
    DBuf part;
    part.alloc_on((size_t)L.total() * sizeof(double), c->stream);
    enqueue_energy(c, h, L, part.as<double>());
    std::vector<double> hp(L.total());
    CK(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return reduce_energy(L, hp.data(), max_gap);
}

extern "C" {

int vbd_energy_metrics(vbd_ctx* c, double h, double* G, int64_t* contacts, double* max_gap)
{
    return guarded([&] {
        if (!c || !G) fail(VBD_ERR_ARG, "NULL argument");
        if (!(h > 0.0)) fail(VBD_ERR_ARG, "h must be positive");
        CK(cudaSetDevice(c->device));
        double mx = 0.0;
        *G = energy_now(c, h, &mx);
        if (contacts) *contacts = c->ncontacts;
        if (max_gap) *max_gap = mx;
    });
}

int vbd_energy(vbd_ctx* c, double h, double* G) { return vbd_energy_metrics(c, h, G, nullptr, nullptr); }

}  // extern "C"

// ---- baselines.descend on the device (baselines.py:152-189) ---------------------------------

template <typename R>
void descend_impl(vbd_ctx* c, int method, int n_iters, double h, double rho, double eps_det, int ls,
                  double* g, double* wall_ms)
{
    typedef typename Vec4<R>::T R4;
    Nvtx nv_("vbd_descend (method %d, %d iterations)", method, n_iters);
    cudaStream_t s = c->stream;
    const size_t vb = (size_t)c->n * c->r4();
    ensure_materials<R>(c, h);
    k_fill_mih2<R><<<blocks_for(std::max<long long>(c->n, 1)), 256, 0, s>>>(c->y.as<R4>(), c->mass.as<R>(),
                                                                          (int)c->n, h * h);
    vbd_step_params p{};
    p.h = h;
    p.n_max = n_iters;
    p.rho = method == 1 ? rho : 0.0;  // plain vbd never blends (omega_n == 1 for rho == 0)
    p.eps_det = eps_det;
    p.line_search = ls;
    c->cur = p;
    c->omegas = omega_table(p.rho, n_iters);
    CK(cudaMemsetAsync(c->flag.p, 0xff, 8, s));
    CK(cudaMemsetAsync(c->stepctr.p, 0, 4, s));
    // x_prev1 = x, x_pp = None (baselines.py:165-166): K3's history at iteration 2 reads ha
    if (p.rho != 0.0) CK(cudaMemcpyAsync(c->ha.p, c->pos.p, vb, cudaMemcpyDeviceToDevice, s));
    const EnergyLayout L = energy_layout(c);
    DBuf part, ckpt, xn;
    part.alloc_on((size_t)(n_iters + 1) * L.total() * sizeof(double), s);
    double* pp = part.as<double>();
    const bool sweep = method <= 1;
    double g_check = 0.0;
    std::vector<double> hp(L.total());
    auto sync_energy = [&](double* slot) {
        CK(cudaMemcpyAsync(hp.data(), slot, L.total() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return reduce_energy(L, hp.data());
    };
    enqueue_energy(c, h, L, pp);
    if (!sweep) {
        ckpt.alloc_on(vb, s);
        xn.alloc_on(vb, s);
        CK(cudaMemcpyAsync(ckpt.p, c->pos.p, vb, cudaMemcpyDeviceToDevice, s));
        g_check = sync_energy(pp);
    }
    std::vector<cudaEvent_t> ev(n_iters + 1);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], s));
    for (int n = 1; n <= n_iters; ++n) {
        if (sweep) {
            for (int col = 0; col < c->ncolors; ++col) color_sweep<R>(c, col, n, false);
            enqueue_iter_end<R>(c, n);
        } else {
            // block_jacobi_step / gd_step (baselines.py:92-104): every vertex against the previous
            // iterate, mode 0 block solves or mode 1 preconditioned gradient steps
            K1Args<R> a = k1_args<R>(c, eps_det, method == 3 ? 1 : 0, false, n);
            a.line_search = ls;
            a.vbeg = 0;
            a.count = (int)c->nsolve;
            a.out = c->out.as<R4>();
            launch_k1<R>(c, a, s);
            CK(cudaMemcpyAsync(c->pos.p, c->out.p, (size_t)c->nsolve * c->r4(), cudaMemcpyDeviceToDevice, s));
            if (n % 8 == 0) {  // _LS_PERIOD (baselines.py:22, 180-183)
                CK(cudaMemcpyAsync(xn.p, c->pos.p, vb, cudaMemcpyDeviceToDevice, s));
                double alpha = 1.0;
                bool ok = false;
                for (int k = 0; k <= 16 && !ok; ++k) {  // _MAX_HALVINGS (baselines.py:23, 139-149)
                    k_ls_blend<R><<<blocks_for(c->n), 256, 0, s>>>(c->pos.as<R4>(), ckpt.as<R4>(),
                                                                 xn.as<R4>(), alpha, (int)c->n);
                    enqueue_energy(c, h, L, pp + (size_t)n * L.total());
                    ok = sync_energy(pp + (size_t)n * L.total()) <= g_check;
                    alpha *= 0.5;
                }
                if (!ok) CK(cudaMemcpyAsync(c->pos.p, ckpt.p, vb, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(ckpt.p, c->pos.p, vb, cudaMemcpyDeviceToDevice, s));
                enqueue_energy(c, h, L, pp + (size_t)n * L.total());
                g_check = sync_energy(pp + (size_t)n * L.total());
            }
        }
        enqueue_energy(c, h, L, pp + (size_t)n * L.total());
        CK(cudaEventRecord(ev[n], s));
    }
    CK(cudaGetLastError());
    std::vector<double> all((size_t)(n_iters + 1) * L.total());
    CK(cudaMemcpyAsync(all.data(), pp, all.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int n = 0; n <= n_iters; ++n) {
        g[n] = reduce_energy(L, all.data() + (size_t)n * L.total());
        float ms = 0.f;
        if (n) CK(cudaEventElapsedTime(&ms, ev[0], ev[n]));
        if (wall_ms) wall_ms[n] = ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
}

extern "C" {

int vbd_descend(vbd_ctx* c, int32_t method, int32_t n_iters, double h, double rho, double eps_det,
                int32_t line_search, double* g, double* wall_ms)
{
    return guarded([&] {
        if (!c || !g) fail(VBD_ERR_ARG, "NULL argument");
        if (c->in_step) fail(VBD_ERR_ARG, "a fine-grained step is in progress");
        if (method < 0 || method > 3) fail(VBD_ERR_ARG, "method must be 0 vbd, 1 vbd-cheb, 2 jacobi or 3 gd");
        if (n_iters < 0) fail(VBD_ERR_ARG, "n_iters must be >= 0");
        if (!(h > 0.0)) fail(VBD_ERR_ARG, "h must be positive");
        if (!(rho >= 0.0 && rho < 1.0)) fail(VBD_ERR_ARG, "rho must be in [0, 1)");
        CK(cudaSetDevice(c->device));
        if (c->precision == VBD_PREC_F64) descend_impl<double>(c, method, n_iters, h, rho, eps_det, line_search, g, wall_ms);
        else descend_impl<float>(c, method, n_iters, h, rho, eps_det, line_search, g, wall_ms);
    });
}

int vbd_resident_timeline(vbd_ctx* c, int64_t* out, int64_t cap, int64_t* n)
{
    return guarded([&] {
        if (!c || !n) fail(VBD_ERR_ARG, "NULL argument");
        *n = 0;
        if (!c->res_prof.p || c->res_mode <= 0) return;
        const int64_t have = (int64_t)(c->res_prof.bytes / 8);
        const int64_t m = std::min<int64_t>(cap, have);
        if (m > 0 && out) {
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaMemcpy(out, c->res_prof.p, (size_t)m * 8, cudaMemcpyDeviceToHost));
        }
        *n = m;
    });
}

int vbd_profile_color_pass(vbd_ctx* c, double h, int32_t reps, double* ms)
{
    return guarded([&] {
        if (!c || !ms || reps < 1) fail(VBD_ERR_ARG, "bad argument");
        CK(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        c->cur.eps_det = c->cur.eps_det > 0 ? c->cur.eps_det : 1e-10;
        if (c->precision == VBD_PREC_F64) ensure_materials<double>(c, h);
        else ensure_materials<float>(c, h);
        auto sweep = [&](int col) {
            if (c->precision == VBD_PREC_F64) color_sweep<double>(c, col, 1, false);
            else color_sweep<float>(c, col, 1, false);
        };
        // colours in step order (each launch reads what the previous colours wrote, as in
        // the step); one event pair per launch
        const int nc = c->ncolors;
        std::vector<cudaEvent_t> ev(2 * (size_t)nc * reps);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        for (int col = 0; col < nc; ++col) sweep(col);  // warm-up sweep
        for (int r = 0; r < reps; ++r)
            for (int col = 0; col < nc; ++col) {
                const size_t k = 2 * ((size_t)r * nc + col);
                CK(cudaEventRecord(ev[k], s));
                sweep(col);
                CK(cudaEventRecord(ev[k + 1], s));
            }
        CK(cudaStreamSynchronize(s));
        for (int col = 0; col < nc; ++col) {
            double acc = 0.0;
            for (int r = 0; r < reps; ++r) {
                const size_t k = 2 * ((size_t)r * nc + col);
                float t = 0;
                CK(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
                acc += t;
            }
            ms[col] = acc / reps;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

int vbd_fma_peak(int device, int precision, int packed, double seconds, double* tflops)
{
    return guarded([&] {
        if (!tflops || seconds <= 0) fail(VBD_ERR_ARG, "bad argument");
        CK(cudaSetDevice(device));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const int mode = precision == VBD_PREC_F64 ? 2 : (packed ? 1 : 0);
        auto launch = [&](int iters, cudaStream_t s) {
            const unsigned grid = 8u * (unsigned)sms;  // 8 x 256 threads = 64 warps per SM
            if (mode == 0) k_fma_peak<0><<<grid, 256, 0, s>>>(nullptr, iters, 0.999f, 1e-3f);
            else if (mode == 1) k_fma_peak<1><<<grid, 256, 0, s>>>(nullptr, iters, 0.999f, 1e-3f);
            else k_fma_peak<2><<<grid, 256, 0, s>>>(nullptr, iters, 0.999f, 1e-3f);
            CK(cudaGetLastError());
        };
        const double fma_per_iter = 8.0 * sms * 256.0 * 8.0 * (mode == 1 ? 2.0 : 1.0);
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        // calibrate one launch to ~20 ms, then repeat for `seconds`
        int iters = 1 << 12;
        float ms = 0.f;
        for (;;) {
            CK(cudaEventRecord(e0, s));
            launch(iters, s);
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms >= 5.0f || iters >= (1 << 26)) break;
            iters *= 4;
        }
        iters = (int)std::min<double>((double)(1 << 28), iters * (20.0 / std::max(ms, 1e-3f)));
        const int reps = std::max(1, (int)(seconds * 1e3 / 20.0));
        CK(cudaEventRecord(e0, s));
        for (int r = 0; r < reps; ++r) launch(iters, s);
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *tflops = 2.0 * fma_per_iter * (double)iters * reps / (ms * 1e-3) / 1e12;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(s);
    });
}

}  // extern "C"
