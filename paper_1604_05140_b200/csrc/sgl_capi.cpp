// C ABI of the B200 SGL transform (include/sglgpu.h): plans, device tables,
// workspaces, tile schedules and the stage sequences of fsglft / ifsglft
// (sgl_transform.cpp:274-348).  No CPU compute path: every transform runs the
// sm_100a kernels of sgl_kernels.cu.
#include "sglgpu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <tuple>
#include <vector>

#include "sgl_kernels.cuh"
#include "sgl_ozaki.cuh"
#include "sgl_tables.hpp"

namespace {

thread_local std::string g_last_error;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(e == cudaErrorMemoryAllocation ? SGLGPU_ENOMEM : SGLGPU_ECUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}

void ck_launch(int n, const char* what) {
    if (n < 0) ck(cudaGetLastError(), what);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SGLGPU_OK;
    } catch (const Fail& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SGLGPU_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SGLGPU_ECUDA;
    }
}

long long coefficient_count(int B) { return (long long)B * (B + 1) * (2 * B + 1) / 6; }
long long sample_count(int B) { return 8LL * B * B * B; }

template <class T>
T* dev_upload(const std::vector<T>& h) {
    T* d = nullptr;
    const size_t bytes = std::max<size_t>(sizeof(T), h.size() * sizeof(T));
    ck(cudaMalloc(&d, bytes), "cudaMalloc(table)");
    if (!h.empty()) ck(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return d;
}

struct DevBuf {
    double* p = nullptr;
    size_t cap = 0;  // doubles
    void ensure(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        ck(cudaMalloc(&p, n * sizeof(double)), "cudaMalloc(workspace)");
        cap = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// kLegFwdS: the Legendre forward over one shell slice of the fused spherical
// forward (tiles straddle the +m / -m halves).
// Device workspaces of one transform in flight: the intermediates G and S and
// the work-queue counters of the fused kernels.
struct Work {
    DevBuf G, S, counters;
    // pipelined spherical stage (SGL_PIPE): a second, high-priority stream for the
    // azimuthal launches and the events that chain them to the Legendre launches
    cudaStream_t st2 = nullptr;
    cudaEvent_t pev[10] = {};
    void ensure_pipe() {
        if (st2) return;
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        const char* e = std::getenv("SGL_PIPE_PRIO");
        const int pr = e && e[0] == '0' ? lo : hi;  // default: the azimuthal stream has priority
        ck(cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, pr), "cudaStreamCreateWithPriority");
        for (cudaEvent_t& ev : pev) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    }
    void release() {
        G.release();
        S.release();
        counters.release();
        if (st2) {
            cudaStreamDestroy(st2);
            for (cudaEvent_t& ev : pev) cudaEventDestroy(ev);
            st2 = nullptr;
        }
    }
};

// One host-memory call in flight (sglgpu_* with SGLGPU_MEM_HOST): its own
// workspaces, double-buffered device staging of inputs and outputs, three
// streams (H2D, compute, D2H) so that chunk k+1 uploads while chunk k computes
// and chunk k-1 downloads, and pinned host staging for pageable user memory.
// A plan keeps up to kHostSlots of them, so that host calls from several threads
// run concurrently (PCIe is full duplex: one caller's downloads overlap
// another's uploads).
constexpr int kHostSlots = 8;
struct HostSlot {
    Work w;
    DevBuf din[2], dout[2];
    double* hst[2] = {nullptr, nullptr};  // pinned staging pieces (pageable user memory)
    size_t hst_cap = 0;                   // doubles per staging piece
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    cudaEvent_t eh[2] = {}, ec[2] = {}, ed[2] = {}, es[2] = {};
    bool busy = false;
    void release() {
        w.release();
        for (int b = 0; b < 2; ++b) {
            din[b].release();
            dout[b].release();
            if (hst[b]) cudaFreeHost(hst[b]);
            hst[b] = nullptr;
            for (cudaEvent_t* e : {&eh[b], &ec[b], &ed[b], &es[b]})
                if (*e) cudaEventDestroy(*e);
        }
        for (cudaStream_t* q : {&sh, &sc, &sd})
            if (*q) cudaStreamDestroy(*q);
    }
};

enum Kind { kLegFwd = 0, kLegInv = 1, kRadFwd = 2, kRadInv = 3, kLegFwdS = 4 };

}  // namespace

struct sglgpu_plan {
    int B = 0;
    int device = 0;
    int num_sms = 148;
    size_t table_bytes = 0;
    double* d_tw = nullptr;
    double* d_bcal = nullptr;
    double* d_leg = nullptr;
    long long* d_leg_off = nullptr;
    double* d_W = nullptr;
    long long* d_W_off = nullptr;
    double* d_V = nullptr;
    long long* d_V_off = nullptr;
    double* d_r = nullptr;     // radial rule (separated cross-oracle only)
    double* d_amod = nullptr;
    // INT8 tensor-core (fixed-point slice) tables, sgl_ozaki.cuh
    struct OzTable {
        uint8_t* img = nullptr;
        long long* off = nullptr;
        int* rexp = nullptr;
        int* kpad = nullptr;
        int* corr = nullptr;
        int mtiles = 1;
    } oz_li;  // built on the first INT8 call (ensure_oz_li), not at plan creation
    size_t leg_count = 0;  // doubles of d_leg
    std::map<std::tuple<long long, int, int>, std::pair<sglk::oz::Unit*, int>> oz_units;
    Work main;  // workspaces of device-memory calls and the stage entry points (under mu)
    std::vector<std::unique_ptr<HostSlot>> slots;  // host-memory calls (acquired under mu)
    std::condition_variable slot_cv;
    std::map<std::tuple<int, int, int, int, int, int, int>, std::pair<sglk::TileMap*, int>> tiles;
    std::mutex mu;       // device-memory calls, stage entry points, slot acquisition
    std::mutex meta_mu;  // the tile-map cache and the profiling records
    std::atomic<int> last_launches{0};
    // live per-stage timing (sglgpu_profile_begin/end)
    bool profiling = false;
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> prof;
    std::vector<cudaEvent_t> ev_pool;
    // CUDA graphs of whole device-memory transforms, keyed by
    // (direction, batch, in, out, stream); replayed with one launch
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        int launches = 0;
        unsigned long long last_use = 0;
    };
    // key: direction, batch, in, out, stream, G workspace, S workspace (a graph is
    // never replayed after a workspace it references was reallocated)
    using GraphKey = std::tuple<int, size_t, const void*, void*, void*, void*, void*>;
    std::map<GraphKey, GraphEntry> graphs;
    std::map<GraphKey, int> seen;
    unsigned long long tick = 0;
};

namespace {

// Host-side mirror of the per-problem shapes in sgl_kernels.cu.
void problem_shape(Kind kind, int B, int batch, long long NB, int pid, bool real, int& M, int& N, int& K) {
    switch (kind) {
        case kLegFwdS:
        case kLegFwd: {
            const int am = pid >> 1, r = B - am - (pid & 1);
            M = r > 0 ? (r + 1) / 2 : 0;
            N = am == 0 || real ? (int)NB : 2 * (int)NB;
            K = B;
            break;
        }
        case kLegInv: {
            const int am = pid >> 1, r = B - am - (pid & 1);
            M = B;
            N = am == 0 || real ? (int)NB : 2 * (int)NB;
            K = r > 0 ? (r + 1) / 2 : 0;
            break;
        }
        case kRadFwd:
            M = B - pid;
            N = (real ? pid + 1 : 2 * pid + 1) * batch * 2;
            K = 2 * B;
            break;
        case kRadInv:
            M = 2 * B;
            N = (real ? pid + 1 : 2 * pid + 1) * batch * 2;
            K = B - pid;
            break;
    }
}

// Tile table for one grouped contraction (problems heaviest tile first), cached
// per shape.  Each problem gets the warp layout wm with the fewest
// (32 wm) x (128 / wm) tiles; SGL_WM_LEG / SGL_WM_RAD force one.
// sub_n > 0 restricts a Legendre launch to a sub-range of its tiles (the pipelined
// spherical stage): row blocks [sub_lo, sub_lo + sub_n) of every problem for the
// Legendre inverse (a slab of polar nodes), n-blocks [sub_lo, sub_lo + sub_n) of
// every sign half for the Legendre forward (a range of shells).
// wp: the caller runs the whole-transform radial forward (one S block, every degree), for
// which batched small bandlimits use the warp-private kernel (n-block sequences).
std::pair<sglk::TileMap*, int> tiles_for(sglgpu_plan* p, Kind kind, int batch, int SC, int lo, int hi,
                                         bool real = false, int sub_lo = 0, int sub_n = 0, bool wp = false) {
    const auto key = std::make_tuple((int)kind + (real ? 16 : 0) + (wp ? 32 : 0), batch, SC, lo, hi, sub_lo, sub_n);
    std::lock_guard<std::mutex> meta(p->meta_mu);
    auto it = p->tiles.find(key);
    if (it != p->tiles.end()) return it->second;
    const int B = p->B;
    const long long NB = 2LL * batch * SC;
    int plo = lo, phi = hi;
    const bool leg = kind == kLegFwd || kind == kLegInv || kind == kLegFwdS;
    if (leg) {
        plo = 0;
        phi = 2 * B;
    }
    static const char* const kind_env[5] = {"SGL_WM_LEGFWD", "SGL_WM_LEGINV", "SGL_WM_RADFWD", "SGL_WM_RADINV",
                                            "SGL_WM_LEGFWD"};
    const char* wm_env = std::getenv(kind_env[kind]);  // experiments: force one kind's warp layout
    if (!wm_env) wm_env = std::getenv(leg ? "SGL_WM_LEG" : "SGL_WM_RAD");
    const int wm_force = wm_env ? std::atoi(wm_env) : 0;
    struct Entry {
        int pid, lwm, halves, tm, tn, h0, mi0, ni0;
        long long work;  // per tile, for heaviest-first ordering
    };
    // radial forward on warp-private pipelines: batched small bandlimits, several waves deep
    bool radfwd_wp = false;
    if (kind == kRadFwd && wp && SC == 2 * B && lo == 0 && hi == B) {
        const char* e = std::getenv("SGL_RADFWD_WP");
        sglk::Geo gq{B, SC, batch, NB};
        long long cols = 0;
        for (int l = 0; l < B; ++l) cols += ((real ? l + 1 : 2 * l + 1) * 2LL * batch + 127) / 128 * ((B - l + 31) / 32);
        // opt-in: measured equal or slower (B = 64 x 64: 209 vs 209 us, real B = 32 x 4096: 864 -> 877,
        // sequences of 2 / 8: 835 / 950) -- at K = 2B <= 128 these tiles are bound by their epilogue
        // (the omega-order scatter with its per-column divisions), not by barriers or chunk issue
        radfwd_wp = (e && std::atoi(e)) && sglk::radfwd_wp_ok(gq, sglk::RadialBlocks{2 * B, 0, 0}) &&
                    cols >= 8LL * 4 * p->num_sms;
    }
    std::vector<Entry> ents;
    long long ntiles = 0;
    for (int pid = plo; pid < phi; ++pid) {
        int M, N, K;
        problem_shape(kind, B, batch, NB, pid, real, M, N, K);
        if (M <= 0 || N <= 0) continue;
        if (K <= 0 && kind != kLegInv) continue;  // LegInv with K = 0 must still write zeros
        // Legendre tiles never straddle the +m / -m halves of N (column addresses
        // stay affine inside a tile)
        const long long half = leg && kind != kLegFwdS ? NB : N;  // kLegFwdS: one tile spans both halves
        const int halves = (int)(N / half);
        // ties: the widest tile, except for the radial inverse (M = 2B rows of
        // V_l against a few coefficient columns), where 128 x 32 measured faster
        int lwm = 0;
        long long best = -1;
        for (int c = 0; c < 3; ++c) {
            const int l2 = kind == kRadInv ? 2 - c : c;
            const long long nt = (long long)((M + (32 << l2) - 1) / (32 << l2)) * ((half + (128 >> l2) - 1) / (128 >> l2));
            if (best < 0 || nt < best) {
                best = nt;
                lwm = l2;
            }
        }
        // radial forward at B >= 256: 64 x 64 tiles (measured: 493 -> 477 us at B = 256; no gain at B = 128)
        if (kind == kRadFwd && B >= 256 && !wm_force) lwm = 1;
        if (wm_force == 1 || wm_force == 2 || wm_force == 4) lwm = wm_force == 1 ? 0 : wm_force == 2 ? 1 : 2;
        if (radfwd_wp) lwm = 0;  // 32 x 128 tiles: one warp per 32 columns
        const int max_wm = kind == kLegFwdS ? 1 : kind == kLegFwd ? SGL_MAXWM_LEGFWD : kind == kLegInv ? SGL_MAXWM_LEGINV
                         : kind == kRadFwd ? SGL_MAXWM_RADFWD : SGL_MAXWM_RADINV;
        while ((1 << lwm) > max_wm) --lwm;
        const int bm = 32 << lwm, bn = 128 >> lwm;
        int tm = (M + bm - 1) / bm;
        long long tn = (half + bn - 1) / bn;
        if (tn > (1 << 30) / 2) fail(SGLGPU_EINVAL, "tile table: problem too wide");
        int mi0 = 0, ni0 = 0;
        if (sub_n > 0 && kind == kLegInv) {
            mi0 = sub_lo;
            tm = std::min(sub_n, tm - sub_lo);
        } else if (sub_n > 0 && kind == kLegFwd) {
            ni0 = sub_lo;
            tn = std::min<long long>(sub_n, tn - sub_lo);
        }
        if (tm <= 0 || tn <= 0) continue;
        const long long kk = std::max(K, 1);
        ents.push_back({pid, lwm, halves, tm, (int)tn, 0, mi0, ni0,
                        (std::min(bm, M) + 7) / 8 * 8 * ((std::min<long long>(bn, half) + 7) / 8 * 8) * kk});
        ntiles += (long long)tm * halves * tn;
    }
    // n-blocks per CTA for kinds built with sequences: short-K problems amortize
    // the CTA prologue and overlap each tile's epilogue with the next tile's
    // loads (LegInv, B = 128: 114.5 -> 112.6 us with 2; B = 64 x 64: 652 -> 588 us
    // and B = 32 x 4096: 4378 -> 3672 us with 4)
    int seq = 1;
    if (kind == kLegInv) {
        const int kmax = (B + 1) / 2;  // the Legendre inverse's K (degrees of one parity)
        // measured: B = 32, 64: 4; B = 128: 2; B = 256: the one-tile kernel (seq 2: +4%)
        seq = kmax <= 32 ? 4 : kmax <= 64 ? 2 : 1;
        {
            // the warp-private kernel loads its A panel once per sequence: 4 n-blocks at B >= 128
            // (B = 128: 95.2 us with 2, 94.8 with 4), 2 at B = 64, whose panel is small (B = 64 x 64:
            // 556 us with 1, 482 with 2, 493 with 3, 501 with 4, 526 with 8)
            const char* e = std::getenv("SGL_LEGINV_WP");
            sglk::Geo gq{B, SC, batch, NB};
            if ((!e || std::atoi(e)) && sglk::leginv_wp_ok(gq)) seq = kmax <= 32 ? 2 : kmax <= 64 ? 4 : 8;  // B = 256: 1190 us with 4, 1182 with 8
        }
        // sequences pay only when the launch is several waves deep: a single B = 64
        // function (~1k tiles) runs 18.7 -> 17.1 us without them
        if (ntiles < 2LL * 4 * p->num_sms) seq = 1;
        if (const char* e = std::getenv("SGL_SEQ")) seq = std::max(1, std::min(8, std::atoi(e)));
    }
    if (kind == kLegFwd && wp && sub_n == 0) {  // whole-transform Legendre forward on warp-private pipelines
        sglk::Geo gq{B, SC, batch, NB};
        gq.real = real ? 1 : 0;
        if (sglk::legfwd_wp_ok(gq)) {
            seq = 4;
            if (const char* e = std::getenv("SGL_SEQ_LEGFWD")) seq = std::max(2, std::min(8, std::atoi(e)));
        }
    }
    if (radfwd_wp) {
        seq = 4;
        if (const char* e = std::getenv("SGL_SEQ_RADFWD")) seq = std::max(2, std::min(8, std::atoi(e)));
    }
    if (kind == kRadInv && batch == 1 && !real) {  // RadInvSeq (one complex function)
        if (const char* e = std::getenv("SGL_SEQ_RADINV")) seq = std::max(1, std::min(8, std::atoi(e)));
    }
    if (seq == 1 && ntiles <= sglk::kMaxProblems) {  // one entry per tile, exact per-tile work
        std::vector<Entry> per;
        for (const Entry& e : ents) {
            int M, N, K;
            problem_shape(kind, B, batch, NB, e.pid, real, M, N, K);
            const long long half = leg && kind != kLegFwdS ? NB : N, kk = std::max(K, 1);
            const int bm = 32 << e.lwm, bn = 128 >> e.lwm;
            for (int mi = 0; mi < e.tm; ++mi)
                for (int h = 0; h < e.halves; ++h)
                    for (int ni = 0; ni < e.tn; ++ni) {
                        const int gm = e.mi0 + mi, gn = e.ni0 + ni;
                        const long long rows = std::min(bm, M - gm * bm), cols = std::min<long long>(bn, half - (long long)gn * bn);
                        per.push_back({e.pid, e.lwm, 1, 1, 1, h, gm, gn, (rows + 7) / 8 * 8 * ((cols + 7) / 8 * 8) * kk});
                    }
        }
        ents.swap(per);
    }
    // Legendre inverse, polar-slab-major order: all problems of row block mi (32
    // nodes j') before the next block, so G is written slab by slab and the slab
    // written last is still in L2 when the azimuthal inverse starts with it.
    // SGL_LEGINV_ORDER: 0 = problem-major, 1 = slabs ascending, 2 = descending.
    int slab_order = 0;
    const bool per_tile = seq == 1 && ntiles <= sglk::kMaxProblems;  // expanded above
    if (kind == kLegInv && !per_tile) {
        if (const char* e = std::getenv("SGL_LEGINV_ORDER")) slab_order = std::atoi(e);
        long long need = 0;
        for (const Entry& e : ents) need += e.tm;
        if (need > sglk::kMaxProblems) slab_order = 0;  // B = 256: 8 slabs x 512 problems
        if (slab_order) {
            std::vector<Entry> per;
            for (const Entry& e : ents)
                for (int mi = 0; mi < e.tm; ++mi)
                    per.push_back({e.pid, e.lwm, e.halves, 1, e.tn, 0, e.mi0 + mi, e.ni0, e.work});
            ents.swap(per);
        }
    }
    if ((int)ents.size() > sglk::kMaxProblems) fail(SGLGPU_EINVAL, "tile table: too many problems");
    std::stable_sort(ents.begin(), ents.end(), [slab_order](const Entry& a, const Entry& b) {
        if (slab_order && a.mi0 != b.mi0) return slab_order == 1 ? a.mi0 < b.mi0 : a.mi0 > b.mi0;
        return a.work > b.work;
    });
    auto* tm = new sglk::TileMap{};
    long long n = 0;
    tm->nprob = (int)ents.size();
    tm->seq = seq;
    for (size_t q = 0; q < ents.size(); ++q) {
        const Entry& e = ents[q];
        tm->first[q] = (int)n;
        tm->info[q] = e.pid | e.lwm << 16 | (e.halves - 1) << 18 | e.h0 << 19 | e.mi0 << 20 | (seq - 1) << 26;
        tm->tn[q] = e.tn;
        tm->ni0[q] = e.ni0;
        n += (long long)e.tm * e.halves * ((e.tn + seq - 1) / seq);
    }
    if (n >= (1LL << 31) - 1) fail(SGLGPU_EINVAL, "tile table: too many tiles");
    tm->first[ents.size()] = (int)n;
    const auto res = std::make_pair(tm, (int)n);
    p->tiles[key] = res;
    return res;
}

// INT8 tensor-core contractions (sgl_ozaki.cu): SGL_I8 = 0 (off), 1 (every kind
// built so far) or a comma list of kinds ("leginv").
bool i8_on(const char* kind) {
    const char* e = std::getenv("SGL_I8");
    if (!e) return false;
    if (e[0] == '0' && e[1] == 0) return false;
    if (e[0] == '1' && e[1] == 0) return true;
    return std::strstr(e, kind) != nullptr;
}

int i8_tpc() {
    const char* e = std::getenv("SGL_I8_TPC");
    return e ? std::max(1, std::atoi(e)) : 4;
}

// The INT8 Legendre-inverse table image (sgl_ozaki.cu), built from the plan's
// Legendre table on the first call that asks for it: the opt-in path costs
// default users neither plan-creation time nor memory.  Called outside graph
// capture (graphs are captured from the second call of a shape on).
void ensure_oz_li(sglgpu_plan* p) {
    std::lock_guard<std::mutex> meta(p->meta_mu);
    if (p->oz_li.img) return;
    const int B = p->B;
    std::vector<double> leg(p->leg_count);
    std::vector<long long> off(2 * B + 1);
    ck(cudaMemcpy(leg.data(), p->d_leg, leg.size() * sizeof(double), cudaMemcpyDeviceToHost), "download(legendre)");
    ck(cudaMemcpy(off.data(), p->d_leg_off, off.size() * sizeof(long long), cudaMemcpyDeviceToHost),
       "download(legendre_off)");
    const auto im = sglk::oz::build_leginv_image(B, leg, off);
    p->oz_li.off = dev_upload(im.off);
    p->oz_li.rexp = dev_upload(im.rexp);
    p->oz_li.kpad = dev_upload(im.kpad);
    p->oz_li.corr = dev_upload(im.corr);
    p->oz_li.mtiles = im.mtiles;
    p->oz_li.img = dev_upload(im.bytes);
}

// Legendre inverse: the INT8 tensor-core kernel when enabled, else the DMMA GEMM.
int leginv(sglgpu_plan* p, Work& w, const sglk::Geo& g, const sglk::SView& sv, const double* S, double* G,
           std::pair<sglk::TileMap*, int> lt, cudaStream_t st) {
    const bool ws = i8_on("ws");
    if (ws || i8_on("leginv")) {
        ensure_oz_li(p);
        const int tpc = ws ? -1 : i8_tpc();
        std::pair<sglk::oz::Unit*, int> un;
        {
            std::lock_guard<std::mutex> meta(p->meta_mu);
            const auto key = std::make_tuple(g.NB, g.real, tpc);
            auto it = p->oz_units.find(key);
            if (it == p->oz_units.end()) {
                const auto hu = ws ? sglk::oz::leginv_ws_units(p->B, g.NB, g.real != 0)
                                   : sglk::oz::leginv_units(p->B, g.NB, g.real != 0, tpc);
                sglk::oz::Unit* d = nullptr;
                ck(cudaMalloc(&d, std::max<size_t>(1, hu.size()) * sizeof(sglk::oz::Unit)), "cudaMalloc(units)");
                ck(cudaMemcpy(d, hu.data(), hu.size() * sizeof(sglk::oz::Unit), cudaMemcpyHostToDevice), "upload units");
                it = p->oz_units.emplace(key, std::make_pair(d, (int)hu.size())).first;
            }
            un = it->second;
        }
        sglk::oz::LegInvI8 prm{g, sv, S, G, p->oz_li.img, p->oz_li.off, p->oz_li.rexp, p->oz_li.kpad, un.first, tpc,
                               p->oz_li.mtiles};
        if (const char* tr = std::getenv("SGL_I8_TRACE")) prm.trace = reinterpret_cast<long long*>(std::strtoull(tr, nullptr, 0));
        prm.corr = p->oz_li.corr;
        w.counters.ensure(1);  // the call's own unit ticket (host slots run concurrently)
        prm.counter = reinterpret_cast<int*>(w.counters.p);
        prm.grid = p->num_sms;
        return ws ? sglk::oz::launch_legendre_inverse_ws(prm, un.second, st)
                  : sglk::oz::launch_legendre_inverse_i8(prm, un.second, st);
    }
    return sglk::launch_legendre_inverse(g, sv, S, G, p->d_leg, p->d_leg_off, lt.first, lt.second, st);
}

void set_device(sglgpu_plan* p) { ck(cudaSetDevice(p->device), "cudaSetDevice"); }

cudaEvent_t pool_event(sglgpu_plan* p) {
    std::lock_guard<std::mutex> meta(p->meta_mu);
    if (!p->ev_pool.empty()) {
        cudaEvent_t e = p->ev_pool.back();
        p->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

// Pipelined spherical stage of a single large transform (SGL_PIPE = slices, 0 = off):
// the azimuthal kernels are HBM-bound and the Legendre kernels FP64-bound, so the
// stage is cut into slices whose azimuthal and Legendre launches overlap on two
// streams -- by shell range in the forward direction (az(k+1) || legendre(k)), by
// slab of polar nodes in the inverse (legendre(k+1) || az(k)).
int pipe_slices(int B, int nb) {
    const char* e = std::getenv("SGL_PIPE");
    const int ns = e ? std::atoi(e) : 0;
    if (ns < 2 || nb != 1 || (B & (B - 1)) || B < 64) return 0;
    return (B / 32) % ns == 0 ? ns : 0;
}

// 16-shell G groups for large complex batches at B = 64 (sglk::Geo::az2x): -72 us per round
// trip of 64 functions (Legendre -106, azimuthal +35), even at 8, worse for one.
bool az2x_on(int B, int fb) {
    const char* e = std::getenv("SGL_AZ2X");
    if (e) return std::atoi(e) != 0 && B == 64;
    return B == 64 && fb >= 32;
}

// Brackets one stage launch with events when profiling is on.
template <class F>
int staged(sglgpu_plan* p, int stage, cudaStream_t st, F&& launch) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (p->profiling) {
        a = pool_event(p);
        b = pool_event(p);
        ck(cudaEventRecord(a, st), "cudaEventRecord");
    }
    const int k = launch();
    if (p->profiling) {
        ck(cudaEventRecord(b, st), "cudaEventRecord");
        std::lock_guard<std::mutex> meta(p->meta_mu);
        p->prof.emplace_back(stage, a, b);
    }
    return k;
}


// Second call with the same graph key?  (The table is bounded: callers that
// pass fresh buffers every call never reach the graph path.)
bool seen_twice(sglgpu_plan* p, const sglgpu_plan::GraphKey& key) {
    if (p->seen.size() > 4096) p->seen.clear();
    return p->seen[key]++ >= 1;
}

// Graph replay trims the gaps between kernels (eager launches leave ~1.5 us per
// kernel boundary at B = 128) and the host launch cost of small transforms.
bool use_graphs(int B, size_t batch) {
    const char* e = std::getenv("SGL_GRAPHS");
    if (e) return e[0] == '1';
    // measured (exp/step_time.py): B = 128, one function: 538.6 -> 529.8 us per round trip
    return (double)B * B * B * (double)batch <= 128.0 * 128 * 128 * 2;
}

// Largest batch chunk whose G + S workspaces stay under the budget
// (SGL_WORKSPACE_GB, default 6 GiB).
size_t batch_chunk(int B, size_t batch) {
    const size_t per = (size_t)(16 + 4) * B * B * B * sizeof(double);  // G + S per function
    static const size_t budget = [] {
        const char* e = std::getenv("SGL_WORKSPACE_GB");
        const double gb = e ? std::atof(e) : 6.0;
        return (size_t)(std::max(0.25, gb) * (double)(1ULL << 30));
    }();
    // the GEMM kernels index G, S and the coefficients of one call in 32 bits
    const size_t idx_cap = ((size_t)1 << 31) / ((size_t)16 * B * B * B);  // G: 16 B^3 doubles per function
    return std::max<size_t>(1, std::min({batch, budget / per, idx_cap}));
}

// Stage entry points run one launch per stage over the caller's whole batch: the
// GEMM kernels' 32-bit indexing bounds it (G: 16 B^3 doubles per function).
void check_stage_batch(int B, size_t batch, const char* who) {
    if ((double)batch * 16.0 * B * B * B >= 2147483648.0)
        fail(SGLGPU_EINVAL, std::string(who) + ": batch too large for one stage call (split it)");
}

// L2 residency of the azimuthal -> polar intermediate G: the spherical stage
// runs in slices whose G slice (64 B^2 bytes per shell and function) stays
// below ~SGL_G_CHUNK_MB, so the Legendre kernel reads (forward) / the inverse FFT
// reads (inverse) it from L2 right after it was written, instead of from HBM.
// For batch == 1 the slice is a shell range; for batches it is a function range.
struct Slices {
    int count;       // number of slices
    int shells;      // shells per slice (batch == 1) or 2B
    int functions;   // functions per slice (batch > 1) or 1
};

Slices plan_slices(int B, int nb) {
    // Measured on B200: slices cost more in per-launch tails than the L2 reuse
    // saves -- B = 128, one function: 16-64 MiB shell slices, 1800 -> 1374
    // transforms/s; B = 64 x 64 and B = 32 x 4096: 1 GiB function slices 2%
    // slower than none -- so transforms run unsliced (the workspace is bounded
    // by batch_chunk).  SGL_G_CHUNK_MB sets a slice size for experiments.
    double mb = 0.0;
    if (const char* e = std::getenv("SGL_G_CHUNK_MB")) mb = std::atof(e);
    const double per_shell = 64.0 * B * B;  // bytes of G per (shell, function)
    const long long cap = std::max(1LL, (long long)(mb * 1048576.0 / per_shell));
    Slices sl{1, 2 * B, nb};
    if (mb <= 0) return sl;
    if (nb == 1) {
        int sh = 2 * B;
        while (sh > cap && sh % 2 == 0) sh /= 2;  // 2B is a power of two for the FFT path
        sl.shells = sh;
        sl.count = (2 * B) / sh;
    } else {
        const long long per_fn = cap / (2 * B);
        const int fpc = (int)std::max(1LL, std::min<long long>(nb, per_fn));
        sl.functions = fpc;
        sl.count = (nb + fpc - 1) / fpc;
    }
    return sl;
}

// Stage sequences on device memory.  X: samples (function stride Psi complex),
// C: coefficients (function stride Omega complex).
// The fused persistent spherical forward (launch_spherical_forward_fused), opt-in
// with SGL_FUSED=1 for power-of-two 2B in [32, 256].  Measured at B = 128 (one
// function): 218 us against 95.5 + 94.2 us for the two kernels it replaces (its
// azimuthal items alone 125 us, its Legendre tiles alone 109 us -- the two
// latency-bound halves do not overlap on the same SMs, and the persistent loop
// adds per-item cost), with the L2 discard of consumed G lines 469 us.  Kept as a
// tested alternative; DESIGN.md section 4.  SGL_FUSED_SLICE sets the shell slice
// (default 32), SGL_FUSED_DISCARD=1 drops consumed G lines from L2,
// SGL_FUSED_GRID overrides the persistent grid.
int fused_slice_shells(int B, int nb, int lgib) {
    const char* e = std::getenv("SGL_FUSED");
    if (!e || e[0] != '1') return 0;
    if (B < 16 || B > 128 || (B & (B - 1))) return 0;
    int sls = 32;
    if (const char* v = std::getenv("SGL_FUSED_SLICE")) sls = std::atoi(v);
    if (sls < (1 << lgib) || sls > 32 || sls % (1 << lgib) || (2 * B) % sls) return 0;
    (void)nb;
    return sls;
}

// The fused small-bandlimit path (sgl_small.cu) for 2B <= 32 and batches of at most
// kSmallBatch functions (beyond that the staged path's wide kernels win: B = 16,
// 4 functions 157k vs 116k transforms/s, 16 functions 306k vs 369k);
// SGL_SMALL=0 turns it off.
constexpr int kSmallBatch = 8;
bool small_on(int B, int nb) {
    if (!sglk::small_path_ok(B) || nb > kSmallBatch) return false;
    const char* e = std::getenv("SGL_SMALL");
    return !(e && e[0] == '0');
}

int forward_device(sglgpu_plan* p, Work& w, const double* X, double* C, int nb, cudaStream_t st) {
    const int B = p->B;
    const size_t psi2 = 2 * (size_t)sample_count(B), om2 = 2 * (size_t)coefficient_count(B);
    if (small_on(B, nb)) {
        const int k = staged(p, 6, st, [&] {
            return sglk::launch_small_forward(B, nb, X, (long long)psi2 / 2, C, (long long)om2 / 2, p->d_leg, p->d_W,
                                              p->d_bcal, p->d_tw, st);
        });
        ck_launch(k, "small_forward");
        return k;
    }
    const Slices sl = plan_slices(B, nb);
    w.S.ensure((size_t)4 * B * B * B * nb);
    int n = 0, k;
    {
        sglk::Geo g{B, 2 * B, nb, 2LL * nb * 2 * B};
        const long long gsize = sglk::g_layout(g);
        const int sls = sl.count == 1 ? fused_slice_shells(B, nb, g.lgib) : 0;
        if (sls > 0) {
            w.G.ensure(2 * (size_t)gsize);
            const int nslices = nb * 2 * B / sls;
            w.counters.ensure((size_t)(1 + 2 * nslices + 1) / 2 + 1);
            auto lt = tiles_for(p, kLegFwdS, 1, sls, 0, 2 * B);
            const char* dz = std::getenv("SGL_FUSED_DISCARD");
            const char* gr = std::getenv("SGL_FUSED_GRID");
            k = staged(p, 6, st, [&] {
                return sglk::launch_spherical_forward_fused(
                    g, X, psi2, w.G.p, p->d_bcal, p->d_tw, w.S.p, sglk::SView{g.NB, 2 * B, 0}, p->d_leg,
                    p->d_leg_off, lt.first, lt.second, sls, reinterpret_cast<int*>(w.counters.p), dz && dz[0] == '1',
                    gr ? std::atoi(gr) : 0, st);
            });
            if (k != -2) {
                ck_launch(k, "spherical_forward_fused");
                n += k;
                auto rt = tiles_for(p, kRadFwd, nb, 2 * B, 0, B);
                k = staged(p, 2, st, [&] {
                    return sglk::launch_radial_forward(g, sglk::RadialBlocks{2 * B, 0, 0}, w.S.p, C, p->d_W, p->d_W_off,
                                                       rt.first, rt.second, st);
                });
                ck_launch(k, "radial_forward");
                return n + k;
            }
        }
    }
    if (nb == 1) {
        // shell slices: az + Legendre per slice into the full S, then radial once
        const int SC = sl.shells;
        sglk::Geo gc{B, SC, 1, 2LL * SC};
        w.G.ensure(2 * (size_t)sglk::g_layout(gc));
        const sglk::SView sv{2LL * 2 * B, 2 * B, 0};
        auto lt = tiles_for(p, kLegFwd, 1, SC, 0, 2 * B, false, 0, 0, true);
        if (const int ns = sl.count == 1 && !p->profiling ? pipe_slices(B, nb) : 0) {
            w.ensure_pipe();
            sglk::g_layout(gc);
            const int gper = (int)(gc.ngx / ns);       // shell groups per slice
            const int nper = (int)(gc.NB / 128 / ns);  // 128-column n-blocks per sign half and slice
            if (gper > 0 && nper > 0 && (long long)gper * ns == gc.ngx && (long long)nper * ns * 128 == gc.NB) {
                ck(cudaEventRecord(w.pev[8], st), "cudaEventRecord");
                ck(cudaStreamWaitEvent(w.st2, w.pev[8], 0), "cudaStreamWaitEvent");
                for (int c = 0; c < ns; ++c) {
                    sglk::Geo ga = gc;
                    ga.gx0 = c * gper;
                    ga.gxn = gper;
                    ck_launch(sglk::launch_az_forward(ga, X, psi2, w.G.p, p->d_bcal, p->d_tw, w.st2), "az_forward");
                    ck(cudaEventRecord(w.pev[c], w.st2), "cudaEventRecord");
                    ck(cudaStreamWaitEvent(st, w.pev[c], 0), "cudaStreamWaitEvent");
                    auto ltc = tiles_for(p, kLegFwd, 1, SC, 0, 2 * B, false, c * nper, nper);
                    ck_launch(sglk::launch_legendre_forward(gc, sv, w.G.p, w.S.p, p->d_leg, p->d_leg_off, ltc.first,
                                                            ltc.second, st),
                              "legendre_forward");
                    n += 2;
                }
                sglk::Geo g{B, 2 * B, 1, 2LL * 2 * B};
                auto rt = tiles_for(p, kRadFwd, 1, 2 * B, 0, B);
                k = sglk::launch_radial_forward(g, sglk::RadialBlocks{2 * B, 0, 0}, w.S.p, C, p->d_W, p->d_W_off, rt.first,
                                                rt.second, st);
                ck_launch(k, "radial_forward");
                return n + k;
            }
        }
        for (int c = 0; c < sl.count; ++c) {
            const int i0 = c * SC;
            k = staged(p, 0, st, [&] {
                return sglk::launch_az_forward(gc, X + (size_t)i0 * 2 * 4 * B * B, psi2, w.G.p, p->d_bcal, p->d_tw, st);
            });
            ck_launch(k, "az_forward");
            n += k;
            sglk::SView v = sv;
            v.i0 = i0;
            k = staged(p, 1, st, [&] {
                return sglk::launch_legendre_forward(gc, v, w.G.p, w.S.p, p->d_leg, p->d_leg_off, lt.first, lt.second, st);
            });
            ck_launch(k, "legendre_forward");
            n += k;
        }
        sglk::Geo g{B, 2 * B, 1, 2LL * 2 * B};
        auto rt = tiles_for(p, kRadFwd, 1, 2 * B, 0, B);
        k = staged(p, 2, st, [&] {
            return sglk::launch_radial_forward(g, sglk::RadialBlocks{2 * B, 0, 0}, w.S.p, C, p->d_W, p->d_W_off,
                                               rt.first, rt.second, st);
        });
        ck_launch(k, "radial_forward");
        return n + k;
    }
    // function slices: the whole forward per slice (G and S slices stay in L2)
    for (int f0 = 0; f0 < nb; f0 += sl.functions) {
        const int fb = std::min(sl.functions, nb - f0);
        sglk::Geo g{B, 2 * B, fb, 2LL * fb * 2 * B};
        g.az2x = az2x_on(B, fb);
        w.G.ensure(2 * (size_t)sglk::g_layout(g));
        const sglk::SView sv{g.NB, 2 * B, 0};
        auto lt = tiles_for(p, kLegFwd, fb, 2 * B, 0, 2 * B, false, 0, 0, true);
        auto rt = tiles_for(p, kRadFwd, fb, 2 * B, 0, B, false, 0, 0, true);
        k = staged(p, 0, st, [&] {
            return sglk::launch_az_forward(g, X + (size_t)f0 * psi2, psi2, w.G.p, p->d_bcal, p->d_tw, st);
        });
        ck_launch(k, "az_forward");
        n += k;
        k = staged(p, 1, st, [&] {
            return sglk::launch_legendre_forward(g, sv, w.G.p, w.S.p, p->d_leg, p->d_leg_off, lt.first, lt.second, st);
        });
        ck_launch(k, "legendre_forward");
        n += k;
        k = staged(p, 2, st, [&] {
            return sglk::launch_radial_forward(g, sglk::RadialBlocks{2 * B, 0, 0}, w.S.p, C + (size_t)f0 * om2,
                                               p->d_W, p->d_W_off, rt.first, rt.second, st);
        });
        ck_launch(k, "radial_forward");
        n += k;
    }
    return n;
}

int inverse_device(sglgpu_plan* p, Work& w, const double* C, double* X, int nb, cudaStream_t st) {
    const int B = p->B;
    const size_t psi2 = 2 * (size_t)sample_count(B), om2 = 2 * (size_t)coefficient_count(B);
    if (small_on(B, nb)) {
        const int k = staged(p, 7, st, [&] {
            return sglk::launch_small_inverse(B, nb, C, (long long)om2 / 2, X, (long long)psi2 / 2, p->d_leg, p->d_V,
                                              p->d_tw, st);
        });
        ck_launch(k, "small_inverse");
        return k;
    }
    const Slices sl = plan_slices(B, nb);
    w.S.ensure((size_t)4 * B * B * B * nb);
    int n = 0, k;
    if (nb == 1) {
        sglk::Geo g{B, 2 * B, 1, 2LL * 2 * B};
        auto rt = tiles_for(p, kRadInv, 1, 2 * B, 0, B);
        k = staged(p, 3, st, [&] {
            return sglk::launch_radial_inverse(g, sglk::RadialBlocks{2 * B, 0, 0}, C, w.S.p, p->d_V, p->d_V_off,
                                               rt.first, rt.second, st);
        });
        ck_launch(k, "radial_inverse");
        n += k;
        const int SC = sl.shells;
        sglk::Geo gc{B, SC, 1, 2LL * SC};
        w.G.ensure(2 * (size_t)sglk::g_layout(gc));
        auto lt = tiles_for(p, kLegInv, 1, SC, 0, 2 * B);
        if (const int ns = sl.count == 1 && !p->profiling && !i8_on("ws") && !i8_on("leginv") ? pipe_slices(B, nb) : 0) {
            w.ensure_pipe();
            const int rb = B / 32 / ns;  // 32-node row blocks of the Legendre inverse per slab
            const sglk::SView v{2LL * 2 * B, 2 * B, 0};
            for (int c = 0; c < ns; ++c) {
                auto ltc = tiles_for(p, kLegInv, 1, SC, 0, 2 * B, false, c * rb, rb);
                ck_launch(leginv(p, w, gc, v, w.S.p, w.G.p, ltc, st), "legendre_inverse");
                ck(cudaEventRecord(w.pev[c], st), "cudaEventRecord");
                ck(cudaStreamWaitEvent(w.st2, w.pev[c], 0), "cudaStreamWaitEvent");
                sglk::Geo ga = gc;
                ga.jp0 = c * rb * 32;
                ga.jpn = rb * 32;
                ck_launch(sglk::launch_az_inverse(ga, w.G.p, X, psi2, p->d_tw, w.st2), "az_inverse");
                n += 2;
            }
            ck(cudaEventRecord(w.pev[9], w.st2), "cudaEventRecord");
            ck(cudaStreamWaitEvent(st, w.pev[9], 0), "cudaStreamWaitEvent");
            return n;
        }
        for (int c = 0; c < sl.count; ++c) {
            const int i0 = c * SC;
            const sglk::SView v{2LL * 2 * B, 2 * B, i0};
            k = staged(p, 4, st, [&] {
                return leginv(p, w, gc, v, w.S.p, w.G.p, lt, st);
            });
            ck_launch(k, "legendre_inverse");
            n += k;
            k = staged(p, 5, st, [&] {
                return sglk::launch_az_inverse(gc, w.G.p, X + (size_t)i0 * 2 * 4 * B * B, psi2, p->d_tw, st);
            });
            ck_launch(k, "az_inverse");
            n += k;
        }
        return n;
    }
    for (int f0 = 0; f0 < nb; f0 += sl.functions) {
        const int fb = std::min(sl.functions, nb - f0);
        sglk::Geo g{B, 2 * B, fb, 2LL * fb * 2 * B};
        g.az2x = az2x_on(B, fb);
        w.G.ensure(2 * (size_t)sglk::g_layout(g));
        const sglk::SView sv{g.NB, 2 * B, 0};
        auto rt = tiles_for(p, kRadInv, fb, 2 * B, 0, B);
        auto lt = tiles_for(p, kLegInv, fb, 2 * B, 0, 2 * B);
        k = staged(p, 3, st, [&] {
            return sglk::launch_radial_inverse(g, sglk::RadialBlocks{2 * B, 0, 0}, C + (size_t)f0 * om2, w.S.p,
                                               p->d_V, p->d_V_off, rt.first, rt.second, st);
        });
        ck_launch(k, "radial_inverse");
        n += k;
        k = staged(p, 4, st, [&] {
            return leginv(p, w, g, sv, w.S.p, w.G.p, lt, st);
        });
        ck_launch(k, "legendre_inverse");
        n += k;
        k = staged(p, 5, st, [&] {
            return sglk::launch_az_inverse(g, w.G.p, X + (size_t)f0 * psi2, psi2, p->d_tw, st);
        });
        ck_launch(k, "az_inverse");
        n += k;
    }
    return n;
}

void check_plan(const sglgpu_plan* p) {
    if (!p) fail(SGLGPU_EINVAL, "sglgpu: null plan");
}

// Real-valued fast path (samples real, coefficients Hermitian in m): same three
// stages with only m >= 0 computed; the radial epilogue writes m < 0 by symmetry.
int real_device(sglgpu_plan* p, Work& w, const double* in, double* out, int nb, cudaStream_t st, bool forward) {
    const int B = p->B;
    const size_t psi = (size_t)sample_count(B), om2 = 2 * (size_t)coefficient_count(B);
    const Slices sl = plan_slices(B, nb);
    w.S.ensure((size_t)4 * B * B * B * nb);
    int n = 0, k;
    for (int f0 = 0; f0 < nb; f0 += sl.functions) {
        const int fb = std::min(sl.functions, nb - f0);
        sglk::Geo g{B, 2 * B, fb, 2LL * fb * 2 * B, 1};
        w.G.ensure(2 * (size_t)sglk::g_layout(g));
        const sglk::SView sv{g.NB, 2 * B, 0};
        if (forward) {
            auto lt = tiles_for(p, kLegFwd, fb, 2 * B, 0, 2 * B, true, 0, 0, true);
            auto rt = tiles_for(p, kRadFwd, fb, 2 * B, 0, B, true, 0, 0, true);
            k = staged(p, 0, st, [&] {
                return sglk::launch_az_forward_real(g, in + (size_t)f0 * psi, psi, w.G.p, p->d_bcal, p->d_tw, st);
            });
            if (k == -2) fail(SGLGPU_EINVAL, "sglgpu real path: 2B must be a power of two >= 4");
            ck_launch(k, "az_forward_real");
            n += k;
            k = staged(p, 1, st, [&] {
                return sglk::launch_legendre_forward(g, sv, w.G.p, w.S.p, p->d_leg, p->d_leg_off, lt.first, lt.second, st);
            });
            ck_launch(k, "legendre_forward");
            n += k;
            k = staged(p, 2, st, [&] {
                return sglk::launch_radial_forward(g, sglk::RadialBlocks{2 * B, 0, 0}, w.S.p, out + (size_t)f0 * om2,
                                                   p->d_W, p->d_W_off, rt.first, rt.second, st);
            });
            ck_launch(k, "radial_forward");
            n += k;
        } else {
            auto rt = tiles_for(p, kRadInv, fb, 2 * B, 0, B, true);
            auto lt = tiles_for(p, kLegInv, fb, 2 * B, 0, 2 * B, true);
            k = staged(p, 3, st, [&] {
                return sglk::launch_radial_inverse(g, sglk::RadialBlocks{2 * B, 0, 0}, in + (size_t)f0 * om2, w.S.p,
                                                   p->d_V, p->d_V_off, rt.first, rt.second, st);
            });
            ck_launch(k, "radial_inverse");
            n += k;
            k = staged(p, 4, st, [&] {
                return leginv(p, w, g, sv, w.S.p, w.G.p, lt, st);
            });
            ck_launch(k, "legendre_inverse");
            n += k;
            k = staged(p, 5, st, [&] {
                return sglk::launch_az_inverse_real(g, w.G.p, out + (size_t)f0 * psi, psi, p->d_tw, st);
            });
            if (k == -2) fail(SGLGPU_EINVAL, "sglgpu real path: 2B must be a power of two >= 4");
            ck_launch(k, "az_inverse_real");
            n += k;
        }
    }
    return n;
}

// ------------------------------------------------------------------ host-memory calls
// Acquires a free host slot of the plan (creating up to kHostSlots), waiting if
// all are busy; released by the guard's destructor.
struct SlotGuard {
    sglgpu_plan* p;
    HostSlot* s;
    explicit SlotGuard(sglgpu_plan* plan) : p(plan), s(nullptr) {
        std::unique_lock<std::mutex> lock(p->mu);
        for (;;) {
            for (auto& sl : p->slots)
                if (!sl->busy) {
                    s = sl.get();
                    break;
                }
            if (!s && (int)p->slots.size() < kHostSlots) {
                p->slots.push_back(std::make_unique<HostSlot>());
                s = p->slots.back().get();
            }
            if (s) break;
            p->slot_cv.wait(lock);
        }
        s->busy = true;
    }
    ~SlotGuard() {
        {
            std::lock_guard<std::mutex> lock(p->mu);
            s->busy = false;
        }
        p->slot_cv.notify_one();
    }
};

void slot_init(HostSlot& s) {
    if (s.sh) return;
    for (cudaStream_t* q : {&s.sh, &s.sc, &s.sd}) ck(cudaStreamCreateWithFlags(q, cudaStreamNonBlocking), "stream");
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t* e : {&s.eh[b], &s.ec[b], &s.ed[b], &s.es[b]})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
}

bool is_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// memcpy with a few host threads (pageable <-> pinned staging).
void par_memcpy(void* dst, const void* src, size_t bytes) {
    static const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
    if (bytes < (4u << 20) || nt == 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = (bytes / nt + 4095) & ~(size_t)4095;
    std::vector<std::thread> ts;
    for (unsigned t = 1; t < nt && t * per < bytes; ++t)
        ts.emplace_back([=] {
            const size_t o = t * per;
            std::memcpy((char*)dst + o, (const char*)src + o, std::min(per, bytes - o));
        });
    std::memcpy(dst, src, std::min(per, bytes));
    for (auto& t : ts) t.join();
}

constexpr size_t kStagePiece = (size_t)4 << 20;  // doubles per pinned staging piece (32 MiB)

void ensure_staging(HostSlot& s) {
    if (s.hst_cap) return;
    for (int b = 0; b < 2; ++b) ck(cudaMallocHost(&s.hst[b], kStagePiece * sizeof(double)), "cudaMallocHost(staging)");
    s.hst_cap = kStagePiece;
}

// H2D of n doubles on stream q: direct from pinned memory, else through the
// pinned staging pieces (the host copy of piece k+1 overlaps the DMA of piece k).
void upload(HostSlot& s, double* dst, const double* src, size_t n, bool pinned, cudaStream_t q) {
    if (pinned) {
        ck(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, q), "H2D");
        return;
    }
    ensure_staging(s);
    int k = 0;
    for (size_t o = 0; o < n; o += kStagePiece, ++k) {
        const size_t m = std::min(kStagePiece, n - o);
        const int b = k & 1;
        if (k >= 2) ck(cudaEventSynchronize(s.es[b]), "staging");  // the DMA of piece k-2 has left hst[b]
        par_memcpy(s.hst[b], src + o, m * sizeof(double));
        ck(cudaMemcpyAsync(dst + o, s.hst[b], m * sizeof(double), cudaMemcpyHostToDevice, q), "H2D");
        ck(cudaEventRecord(s.es[b], q), "event");
    }
}

// D2H of n doubles on stream q (after what q already waits for); pinned: async,
// else through the staging pieces (DMA of piece k+1 overlaps the host copy of k)
// and synchronous.
void download(HostSlot& s, double* dst, const double* src, size_t n, bool pinned, cudaStream_t q) {
    if (pinned) {
        ck(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, q), "D2H");
        return;
    }
    ensure_staging(s);
    const size_t pieces = (n + kStagePiece - 1) / kStagePiece;
    auto issue = [&](size_t k) {
        const size_t o = k * kStagePiece, m = std::min(kStagePiece, n - o);
        ck(cudaMemcpyAsync(s.hst[k & 1], src + o, m * sizeof(double), cudaMemcpyDeviceToHost, q), "D2H");
        ck(cudaEventRecord(s.es[k & 1], q), "event");
    };
    if (pieces) issue(0);
    for (size_t k = 0; k < pieces; ++k) {
        if (k + 1 < pieces) issue(k + 1);  // hst[(k+1)&1] was emptied by the host copy of piece k-1
        ck(cudaEventSynchronize(s.es[k & 1]), "D2H");
        const size_t o = k * kStagePiece, m = std::min(kStagePiece, n - o);
        par_memcpy(dst + o, s.hst[k & 1], m * sizeof(double));
    }
}

// A host-memory transform of `batch` functions through one slot: chunks of
// `chunk` functions, H2D (stream sh) -> compute (sc) -> D2H (sd), double-buffered
// so that consecutive chunks overlap.  compute(work, d_in, d_out, nb, stream)
// enqueues the kernels and returns their count.  Returns after the result is in
// host memory.
template <class Compute>
int host_pipeline(sglgpu_plan* p, const double* in, double* out, size_t batch, size_t in_len, size_t out_len,
                  size_t chunk, void* user_stream, Compute&& compute) {
    SlotGuard guard(p);
    HostSlot& s = *guard.s;
    set_device(p);
    slot_init(s);
    if (user_stream) {  // order after the caller's earlier work on its stream
        ck(cudaEventRecord(s.ed[0], static_cast<cudaStream_t>(user_stream)), "event");
        ck(cudaStreamWaitEvent(s.sh, s.ed[0], 0), "wait");
    }
    const bool pin_in = is_pinned(in), pin_out = is_pinned(out);
    const size_t nchunks = (batch + chunk - 1) / chunk;
    const size_t cap_in = in_len * std::min(chunk, batch), cap_out = out_len * std::min(chunk, batch);
    const int nbuf = nchunks > 1 ? 2 : 1;
    for (int b = 0; b < nbuf; ++b) {
        s.din[b].ensure(cap_in);
        s.dout[b].ensure(cap_out);
    }
    int launches = 0;
    auto h2d = [&](size_t c) {
        const int b = (int)(c & 1);
        const size_t b0 = c * chunk, nb = std::min(chunk, batch - b0);
        if (c >= 2) ck(cudaStreamWaitEvent(s.sh, s.ec[b], 0), "wait");  // din[b] consumed by chunk c-2
        upload(s, s.din[b].p, in + b0 * in_len, nb * in_len, pin_in, s.sh);
        ck(cudaEventRecord(s.eh[b], s.sh), "event");
    };
    h2d(0);
    for (size_t c = 0; c < nchunks; ++c) {
        const int b = (int)(c & 1);
        const size_t b0 = c * chunk, nb = std::min(chunk, batch - b0);
        ck(cudaStreamWaitEvent(s.sc, s.eh[b], 0), "wait");
        if (c >= 2) ck(cudaStreamWaitEvent(s.sc, s.ed[b], 0), "wait");  // dout[b] drained by chunk c-2
        launches += compute(s.w, s.din[b].p, s.dout[b].p, (int)nb, s.sc);
        ck(cudaEventRecord(s.ec[b], s.sc), "event");
        if (c + 1 < nchunks) h2d(c + 1);
        ck(cudaStreamWaitEvent(s.sd, s.ec[b], 0), "wait");
        download(s, out + b0 * out_len, s.dout[b].p, nb * out_len, pin_out, s.sd);
        ck(cudaEventRecord(s.ed[b], s.sd), "event");
    }
    ck(cudaStreamSynchronize(s.sd), "cudaStreamSynchronize");
    return launches;
}

// Functions per pipelined chunk of a host call: about four chunks per call (so
// transfers overlap compute), at least ~64 MB of samples per chunk, within the
// workspace budget (batch_chunk).
size_t host_chunk(int B, size_t batch) {
    const size_t cap = batch_chunk(B, batch);
    const size_t min_fn = std::max<size_t>(1, ((size_t)64 << 20) / ((size_t)128 * B * B * B));
    return std::max<size_t>(1, std::min(cap, std::max(min_fn, (batch + 3) / 4)));
}

int run_real(sglgpu_plan* p, const double* in, double* out, size_t batch, int mem_kind, void* stream, bool forward) {
    return guarded([&] {
        check_plan(p);
        if (mem_kind != SGLGPU_MEM_HOST && mem_kind != SGLGPU_MEM_DEVICE)
            fail(SGLGPU_EINVAL, "sglgpu: unknown mem_kind");
        if (batch == 0) return;
        if (!in || !out) fail(SGLGPU_EINVAL, "sglgpu: null data pointer");
        const int B = p->B;
        if (B < 2 || ((2 * B) & (2 * B - 1)) != 0)
            fail(SGLGPU_EINVAL, "sglgpu real path: 2B must be a power of two >= 4");
        const size_t psi = (size_t)sample_count(B), om = 2 * (size_t)coefficient_count(B);
        const size_t in_len = forward ? psi : om, out_len = forward ? om : psi;
        int launches = 0;
        if (mem_kind == SGLGPU_MEM_DEVICE) {
            std::lock_guard<std::mutex> lock(p->mu);
            set_device(p);
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            const size_t chunk = batch_chunk(B, batch);
            for (size_t b0 = 0; b0 < batch; b0 += chunk) {
                const int nb = (int)std::min(chunk, batch - b0);
                launches += real_device(p, p->main, in + b0 * in_len, out + b0 * out_len, nb, st, forward);
            }
        } else {
            launches = host_pipeline(p, in, out, batch, in_len, out_len, host_chunk(B, batch), stream,
                                     [&](Work& w, const double* di, double* dout, int nb, cudaStream_t q) {
                                         return real_device(p, w, di, dout, nb, q, forward);
                                     });
        }
        p->last_launches = launches;
    });
}

// dsglft_separated / idsglft_separated (sgl_transform.cpp:189-272) on the device:
// the cross-oracle rung of SURVEY.md 8(f).  Synchronous w.r.t. host memory.
// naive = true: the O(B^7) naive rung (sgl_transform.cpp:122-187), B <= 32.
int run_separated(sglgpu_plan* p, const double* in, double* out, size_t batch, int mem_kind, void* stream,
                  bool forward, bool naive = false) {
    return guarded([&] {
        check_plan(p);
        if (mem_kind != SGLGPU_MEM_HOST && mem_kind != SGLGPU_MEM_DEVICE)
            fail(SGLGPU_EINVAL, "sglgpu: unknown mem_kind");
        if (batch == 0) return;
        if (!in || !out) fail(SGLGPU_EINVAL, "sglgpu: null data pointer");
        const int B = p->B;
        if (!naive && B > 64)
            fail(SGLGPU_EINVAL, "sglgpu separated transform: bandlimit must be <= 64 (reference validity)");
        if (naive && B > 32) fail(SGLGPU_EINVAL, "sglgpu naive transform: bandlimit must be <= 32 (O(B^7))");
        const size_t psi = 2 * (size_t)sample_count(B), om = 2 * (size_t)coefficient_count(B);
        const size_t in_len = forward ? psi : om, out_len = forward ? om : psi;
        const size_t chunk = std::max<size_t>(1, std::min<size_t>(batch, 64));
        auto compute = [&](Work& w, const double* src, double* dst, int nb, cudaStream_t st) {
            w.S.ensure((size_t)4 * B * B * B * nb);
            const int k = naive ? (forward ? sglk::launch_naive_forward(B, nb, src, dst, p->d_r, p->d_amod,
                                                                        p->d_bcal, st)
                                           : sglk::launch_naive_inverse(B, nb, src, dst, p->d_r, st))
                        : forward ? sglk::launch_separated_forward(B, nb, src, dst, w.S.p, p->d_r, p->d_amod,
                                                                   p->d_bcal, st)
                                  : sglk::launch_separated_inverse(B, nb, src, dst, w.S.p, p->d_r, st);
            ck_launch(k, naive ? "naive transform" : forward ? "separated_forward" : "separated_inverse");
            return k;
        };
        int launches = 0;
        if (mem_kind == SGLGPU_MEM_HOST) {
            launches = host_pipeline(p, in, out, batch, in_len, out_len, chunk, stream, compute);
        } else {
            std::lock_guard<std::mutex> lock(p->mu);
            set_device(p);
            for (size_t b0 = 0; b0 < batch; b0 += chunk) {
                const int nb = (int)std::min(chunk, batch - b0);
                launches += compute(p->main, in + b0 * in_len, out + b0 * out_len, nb, static_cast<cudaStream_t>(stream));
            }
        }
        p->last_launches = launches;
    });
}

int run(sglgpu_plan* p, const double* in, double* out, size_t batch, int mem_kind, void* stream,
        bool forward) {
    return guarded([&] {
        check_plan(p);
        if (mem_kind != SGLGPU_MEM_HOST && mem_kind != SGLGPU_MEM_DEVICE)
            fail(SGLGPU_EINVAL, "sglgpu: unknown mem_kind");
        if (batch == 0) return;
        if (!in || !out) fail(SGLGPU_EINVAL, "sglgpu: null data pointer");
        const int B = p->B;
        if (mem_kind == SGLGPU_MEM_HOST) {
            const size_t psi = 2 * (size_t)sample_count(B), om = 2 * (size_t)coefficient_count(B);
            p->last_launches = host_pipeline(
                p, in, out, batch, forward ? psi : om, forward ? om : psi, host_chunk(B, batch), stream,
                [&](Work& w, const double* di, double* dout, int nb, cudaStream_t q) {
                    return forward ? forward_device(p, w, di, dout, nb, q) : inverse_device(p, w, di, dout, nb, q);
                });
            return;
        }
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t psi = 2 * (size_t)sample_count(B), om = 2 * (size_t)coefficient_count(B);
        const size_t in_len = forward ? psi : om, out_len = forward ? om : psi;
        const size_t chunk = batch_chunk(B, batch);
        int launches = 0;
        auto body = [&]() {
            int n = 0;
            for (size_t b0 = 0; b0 < batch; b0 += chunk) {
                const int nb = (int)std::min(chunk, batch - b0);
                n += forward ? forward_device(p, p->main, in + b0 * in_len, out + b0 * out_len, nb, st)
                             : inverse_device(p, p->main, in + b0 * in_len, out + b0 * out_len, nb, st);
            }
            return n;
        };
        if (mem_kind == SGLGPU_MEM_DEVICE) {
            // Small transforms are launch-bound: from the second call with the same
            // (direction, batch, pointers, stream) the kernel sequence is captured
            // once into a CUDA graph and replayed with a single launch.  Not while
            // profiling (per-stage events) and only for streams other than the
            // legacy default stream.
            const auto key = std::make_tuple(forward ? 1 : 0, batch, (const void*)in, (void*)out, (void*)st,
                                             (void*)p->main.G.p, (void*)p->main.S.p);
            auto git = p->graphs.find(key);
            if (git != p->graphs.end() && !p->profiling) {
                ck(cudaGraphLaunch(git->second.exec, st), "cudaGraphLaunch");
                git->second.last_use = ++p->tick;
                launches = git->second.launches;
            } else if (use_graphs(B, batch) && !p->profiling && st != nullptr && seen_twice(p, key)) {
                if (p->graphs.size() >= 128) {  // evict the least recently used graph
                    auto lru = p->graphs.begin();
                    for (auto it = p->graphs.begin(); it != p->graphs.end(); ++it)
                        if (it->second.last_use < lru->second.last_use) lru = it;
                    cudaGraphExecDestroy(lru->second.exec);
                    p->graphs.erase(lru);
                }
                cudaGraph_t graph = nullptr;
                ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
                try {
                    launches = body();
                } catch (...) {
                    cudaStreamEndCapture(st, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                ck(cudaStreamEndCapture(st, &graph), "cudaStreamEndCapture");
                sglgpu_plan::GraphEntry e;
                const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
                cudaGraphDestroy(graph);
                ck(ie, "cudaGraphInstantiate");
                e.launches = launches;
                e.last_use = ++p->tick;
                ck(cudaGraphLaunch(e.exec, st), "cudaGraphLaunch");
                p->graphs[key] = e;
            } else {
                launches = body();
            }
        }
        p->last_launches = launches;
    });
}

}  // namespace

extern "C" {

const char* sglgpu_last_error(void) { return g_last_error.c_str(); }

int sglgpu_plan_create(const sglgpu_plan_desc* desc, sglgpu_plan** out) {
    return guarded([&] {
        if (!desc || !out) fail(SGLGPU_EINVAL, "sglgpu_plan_create: null argument");
        *out = nullptr;
        const int B = desc->bandlimit;
        if (B < 1 || B > 256) fail(SGLGPU_EINVAL, "sglgpu_plan_create: bandlimit must be in [1, 256]");
        if (!desc->r || !desc->a_mod) fail(SGLGPU_EINVAL, "sglgpu_plan_create: radial rule required");
        for (int i = 0; i < 2 * B; ++i) {
            if (!(desc->r[i] > 0.0) || (i > 0 && !(desc->r[i] > desc->r[i - 1])))
                fail(SGLGPU_EINVAL, "sglgpu_plan_create: radial nodes must be positive and increasing");
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            fail(SGLGPU_ENODEV, "sglgpu_plan_create: no CUDA device");
        }
        int dev = desc->device;
        if (dev < 0) ck(cudaGetDevice(&dev), "cudaGetDevice");
        if (dev >= ndev) fail(SGLGPU_EINVAL, "sglgpu_plan_create: device ordinal out of range");
        std::vector<double> bcal = desc->b_cal ? std::vector<double>(desc->b_cal, desc->b_cal + 2 * B)
                                               : sglhost::sphere_bcal(B);
        const sglhost::Tables t = sglhost::build_tables(B, desc->r, desc->a_mod, bcal.data());
        auto* p = new sglgpu_plan;
        p->B = B;
        p->device = dev;
        cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
        try {
            set_device(p);
            p->d_tw = dev_upload(t.twiddle);
            p->d_bcal = dev_upload(t.bcal);
            p->d_leg = dev_upload(t.legendre);
            p->d_leg_off = dev_upload(t.legendre_off);
            p->d_W = dev_upload(t.radial_fwd);
            p->d_W_off = dev_upload(t.radial_fwd_off);
            p->d_V = dev_upload(t.radial_inv);
            p->d_V_off = dev_upload(t.radial_inv_off);
            p->d_r = dev_upload(std::vector<double>(desc->r, desc->r + 2 * B));
            p->d_amod = dev_upload(std::vector<double>(desc->a_mod, desc->a_mod + 2 * B));
            p->leg_count = t.legendre.size();
        } catch (...) {
            sglgpu_plan_destroy(p);
            throw;
        }
        p->table_bytes = sizeof(double) * (t.twiddle.size() + t.bcal.size() + t.legendre.size() +
                                           t.radial_fwd.size() + t.radial_inv.size()) +
                         sizeof(long long) * (t.legendre_off.size() + t.radial_fwd_off.size() +
                                              t.radial_inv_off.size());
        *out = p;
    });
}

int sglgpu_plan_destroy(sglgpu_plan* p) {
    if (!p) return SGLGPU_OK;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    for (void* q : {(void*)p->d_tw, (void*)p->d_bcal, (void*)p->d_leg, (void*)p->d_leg_off, (void*)p->d_W,
                    (void*)p->d_W_off, (void*)p->d_V, (void*)p->d_V_off, (void*)p->d_r, (void*)p->d_amod,
                    (void*)p->oz_li.img, (void*)p->oz_li.off, (void*)p->oz_li.rexp, (void*)p->oz_li.kpad, (void*)p->oz_li.corr})
        if (q) cudaFree(q);
    for (auto& kv : p->oz_units) cudaFree(kv.second.first);
    for (auto& kv : p->tiles) delete kv.second.first;
    for (auto& [stage, a, b] : p->prof) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    for (auto e : p->ev_pool) cudaEventDestroy(e);
    for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second.exec);
    p->main.release();
    for (auto& sl : p->slots) sl->release();
    delete p;
    return SGLGPU_OK;
}

int sglgpu_plan_bandlimit(const sglgpu_plan* p) { return p ? p->B : 0; }

size_t sglgpu_plan_table_bytes(const sglgpu_plan* p) { return p ? p->table_bytes : 0; }

int sglgpu_last_launch_count(const sglgpu_plan* p) { return p ? p->last_launches.load() : 0; }

int sglgpu_profile_begin(sglgpu_plan* p) {
    return guarded([&] {
        check_plan(p);
        std::lock_guard<std::mutex> lock(p->mu);
        p->profiling = true;
    });
}

int sglgpu_profile_end(sglgpu_plan* p, double* stage_ms, int* stage_launches) {
    return guarded([&] {
        check_plan(p);
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        p->profiling = false;
        for (int s = 0; s < SGLGPU_NUM_STAGES; ++s) {
            if (stage_ms) stage_ms[s] = 0.0;
            if (stage_launches) stage_launches[s] = 0;
        }
        for (auto& [stage, a, b] : p->prof) {
            ck(cudaEventSynchronize(b), "cudaEventSynchronize");
            float ms = 0.f;
            ck(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
            if (stage_ms) stage_ms[stage] += ms;
            if (stage_launches) stage_launches[stage] += 1;
            p->ev_pool.push_back(a);
            p->ev_pool.push_back(b);
        }
        p->prof.clear();
    });
}

int sglgpu_forward(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch, int mem_kind,
                   void* stream) {
    return run(plan, samples, coeffs, batch, mem_kind, stream, true);
}

int sglgpu_inverse(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch, int mem_kind,
                   void* stream) {
    return run(plan, coeffs, samples, batch, mem_kind, stream, false);
}

int sglgpu_forward_separated(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch, int mem_kind,
                             void* stream) {
    return run_separated(plan, samples, coeffs, batch, mem_kind, stream, true);
}

int sglgpu_inverse_separated(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch, int mem_kind,
                             void* stream) {
    return run_separated(plan, coeffs, samples, batch, mem_kind, stream, false);
}

int sglgpu_forward_naive(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch, int mem_kind,
                         void* stream) {
    return run_separated(plan, samples, coeffs, batch, mem_kind, stream, true, true);
}

int sglgpu_inverse_naive(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch, int mem_kind,
                         void* stream) {
    return run_separated(plan, coeffs, samples, batch, mem_kind, stream, false, true);
}

int sglgpu_sample_basis(sglgpu_plan* p, int n, int l, int m, double* samples, int mem_kind, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        if (n < 1 || n > B || l < 0 || l >= n || m < -l || m > l)
            fail(SGLGPU_EINVAL, "sample_sgl_basis: invalid (n, l, m) for this plan");
        if (mem_kind != SGLGPU_MEM_HOST && mem_kind != SGLGPU_MEM_DEVICE)
            fail(SGLGPU_EINVAL, "sglgpu: unknown mem_kind");
        if (!samples) fail(SGLGPU_EINVAL, "sglgpu: null data pointer");
        const size_t len = 2 * (size_t)sample_count(B);
        if (mem_kind == SGLGPU_MEM_HOST) {
            SlotGuard guard(p);
            HostSlot& s = *guard.s;
            set_device(p);
            slot_init(s);
            s.dout[0].ensure(len);
            const int k = sglk::launch_sample_basis(B, n, l, m, s.dout[0].p, p->d_r, s.sc);
            ck_launch(k, "sample_basis");
            ck(cudaEventRecord(s.ec[0], s.sc), "event");
            ck(cudaStreamWaitEvent(s.sd, s.ec[0], 0), "wait");
            download(s, samples, s.dout[0].p, len, is_pinned(samples), s.sd);
            ck(cudaStreamSynchronize(s.sd), "cudaStreamSynchronize");
            p->last_launches = k;
            return;
        }
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        const int k = sglk::launch_sample_basis(B, n, l, m, samples, p->d_r, static_cast<cudaStream_t>(stream));
        ck_launch(k, "sample_basis");
        p->last_launches = k;
    });
}

int sglgpu_forward_real(sglgpu_plan* plan, const double* samples, double* coeffs, size_t batch, int mem_kind,
                        void* stream) {
    return run_real(plan, samples, coeffs, batch, mem_kind, stream, true);
}

int sglgpu_inverse_real(sglgpu_plan* plan, const double* coeffs, double* samples, size_t batch, int mem_kind,
                        void* stream) {
    return run_real(plan, coeffs, samples, batch, mem_kind, stream, false);
}

int sglgpu_spherical_forward(sglgpu_plan* p, const double* samples, size_t sample_stride, double* shells,
                             int shell_begin, int shell_count, size_t batch, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_spherical_forward");
        if (shell_begin < 0 || shell_count < 1 || shell_begin + shell_count > 2 * B)
            fail(SGLGPU_EINVAL, "sglgpu_spherical_forward: shell range out of bounds");
        if (batch == 0) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int nb = (int)batch;
        sglk::Geo g{B, shell_count, nb, 2LL * nb * shell_count};
        p->main.G.ensure(2 * (size_t)sglk::g_layout(g));
        int n = sglk::launch_az_forward(g, samples, 2 * sample_stride, p->main.G.p, p->d_bcal, p->d_tw, st);
        ck_launch(n, "az_forward");
        auto lt = tiles_for(p, kLegFwd, nb, shell_count, 0, 2 * B);
        const sglk::SView sv{g.NB, shell_count, 0};
        int k = sglk::launch_legendre_forward(g, sv, p->main.G.p, shells, p->d_leg, p->d_leg_off, lt.first, lt.second, st);
        ck_launch(k, "legendre_forward");
        p->last_launches = n + k;
    });
}

int sglgpu_spherical_inverse(sglgpu_plan* p, const double* shells, double* samples, size_t sample_stride,
                             int shell_begin, int shell_count, size_t batch, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_spherical_inverse");
        if (shell_begin < 0 || shell_count < 1 || shell_begin + shell_count > 2 * B)
            fail(SGLGPU_EINVAL, "sglgpu_spherical_inverse: shell range out of bounds");
        if (batch == 0) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int nb = (int)batch;
        sglk::Geo g{B, shell_count, nb, 2LL * nb * shell_count};
        p->main.G.ensure(2 * (size_t)sglk::g_layout(g));
        auto lt = tiles_for(p, kLegInv, nb, shell_count, 0, 2 * B);
        const sglk::SView sv{g.NB, shell_count, 0};
        int k = leginv(p, p->main, g, sv, shells, p->main.G.p, lt, st);
        ck_launch(k, "legendre_inverse");
        int n = sglk::launch_az_inverse(g, p->main.G.p, samples, 2 * sample_stride, p->d_tw, st);
        ck_launch(n, "az_inverse");
        p->last_launches = n + k;
    });
}

int sglgpu_radial_forward(sglgpu_plan* p, const double* shells, double* coeffs, int l_begin, int l_end,
                          int shells_per_block, size_t batch, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_radial_forward");
        if (l_begin < 0 || l_end > B || l_begin > l_end) fail(SGLGPU_EINVAL, "sglgpu_radial_forward: bad l range");
        if (shells_per_block < 1 || (2 * B) % shells_per_block != 0)
            fail(SGLGPU_EINVAL, "sglgpu_radial_forward: shells_per_block must divide 2B");
        if (batch == 0 || l_begin == l_end) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        const int nb = (int)batch, sc = shells_per_block;
        sglk::Geo g{B, sc, nb, 2LL * nb * sc};
        const long long nu0 = (long long)l_begin * l_begin, nnu = (long long)l_end * l_end - nu0;
        auto rt = tiles_for(p, kRadFwd, nb, sc, l_begin, l_end);
        int k = sglk::launch_radial_forward(g, sglk::RadialBlocks{sc, nnu * g.NB, nu0}, shells,
                                            coeffs, p->d_W, p->d_W_off, rt.first, rt.second,
                                            static_cast<cudaStream_t>(stream));
        ck_launch(k, "radial_forward");
        p->last_launches = k;
    });
}

int sglgpu_radial_inverse(sglgpu_plan* p, const double* coeffs, double* shells, int l_begin, int l_end,
                          int shells_per_block, size_t batch, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_radial_inverse");
        if (l_begin < 0 || l_end > B || l_begin > l_end) fail(SGLGPU_EINVAL, "sglgpu_radial_inverse: bad l range");
        if (shells_per_block < 1 || (2 * B) % shells_per_block != 0)
            fail(SGLGPU_EINVAL, "sglgpu_radial_inverse: shells_per_block must divide 2B");
        if (batch == 0 || l_begin == l_end) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        const int nb = (int)batch, sc = shells_per_block;
        sglk::Geo g{B, sc, nb, 2LL * nb * sc};
        const long long nu0 = (long long)l_begin * l_begin, nnu = (long long)l_end * l_end - nu0;
        auto rt = tiles_for(p, kRadInv, nb, sc, l_begin, l_end);
        int k = sglk::launch_radial_inverse(g, sglk::RadialBlocks{sc, nnu * g.NB, nu0}, coeffs,
                                            shells, p->d_V, p->d_V_off, rt.first, rt.second,
                                            static_cast<cudaStream_t>(stream));
        ck_launch(k, "radial_inverse");
        p->last_launches = k;
    });
}

// ---------------------------------------------------------------- fused exchange (NVLink peer stores)
int sglgpu_spherical_forward_to(sglgpu_plan* p, const double* samples, size_t sample_stride, int shell_begin,
                                int shell_count, size_t batch, int ndst, double* const* dst, const int* l_bounds,
                                void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_spherical_forward_to");
        if (shell_begin < 0 || shell_count < 1 || shell_begin + shell_count > 2 * B)
            fail(SGLGPU_EINVAL, "sglgpu_spherical_forward_to: shell range out of bounds");
        if (ndst < 1 || ndst > sglk::kMaxPeers || !dst || !l_bounds)
            fail(SGLGPU_EINVAL, "sglgpu_spherical_forward_to: 1..8 destinations with pointers and bounds required");
        if (l_bounds[0] != 0 || l_bounds[ndst] != B)
            fail(SGLGPU_EINVAL, "sglgpu_spherical_forward_to: degree bounds must span [0, B)");
        for (int q = 0; q < ndst; ++q)
            if (l_bounds[q + 1] < l_bounds[q]) fail(SGLGPU_EINVAL, "sglgpu_spherical_forward_to: bounds must increase");
        if (batch == 0) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int nb = (int)batch;
        sglk::Geo g{B, shell_count, nb, 2LL * nb * shell_count};
        p->main.G.ensure(2 * (size_t)sglk::g_layout(g));
        int n = sglk::launch_az_forward(g, samples, 2 * sample_stride, p->main.G.p, p->d_bcal, p->d_tw, st);
        ck_launch(n, "az_forward");
        sglk::PeerDest pd;
        pd.n = ndst;
        for (int q = 0; q < ndst; ++q) {
            pd.bound[q] = l_bounds[q];
            // rows nu of rank q's degrees land at dst[q] + (nu - nu0_q) * NB
            pd.base[q] = dst[q] - (long long)l_bounds[q] * l_bounds[q] * g.NB;
        }
        pd.bound[ndst] = l_bounds[ndst];
        auto lt = tiles_for(p, kLegFwd, nb, shell_count, 0, 2 * B);
        const sglk::SView sv{g.NB, shell_count, 0};
        int k = sglk::launch_legendre_forward_peers(g, sv, p->main.G.p, pd, p->d_leg, p->d_leg_off, lt.first, lt.second,
                                                    st);
        ck_launch(k, "legendre_forward");
        p->last_launches = n + k;
    });
}

int sglgpu_radial_forward_to(sglgpu_plan* p, const double* shells, int l_begin, int l_end, int shells_per_block,
                             size_t batch, int ndst, double* const* dst, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_radial_forward_to");
        if (l_begin < 0 || l_end > B || l_begin > l_end) fail(SGLGPU_EINVAL, "sglgpu_radial_forward_to: bad l range");
        if (shells_per_block < 1 || (2 * B) % shells_per_block != 0)
            fail(SGLGPU_EINVAL, "sglgpu_radial_forward_to: shells_per_block must divide 2B");
        if (ndst < 1 || ndst > sglk::kMaxPeers || !dst)
            fail(SGLGPU_EINVAL, "sglgpu_radial_forward_to: 1..8 destination coefficient vectors required");
        for (int q = 0; q < ndst; ++q)
            if (!dst[q]) fail(SGLGPU_EINVAL, "sglgpu_radial_forward_to: null destination");
        if (batch == 0 || l_begin == l_end) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        const int nb = (int)batch, sc = shells_per_block;
        sglk::Geo g{B, sc, nb, 2LL * nb * sc};
        const long long nu0 = (long long)l_begin * l_begin, nnu = (long long)l_end * l_end - nu0;
        sglk::PeerDest pd;
        pd.n = ndst;
        for (int q = 0; q < ndst; ++q) pd.base[q] = dst[q];
        auto rt = tiles_for(p, kRadFwd, nb, sc, l_begin, l_end);
        int k = sglk::launch_radial_forward_bcast(g, sglk::RadialBlocks{sc, nnu * g.NB, nu0}, shells, pd, p->d_W,
                                                  p->d_W_off, rt.first, rt.second, static_cast<cudaStream_t>(stream));
        ck_launch(k, "radial_forward");
        p->last_launches = k;
    });
}

int sglgpu_radial_inverse_to(sglgpu_plan* p, const double* coeffs, int l_begin, int l_end, int shells_per_block,
                             size_t batch, int ndst, double* const* dst, void* stream) {
    return guarded([&] {
        check_plan(p);
        const int B = p->B;
        check_stage_batch(B, batch, "sglgpu_radial_inverse_to");
        if (l_begin < 0 || l_end > B || l_begin > l_end) fail(SGLGPU_EINVAL, "sglgpu_radial_inverse_to: bad l range");
        if (shells_per_block < 1 || (2 * B) % shells_per_block != 0)
            fail(SGLGPU_EINVAL, "sglgpu_radial_inverse_to: shells_per_block must divide 2B");
        if (ndst != 2 * B / shells_per_block || ndst > sglk::kMaxPeers || !dst)
            fail(SGLGPU_EINVAL, "sglgpu_radial_inverse_to: one destination per shell block (at most 8) required");
        if (batch == 0 || l_begin == l_end) return;
        std::lock_guard<std::mutex> lock(p->mu);
        set_device(p);
        const int nb = (int)batch, sc = shells_per_block;
        sglk::Geo g{B, sc, nb, 2LL * nb * sc};
        const long long nu0 = (long long)l_begin * l_begin;
        sglk::PeerDest pd;
        pd.n = ndst;
        // rank b's S is [nu][f][i_local] over all nu; the kernel's column offset is relative to nu0
        for (int b = 0; b < ndst; ++b) pd.base[b] = dst[b] + nu0 * g.NB;
        auto rt = tiles_for(p, kRadInv, nb, sc, l_begin, l_end);
        int k = sglk::launch_radial_inverse_peers(g, sglk::RadialBlocks{sc, 0, nu0}, coeffs, pd, p->d_V, p->d_V_off,
                                                  rt.first, rt.second, static_cast<cudaStream_t>(stream));
        ck_launch(k, "radial_inverse");
        p->last_launches = k;
    });
}

// Device buffers that peers can map (CUDA IPC), for the fused exchange.
int sglgpu_device_alloc(size_t bytes, void** ptr) {
    return guarded([&] {
        if (!ptr) fail(SGLGPU_EINVAL, "sglgpu_device_alloc: null output");
        ck(cudaMalloc(ptr, std::max<size_t>(bytes, 16)), "cudaMalloc(peer buffer)");
    });
}

int sglgpu_device_free(void* ptr) {
    return guarded([&] { ck(cudaFree(ptr), "cudaFree(peer buffer)"); });
}

int sglgpu_ipc_export(void* ptr, void* handle64) {
    return guarded([&] {
        if (!ptr || !handle64) fail(SGLGPU_EINVAL, "sglgpu_ipc_export: null argument");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
        std::memcpy(handle64, &h, sizeof(h));
    });
}

int sglgpu_ipc_open(const void* handle64, void** ptr) {
    return guarded([&] {
        if (!ptr || !handle64) fail(SGLGPU_EINVAL, "sglgpu_ipc_open: null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        ck(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int sglgpu_ipc_close(void* ptr) {
    return guarded([&] { ck(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); });
}

}  // extern "C"
