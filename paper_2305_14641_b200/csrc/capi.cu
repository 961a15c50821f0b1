// C-ABI of libgqc (include/gqc.h): validation with the reference's error
// semantics, per-sigma constants from the host exp provider, device buffer
// cache, host<->device staging, and orchestration of the kernels in
// kernels.cu. No CPU compute path exists: without a CUDA device every compute
// entry point fails with GQC_ECUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gqc.h"
#include "gqc_internal.h"

namespace gqc {

namespace {

thread_local std::string t_err;
thread_local long long t_launches = 0;

// Options: process-wide, set by gqc_set_option; every call works on a
// snapshot taken when it starts (t_opt), so a concurrent set never changes a
// call halfway.
struct Options {
    int exp_mode = GQC_EXP_EIGEN;
    int kernel = GQC_KERNEL_FASTFWD;
    int device = 0;   // device of the host-buffer entry points (GQC_OPT_DEVICE)
    int hop_cap = 1;  // distance model (GQC_OPT_HOP_CAP): 1 = the reference's
    int gpus = 1;     // devices of the host-buffer sweep entry points (GQC_OPT_GPUS)
};
struct AtomicOptions {
    std::atomic<int> exp_mode{GQC_EXP_EIGEN}, kernel{GQC_KERNEL_FASTFWD}, device{0}, hop_cap{1}, gpus{1};
    Options load() const {
        Options o;
        o.exp_mode = exp_mode.load();
        o.kernel = kernel.load();
        o.device = device.load();
        o.hop_cap = hop_cap.load();
        o.gpus = gpus.load();
        return o;
    }
} g_opt;
thread_local Options t_opt;

// Locking: one mutex per device context instead of one per process. A call
// locks the context of every device it touches for its whole duration (a
// multi-device call locks its devices in ascending order), so calls on
// different devices, from different host threads, run concurrently.
thread_local std::vector<std::mutex*> t_held;

struct Fail {
    gqc_status st;
    std::string msg;
};

[[noreturn]] void fail(gqc_status st, const std::string& msg) { throw Fail{st, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) fail(GQC_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(GQC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void cuda_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

struct HeldLocks {  // releases the device locks a call took, in reverse order
    ~HeldLocks() {
        for (auto it = t_held.rbegin(); it != t_held.rend(); ++it) (*it)->unlock();
        t_held.clear();
    }
};

template <class F>
gqc_status guarded(F&& f) {
    t_launches = 0;
    t_opt = g_opt.load();
    HeldLocks release;
    try {
        f();
        return GQC_OK;
    } catch (const Fail& e) {
        t_err = e.msg;
        return e.st;
    } catch (const std::bad_alloc&) {
        t_err = "allocation failure";
        return GQC_ENOMEM;
    } catch (const std::exception& e) {
        t_err = e.what();
        return GQC_ECUDA;
    }
}

// Opt-in stage tracing (GQC_TRACE=1): CUDA events on the compute stream
// around each stage of a host-API call, printed to stderr when it returns.
struct Tracer {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    explicit Tracer(cudaStream_t s) : st(s) {
        const char* e = std::getenv("GQC_TRACE");
        on = e && *e && *e != '0';
        mark("begin");
    }
    void mark(const char* what) {
        if (!on) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        marks.emplace_back(what, ev);
    }
    ~Tracer() {
        if (!on) return;
        cudaStreamSynchronize(st);
        std::string line = "[gqc trace]";
        for (std::size_t k = 1; k < marks.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[k - 1].second, marks[k].second);
            line += " " + marks[k].first + "=" + std::to_string(ms) + "ms";
        }
        for (auto& m : marks) cudaEventDestroy(m.second);
        std::fprintf(stderr, "%s\n", line.c_str());
    }
};

// Grow-only device buffers, one set per device: repeated calls reuse memory.
struct DevBuf {
    void* p = nullptr;
    std::size_t cap = 0;
    template <class T>
    T* get(std::size_t count) {
        const std::size_t bytes = std::max<std::size_t>(count * sizeof(T), 256);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
};

// Scratch tables of a potential launch on weighted graphs (host-evaluated
// exp values the device reads): one set per context and per multi-device shard.
struct PotScratch {
    DevBuf tail, entry;
};

// Buffers and stream of one shard of a multi-device sweep (gqc_*_multi):
// its sigma chunk's node-major field (written by every shard's potential
// kernel over peer memory), the chunk's GGD outputs and a staging area for
// devices without peer access. Owned by the shard's device context.
struct ShardBufs {
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_pot = nullptr;
    DevBuf v, v_sm, succ, center, ci, nc, ws, intra, send, err;
    PotScratch scr;
    int* nc_host = nullptr;  // pinned counts staging
    int nc_host_cap = 0;
    int* err_host = nullptr;  // pinned: GGD cycle flag readback
};

struct DeviceCtx {
    std::mutex mu;  // held for the whole duration of a call on this device
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;   // host<->device copies overlapped with compute
    cudaStream_t slab[4] = {};     // concurrent per-slab potential launches
    cudaEvent_t ev[16] = {};
    cudaEvent_t slab_done[4] = {};
    cudaMemPool_t pool = nullptr;  // stream-ordered scratch that keeps its memory
    DevBuf off, nbr, w, v_nm, v_sm, succ, center, ci, nc, ws, intra, err;
    PotScratch scr;
    int* err_host = nullptr;  // pinned: GGD cycle flag readback
    int* nc_host = nullptr;  // pinned staging for per-sigma counts (cudaHostAlloc)
    int nc_host_cap = 0;
    DevBuf slab_sync;            // polled upload: [4] slab flags, [4] error word
    int* slab_host = nullptr;    // pinned: [0..3] = 1 (flag sources), [4] error readback
    std::vector<std::unique_ptr<ShardBufs>> shards;  // multi-device shards on this device
};

// Device->host copies into pageable memory block the calling thread until
// they complete, which would stall the launches queued behind them.
bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int* pinned_counts_buf(int*& buf, int& cap, int n) {
    if (cap < n) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&buf), sizeof(int) * n, cudaHostAllocDefault),
                   "cudaHostAlloc");
        cap = n;
    }
    return buf;
}
int* pinned_counts(DeviceCtx& C, int n) { return pinned_counts_buf(C.nc_host, C.nc_host_cap, n); }

// Device word the bounded chase sets when a successor map has a cycle
// (launch_labels), cleared on `st`; its pinned readback slot.
int* ggd_err_word(DevBuf& buf, int*& host, cudaStream_t st) {
    int* d = buf.get<int>(1);
    cuda_check(cudaMemsetAsync(d, 0, sizeof(int), st), "clear error word");
    if (!host) cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&host), sizeof(int), cudaHostAllocDefault), "cudaHostAlloc");
    *host = 0;
    return d;
}

// libgqc carries its own (static) CUDA runtime, whose current device is not
// the caller's (torch.cuda.set_device does not reach it). Every call binds it
// explicitly: device-resident entry points to the device of the caller's
// stream (or of a buffer when the stream is the legacy default), host-buffer
// entry points to GQC_OPT_DEVICE.
void bind_device(cudaStream_t st, const void* dptr) {
    int dev = t_opt.device;
    if (st) {
        cuda_check(cudaStreamGetDevice(st, &dev), "cudaStreamGetDevice");
    } else if (dptr) {
        cudaPointerAttributes a{};
        cuda_check(cudaPointerGetAttributes(&a, dptr), "cudaPointerGetAttributes");
        if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) dev = a.device;
    }
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}

int visible_devices() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        count = 0;
    }
    return count;
}

std::atomic<int> g_ready[64];  // device contexts fully created (gqc_device_ready)

// The context of device `dev`, locked by this call (see t_held) and created
// on first use; the calling thread is bound to the device.
DeviceCtx& ctx_of(int dev) {
    static std::mutex map_mu;
    static std::map<int, DeviceCtx> all;
    DeviceCtx* cp;
    {
        std::lock_guard<std::mutex> l(map_mu);
        cp = &all[dev];
    }
    DeviceCtx& c = *cp;
    if (std::find(t_held.begin(), t_held.end(), &c.mu) == t_held.end()) {
        c.mu.lock();
        t_held.push_back(&c.mu);
    }
    c.dev = dev;
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    if (!c.stream) {
        cuda_check(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking), "cudaStreamCreate");
        for (auto& sl : c.slab) cuda_check(cudaStreamCreateWithFlags(&sl, cudaStreamNonBlocking), "cudaStreamCreate");
        for (auto& e : c.ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        for (auto& e : c.slab_done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    if (!c.pool) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cuda_check(cudaMemPoolCreate(&c.pool, &props), "cudaMemPoolCreate");
        std::uint64_t keep = ~0ull;
        cuda_check(cudaMemPoolSetAttribute(c.pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
    }
    if (dev >= 0 && dev < 64) g_ready[dev].store(1);
    return c;
}

DeviceCtx& ctx(cudaStream_t st = nullptr, const void* dptr = nullptr) {
    if (visible_devices() == 0) fail(GQC_ECUDA, "no CUDA device available (libgqc has no CPU path)");
    bind_device(st, dptr);
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    return ctx_of(dev);
}

ShardBufs& shard_bufs(DeviceCtx& C, std::size_t slot) {
    while (C.shards.size() <= slot) C.shards.emplace_back(new ShardBufs);
    ShardBufs& B = *C.shards[slot];
    if (!B.stream) {
        cuda_check(cudaSetDevice(C.dev), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&B.stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&B.ev_pot, cudaEventDisableTiming), "cudaEventCreate");
    }
    return B;
}

void check_csr_shape(const gqc_csr* g) {
    if (!g) fail(GQC_EINVAL, "graph is null");
    if (g->n < 1) fail(GQC_EINVAL, "graph needs at least one node");  // graph.cpp:28
    if (g->nnz < 0) fail(GQC_EINVAL, "negative edge count");
    if (!g->offsets || (g->nnz > 0 && !g->nbr)) fail(GQC_EINVAL, "graph arrays are null");
    if (!(g->W > 0.0)) fail(GQC_EINVAL, "default distance must be positive");  // graph.cpp:29
}

void check_sigmas(const double* sigmas, int n_sigma) {
    if (n_sigma < 1 || !sigmas) fail(GQC_EINVAL, "sigma grid is empty");
    for (int k = 0; k < n_sigma; ++k)
        if (!(sigmas[k] > 0.0)) fail(GQC_EINVAL, "sigma must be positive");  // potential.cpp:39-42
}

bool all_unit(const double* w, long long nnz) {
    for (long long k = 0; k < nnz; ++k)
        if (w[k] != 1.0) return false;
    return true;
}

// glibc exp over a [count][S] block, split across host threads.
void host_exp_table(const double* d2, long long count, const std::vector<double>& neg_inv, int S, double* out) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const long long per = (count + hw - 1) / hw;
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < hw; ++t) {
        const long long b = t * per, e = std::min(count, b + per);
        if (b >= e) break;
        pool.emplace_back([=, &neg_inv] {
            for (long long k = b; k < e; ++k)
                for (int s = 0; s < S; ++s) out[k * S + s] = host_glibc_exp(neg_inv[s] * d2[k]);
        });
    }
    for (auto& th : pool) th.join();
}

// Potentials of rows [row_begin, row_end) into v_nm[(i-row_begin)*S + s]
// (device), for a device-resident CSR. host_w: the same weights on the host
// (only consulted for weighted graphs), or nullptr to fetch what is needed.
// Polled upload: the slab flag is written by a stream memory operation
// (cuStreamWriteValue32, run by the GPU's front end behind a memory fence
// scoped to the stream, so the slab's copy is visible before the flag) — not
// by a kernel: the potential kernel that waits on the flag occupies every SM,
// so a flag kernel would only run after the wait timed out. Without the
// driver entry point, a copy from pinned memory (copy engine) writes it.
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
    static const WriteValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return static_cast<WriteValue32Fn>(nullptr);
        }
        return reinterpret_cast<WriteValue32Fn>(p);
    }();
    return fn;
}

void set_slab_flag(int* flag, const int* pinned_one, cudaStream_t cs) {
    if (WriteValue32Fn fn = write_value32()) {
        if (fn(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(flag), 1u, 0u) == CUDA_SUCCESS) return;
    }
    cuda_check(cudaMemcpyAsync(flag, pinned_one, sizeof(int), cudaMemcpyHostToDevice, cs), "set slab flag");
}

long long slab_timeout_ms() {  // GQC_SLAB_TIMEOUT_MS: polled-upload flag wait before GQC_ECUDA
    static const long long ms = [] {
        const char* e = std::getenv("GQC_SLAB_TIMEOUT_MS");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? v : 5000ll;
    }();
    return ms;
}

struct SlabSync {  // polled CSR upload (see PotentialLaunch::slab_flags)
    const int* flags = nullptr;
    int bound[5] = {};
    int* err = nullptr;
};

// peer (optional): per sigma chunk q of out_chunk sigmas, where row
// row_begin's slot of that chunk lives (node-major rows of out_chunk values,
// on any device this one can address): the multi-device sweep's fused
// exchange. scr: scratch for weighted tables (default: the context's).
void run_potentials(DeviceCtx& C, const gqc_csr& g, const double* sigmas, int S, int row_begin, int row_end,
                    double* v_nm, const double* host_w, cudaStream_t st, const std::int64_t* host_off = nullptr,
                    int out_chunk = 0, long long out_chunk_stride = 0, const SlabSync* sync = nullptr,
                    double* const* peer = nullptr, PotScratch* scr = nullptr) {
    if (!scr) scr = &C.scr;
    const int n = g.n;
    const int mode = t_opt.exp_mode;
    const bool weighted = g.w != nullptr;
    const bool tail = (mode == GQC_EXP_EIGEN) && (n % 2 == 1);
    const int K = t_opt.hop_cap;
    if (K > 1 && weighted) fail(GQC_EINVAL, "k-hop distances need unit weights");
    if (K > 1 && n >= (1 << 29)) fail(GQC_EINVAL, "k-hop distances need fewer than 2^29 nodes");

    // weighted graphs: the glibc-evaluated entries the device cannot produce
    std::vector<double> last_w;        // weights of row n-1 (Eigen tail)
    std::vector<double> all_d2;        // d2 per entry (glibc mode)
    long long last_beg = 0, last_deg = 0;
    if (weighted && tail) {
        long long o[2];
        if (host_off) {
            o[0] = host_off[n - 1];
            o[1] = host_off[n];
        } else {
            cuda_check(cudaStreamSynchronize(st), "sync");
            cuda_check(cudaMemcpy(o, g.offsets + (n - 1), 2 * sizeof(long long), cudaMemcpyDeviceToHost), "copy offsets");
        }
        last_beg = o[0];
        last_deg = o[1] - o[0];
        last_w.resize(last_deg);
        if (last_deg > 0) {
            if (host_w) {
                std::copy(host_w + last_beg, host_w + last_beg + last_deg, last_w.begin());
            } else {
                cuda_check(cudaStreamSynchronize(st), "sync");
                cuda_check(cudaMemcpy(last_w.data(), g.w + last_beg, last_deg * sizeof(double), cudaMemcpyDeviceToHost),
                           "copy weights");
            }
        }
    }
    if (weighted && mode == GQC_EXP_GLIBC) {
        all_d2.resize(g.nnz);
        std::vector<double> tmp;
        const double* hw = host_w;
        if (!hw) {
            tmp.resize(g.nnz);
            cuda_check(cudaStreamSynchronize(st), "sync");
            if (g.nnz)
                cuda_check(cudaMemcpy(tmp.data(), g.w, g.nnz * sizeof(double), cudaMemcpyDeviceToHost), "copy weights");
            hw = tmp.data();
        }
        for (long long k = 0; k < g.nnz; ++k) all_d2[k] = hw[k] * hw[k];
    }

    for (int s0 = 0; s0 < S; s0 += kMaxSigmaPerLaunch) {
        const int Sc = std::min(kMaxSigmaPerLaunch, S - s0);
        PotentialLaunch P{};
        P.n = n;
        P.n_sigma = Sc;
        P.row_begin = row_begin;
        P.row_end = row_end;
        P.nnz = g.nnz;
        P.offsets = g.offsets;
        P.nbr = g.nbr;
        P.w = g.w;
        P.tail = tail ? 1 : 0;
        P.out = v_nm;
        P.out_col0 = s0;
        P.out_chunk = out_chunk > 0 ? out_chunk : S;  // packed sigma chunks, or plain rows of S
        P.out_ld = P.out_chunk;
        P.out_chunk_stride = out_chunk > 0 ? out_chunk_stride : 0;
        if (peer) {
            P.out_peer = 1;
            const int chunks = (S + P.out_chunk - 1) / P.out_chunk;
            for (int q = 0; q < chunks && q < kMaxShards; ++q) P.out_chunk_ptr[q] = peer[q];
        }
        if (sync) {
            P.slab_flags = sync->flags;
            for (int k = 0; k < 5; ++k) P.slab_bound[k] = sync->bound[k];
            P.slab_err = sync->err;
            P.slab_timeout_ns = slab_timeout_ms() * 1000000ll;
        }
        std::vector<double> neg_inv(Sc);
        for (int s = 0; s < Sc; ++s) {
            P.c[s] = make_sigma_consts(sigmas[s0 + s], g.W, mode);
            neg_inv[s] = P.c[s].neg_inv;
        }
        if (K > 1) {  // k-hop extension (khop.cu)
            P.weight_mode = kUnit;
            KhopTable t{};
            for (int s = 0; s < Sc; ++s) fill_khop_table(t, s, sigmas[s0 + s], K, mode);
            cuda_check(launch_potentials_khop(P, K, t, C.pool, st), "k-hop potential launch");
            continue;
        }
        if (!weighted) {
            P.weight_mode = kUnit;
            // graphs with isolated rows (degree sample, cached per device CSR)
            // take the fast-forward's isolated-row instantiation
            if (t_opt.kernel == GQC_KERNEL_FASTFWD) P.iso = isolated_rows_device(g.offsets, g.n, g.nnz, st);
        } else if (mode == GQC_EXP_EIGEN) {
            P.weight_mode = kDevicePexp;
            if (tail && last_deg > 0) {
                std::vector<double> d2(last_deg), tab(last_deg * Sc);
                for (long long q = 0; q < last_deg; ++q) d2[q] = last_w[q] * last_w[q];
                host_exp_table(d2.data(), last_deg, neg_inv, Sc, tab.data());
                double* dtab = scr->tail.get<double>(tab.size());
                cuda_check(cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st),
                           "copy tail table");
                cuda_check(cudaStreamSynchronize(st), "sync");  // tab is a local
                P.tail_exp = dtab;
            }
        } else {
            P.weight_mode = kEntryTable;
            std::vector<double> tab(static_cast<std::size_t>(g.nnz) * Sc);
            host_exp_table(all_d2.data(), g.nnz, neg_inv, Sc, tab.data());
            double* dtab = scr->entry.get<double>(std::max<std::size_t>(tab.size(), 1));
            if (!tab.empty())
                cuda_check(cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st),
                           "copy entry table");
            cuda_check(cudaStreamSynchronize(st), "sync");
            P.entry_exp = dtab;
            P.entry_ld = Sc;
            P.entry_col0 = 0;
        }
        cuda_check(launch_potentials(P, t_opt.kernel, C.pool, st), "potential kernel launch");
    }
}

// Device copy of a host CSR (cached buffers). Unit weights are detected and
// passed as NULL so the constant-only kernel runs.
gqc_csr upload_csr(DeviceCtx& C, const gqc_csr* g, cudaStream_t st, const double** host_w_out) {
    const long long nnz = g->nnz;
    if (g->offsets[0] != 0 || g->offsets[g->n] != nnz) fail(GQC_EINVAL, "CSR offsets do not match nnz");
    gqc_csr d = *g;
    auto* off = C.off.get<std::int64_t>(g->n + 1);
    auto* nbr = C.nbr.get<std::int32_t>(std::max<long long>(nnz, 1));
    cuda_check(cudaMemcpyAsync(off, g->offsets, (g->n + 1) * sizeof(std::int64_t), cudaMemcpyHostToDevice, st),
               "copy offsets");
    if (nnz)
        cuda_check(cudaMemcpyAsync(nbr, g->nbr, nnz * sizeof(std::int32_t), cudaMemcpyHostToDevice, st), "copy nbr");
    d.offsets = off;
    d.nbr = nbr;
    d.w = nullptr;
    *host_w_out = nullptr;
    if (g->w && !all_unit(g->w, nnz)) {
        auto* w = C.w.get<double>(std::max<long long>(nnz, 1));
        cuda_check(cudaMemcpyAsync(w, g->w, nnz * sizeof(double), cudaMemcpyHostToDevice, st), "copy weights");
        d.w = w;
        *host_w_out = g->w;
    }
    return d;
}


// Degree-class order of a field for the GGD argmin fast path (kernels.cu,
// launch_class_order + successors_class_kernel). Verified per sigma on the
// field, so exact for any input, but OFF by default (GQC_CLASS_ORDER=1 turns
// it on): its sort + per-class min/max pass costs about what it saves.
// Measured (1 B200, 32 sigmas, GGD ms plain -> class order): LFR 1M
// 1.31 -> 1.19, SBM 100k 0.117 -> 0.216, R-MAT scale 22 6.49 -> 6.68.
struct ClassOrderScope {
    ClassOrder co;
    void* mem = nullptr;
    cudaStream_t st = nullptr;
    ClassOrderScope() = default;
    ClassOrderScope(const ClassOrderScope&) = delete;
    ClassOrderScope& operator=(const ClassOrderScope&) = delete;
    ~ClassOrderScope() {
        if (mem) cudaFreeAsync(mem, st);
    }
    const ClassOrder* get() const { return co.dir ? &co : nullptr; }
};

bool polled_upload_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GQC_POLLED_UPLOAD");
        return !(e && *e == '0');
    }();
    return on;
}

// graphs of at least this many nodes start the GGD of a host-API sweep with
// half-size sigma chunks (see cluster_sweep_impl)
constexpr int kSmallFirstChunkRows = 1 << 21;

bool class_order_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GQC_CLASS_ORDER");
        return e && *e == '1';
    }();
    return on;
}

void make_class_order(DeviceCtx& C, const gqc_csr& g, const double* v, int ld, int S, cudaStream_t st,
                      ClassOrderScope& out) {
    // weighted graphs and k-hop fields are not degree-determined: plain argmin
    if (!class_order_enabled() || g.w || t_opt.hop_cap > 1) return;
    const int n = g.n;
    const std::int64_t* off = g.offsets;
    const long long nnz = g.nnz;
    out.st = st;
    cuda_check(launch_class_order(n, off, nnz, v, ld, S, C.pool, st, &out.co, &out.mem), "class order");
}
}  // namespace

void count_launch(int k) { t_launches += k; }

int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cache[dev].load();
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev].store(v);
    }
    return v;
}

}  // namespace gqc

using namespace gqc;

extern "C" {

const char* gqc_last_error(void) { return t_err.c_str(); }
const char* gqc_version(void) { return "gqc 0.1 sm_100a"; }
int64_t gqc_last_launch_count(void) { return t_launches; }

void* gqc_host_alloc(size_t bytes) {
    void* p = nullptr;
    const gqc_status st = guarded([&] {
        ctx();
        cuda_check(cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocDefault), "cudaHostAlloc");
    });
    return st == GQC_OK ? p : nullptr;
}

void gqc_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

gqc_status gqc_host_register(void* p, size_t bytes) {
    return guarded([&] {
        if (!p || bytes == 0) return;
        ctx();
        cuda_check(cudaHostRegister(p, bytes, cudaHostRegisterDefault), "cudaHostRegister");
    });
}

gqc_status gqc_host_unregister(void* p) {
    return guarded([&] {
        if (!p) return;
        ctx();
        cuda_check(cudaHostUnregister(p), "cudaHostUnregister");
    });
}

int32_t gqc_device_ready(void) {
    const int d = g_opt.device.load();
    return d >= 0 && d < 64 ? g_ready[d].load() : 0;
}

int32_t gqc_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

static void cluster_sweep_impl(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out,
                               int32_t* succ_out, int32_t* center_out, int32_t* cluster_index_out,
                               int32_t* num_clusters_out, int64_t* intra_out = nullptr);
static void sweep_multi_impl(const gqc_csr* g, const double* sigmas, int S, const int* devices, int shards,
                             double* v_out, int* succ_out, int* center_out, int* ci_out, int* nc_out,
                             std::int64_t* intra_out, bool potentials_only);
static std::vector<int> option_devices();

gqc_status gqc_init(void) {
    return guarded([&] {
        ctx();
        // two tiny sweeps (8 sigmas and 1): create the context's streams and
        // pool and load the modules of the kernels a sweep launches
        const std::int64_t off[4] = {0, 1, 3, 4};
        const std::int32_t nbr[4] = {1, 0, 2, 1};
        const gqc_csr g{3, 4, off, nbr, nullptr, 10.0};
        double sig[8];
        for (int k = 0; k < 8; ++k) sig[k] = 1.0 + k;
        std::int32_t ci[24], nc[8];
        for (int S : {8, 1}) cluster_sweep_impl(&g, sig, S, nullptr, nullptr, nullptr, ci, nc);
    });
}

gqc_status gqc_reserve(int32_t n, int64_t nnz, int32_t n_sigma) {
    return guarded([&] {
        if (n < 1 || nnz < 0 || n_sigma < 1) fail(GQC_EINVAL, "bad reserve sizes");
        DeviceCtx& C = ctx();
        const std::size_t cells = static_cast<std::size_t>(n) * n_sigma;
        C.off.get<std::int64_t>(static_cast<std::size_t>(n) + 1);
        C.nbr.get<std::int32_t>(std::max<std::int64_t>(nnz, 1));
        C.v_nm.get<double>(cells);
        C.succ.get<int>(cells);
        C.center.get<int>(cells);
        C.ci.get<int>(cells);
        C.nc.get<int>(n_sigma);
        C.intra.get<long long>(n_sigma);
        C.ws.get<char>(labels_workspace_bytes(n, n_sigma));
        C.slab_sync.get<int>(8);
        if (!C.slab_host) {
            cuda_check(cudaHostAlloc(&C.slab_host, 8 * sizeof(int), cudaHostAllocDefault), "cudaHostAlloc");
            for (int k = 0; k < 8; ++k) C.slab_host[k] = 1;
        }
        pinned_counts(C, n_sigma);
        (void)ggd_err_word(C.err, C.err_host, C.stream);
        // the pool keeps what it has held (release threshold: never): one
        // block the size of a sweep's stream-ordered scratch (schedule arrays
        // and sort, prefix tables, argmin lists), handed back at once
        void* p = nullptr;
        const std::size_t est = 20 * static_cast<std::size_t>(n) + (static_cast<std::size_t>(nnz) / 64) + (64u << 20);
        cuda_check(cudaMallocFromPoolAsync(&p, est, C.pool, C.stream), "pool reserve");
        cuda_check(cudaFreeAsync(p, C.stream), "pool reserve");
        cuda_check(cudaStreamSynchronize(C.stream), "sync");
    });
}

gqc_status gqc_set_option(gqc_option key, int64_t value) {
    return guarded([&] {
        if (key == GQC_OPT_EXP_MODE) {
            if (value != GQC_EXP_EIGEN && value != GQC_EXP_GLIBC) fail(GQC_EINVAL, "unknown exp mode");
            g_opt.exp_mode = static_cast<int>(value);
        } else if (key == GQC_OPT_KERNEL) {
            if (value != GQC_KERNEL_FASTFWD && value != GQC_KERNEL_REPLAY) fail(GQC_EINVAL, "unknown kernel");
            g_opt.kernel = static_cast<int>(value);
        } else if (key == GQC_OPT_HOP_CAP) {
            if (value < 1 || value > kMaxHopCap) fail(GQC_EINVAL, "hop cap must be in 1..7");
            g_opt.hop_cap = static_cast<int>(value);
        } else if (key == GQC_OPT_DEVICE) {
            if (value < 0 || value >= visible_devices()) fail(GQC_EINVAL, "device ordinal out of range");
            g_opt.device = static_cast<int>(value);
        } else if (key == GQC_OPT_GPUS) {
            if (value < 1 || value > kMaxShards) fail(GQC_EINVAL, "gpu count must be in 1..32");
            g_opt.gpus = static_cast<int>(value);
        } else {
            fail(GQC_EINVAL, "unknown option");
        }
    });
}

gqc_status gqc_get_option(gqc_option key, int64_t* value) {
    return guarded([&] {
        if (!value) fail(GQC_EINVAL, "null output");
        if (key == GQC_OPT_EXP_MODE) *value = g_opt.exp_mode;
        else if (key == GQC_OPT_KERNEL) *value = g_opt.kernel;
        else if (key == GQC_OPT_DEVICE) *value = g_opt.device;
        else if (key == GQC_OPT_HOP_CAP) *value = g_opt.hop_cap;
        else if (key == GQC_OPT_GPUS) *value = g_opt.gpus;
        else fail(GQC_EINVAL, "unknown option");
    });
}

gqc_status gqc_potentials(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out) {
    return guarded([&] {
        if (t_opt.gpus > 1) {
            const std::vector<int> d = option_devices();
            sweep_multi_impl(g, sigmas, n_sigma, d.data(), static_cast<int>(d.size()), v_out, nullptr, nullptr, nullptr,
                             nullptr, nullptr, true);
            return;
        }
        check_sigmas(sigmas, n_sigma);
        check_csr_shape(g);
        if (!v_out) fail(GQC_EINVAL, "null output");
        DeviceCtx& C = ctx();
        cudaStream_t st = C.stream;
        const double* hw = nullptr;
        gqc_csr d = upload_csr(C, g, st, &hw);
        const std::size_t cells = static_cast<std::size_t>(g->n) * n_sigma;
        double* v_nm = C.v_nm.get<double>(cells);
        run_potentials(C, d, sigmas, n_sigma, 0, g->n, v_nm, hw, st);
        double* src = v_nm;
        if (n_sigma > 1) {
            src = C.v_sm.get<double>(cells);
            cuda_check(launch_transpose(v_nm, g->n, n_sigma, src, st), "transpose");
        }
        cuda_check(cudaMemcpyAsync(v_out, src, cells * sizeof(double), cudaMemcpyDeviceToHost, st), "copy V");
        cuda_check(cudaStreamSynchronize(st), "potential sweep");
    });
}

gqc_status gqc_node_potential(const gqc_csr* g, int32_t node, double sigma, double* out) {
    return guarded([&] {
        check_sigmas(&sigma, 1);  // potential.cpp:47 checks sigma before the node
        check_csr_shape(g);
        if (node < 0 || node >= g->n) fail(GQC_ERANGE, "node id " + std::to_string(node) + " out of range");
        if (!out) fail(GQC_EINVAL, "null output");
        DeviceCtx& C = ctx();
        cudaStream_t st = C.stream;
        const double* hw = nullptr;
        gqc_csr d = upload_csr(C, g, st, &hw);
        double* v = C.v_nm.get<double>(1);
        run_potentials(C, d, &sigma, 1, node, node + 1, v, hw, st);
        cuda_check(cudaMemcpyAsync(out, v, sizeof(double), cudaMemcpyDeviceToHost, st), "copy V");
        cuda_check(cudaStreamSynchronize(st), "node potential");
    });
}

gqc_status gqc_build_successors(const gqc_csr* g, const double* v, int32_t* succ) {
    return guarded([&] {
        check_csr_shape(g);
        if (!v || !succ) fail(GQC_EINVAL, "null buffer");
        DeviceCtx& C = ctx();
        cudaStream_t st = C.stream;
        const double* hw = nullptr;
        gqc_csr d = upload_csr(C, g, st, &hw);
        double* dv = C.v_nm.get<double>(g->n);
        int* ds = C.succ.get<int>(g->n);
        cuda_check(cudaMemcpyAsync(dv, v, g->n * sizeof(double), cudaMemcpyHostToDevice, st), "copy V");
        cuda_check(launch_successors(g->n, d.offsets, d.nbr, dv, 1, 0, 1, 0, g->n, ds, 1, g->n, g->nnz, C.pool, st), "successor kernel");
        cuda_check(cudaMemcpyAsync(succ, ds, g->n * sizeof(int), cudaMemcpyDeviceToHost, st), "copy succ");
        cuda_check(cudaStreamSynchronize(st), "build successors");
    });
}

gqc_status gqc_resolve_centers(int32_t n, const int32_t* succ, int32_t* center, int32_t* cluster_index,
                               int32_t* num_clusters) {
    return guarded([&] {
        if (n < 0) fail(GQC_EINVAL, "negative size");
        if (n == 0) {
            if (num_clusters) *num_clusters = 0;
            return;
        }
        if (!succ || !center || !cluster_index || !num_clusters) fail(GQC_EINVAL, "null buffer");
        DeviceCtx& C = ctx();
        cudaStream_t st = C.stream;
        int* ds = C.succ.get<int>(n);
        int* dc = C.center.get<int>(n);
        int* dci = C.ci.get<int>(n);
        cuda_check(cudaMemcpyAsync(ds, succ, n * sizeof(int), cudaMemcpyHostToDevice, st), "copy succ");
        int err = 0;
        int k = 0;
        cuda_check(resolve_checked(n, ds, dc, dci, &k, &err, C.pool, st), "resolve centers");
        if (err == 1) fail(GQC_EINVAL, "successor id out of range");  // ggd.cpp:37-38
        if (err == 2) fail(GQC_ECYCLE, "successor map contains a cycle");  // ggd.cpp:41
        cuda_check(cudaMemcpyAsync(center, dc, n * sizeof(int), cudaMemcpyDeviceToHost, st), "copy center");
        cuda_check(cudaMemcpyAsync(cluster_index, dci, n * sizeof(int), cudaMemcpyDeviceToHost, st), "copy index");
        cuda_check(cudaStreamSynchronize(st), "resolve centers");
        *num_clusters = k;
    });
}

#ifndef GQC_GGD_CHUNK
#define GQC_GGD_CHUNK 16
#endif
// sigmas per GGD pass of the host pipeline: each pass's labels go down while
// the next pass computes, so the last pass's download is the exposed tail
constexpr int kGgdChunk = GQC_GGD_CHUNK;

// The body of gqc_cluster_sweep (inside guarded()).
static void cluster_sweep_impl(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out, int32_t* succ_out,
                        int32_t* center_out, int32_t* cluster_index_out, int32_t* num_clusters_out,
                        int64_t* intra_out) {
    {
        check_sigmas(sigmas, n_sigma);
        check_csr_shape(g);
        if (!cluster_index_out || !num_clusters_out) fail(GQC_EINVAL, "null output");
        if (g->offsets[0] != 0 || g->offsets[g->n] != g->nnz) fail(GQC_EINVAL, "CSR offsets do not match nnz");
        DeviceCtx& C = ctx();
        cudaStream_t st = C.stream, cs = C.copy;
        Tracer tr(st);
        const int n = g->n;
        const long long nnz = g->nnz;
        const bool weighted = g->w && !all_unit(g->w, nnz);
        if (t_opt.hop_cap > 1 && weighted) fail(GQC_EINVAL, "k-hop distances need unit weights");
        if (intra_out && weighted) fail(GQC_EINVAL, "intra counts need unit weights");

        // Pipeline: the CSR goes up in row slabs on the copy stream while the
        // compute stream runs the potentials of the slabs already resident
        // (rows are independent); GGD then runs in sigma chunks whose labels
        // go down on the copy stream while the next chunk computes.
        gqc_csr d = *g;
        auto* off = C.off.get<std::int64_t>(n + 1);
        auto* nbr = C.nbr.get<std::int32_t>(std::max<long long>(nnz, 1));
        double* w = weighted ? C.w.get<double>(std::max<long long>(nnz, 1)) : nullptr;
        d.offsets = off;
        d.nbr = nbr;
        d.w = w;
        cuda_check(cudaMemcpyAsync(off, g->offsets, (n + 1) * sizeof(std::int64_t), cudaMemcpyHostToDevice, cs),
                   "copy offsets");
        {  // row n-1 first: rows adjacent to the Eigen tail column search its list (weighted graphs)
            const long long a = g->offsets[n - 1], b = g->offsets[n];
            if (b > a) {
                cuda_check(cudaMemcpyAsync(nbr + a, g->nbr + a, (b - a) * sizeof(std::int32_t), cudaMemcpyHostToDevice, cs),
                           "copy nbr");
                if (weighted)
                    cuda_check(cudaMemcpyAsync(w + a, g->w + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice, cs),
                               "copy weights");
            }
        }
        // (k-hop rows read their neighbours' rows too: one slab, the whole CSR)
        const int slabs = (nnz >= (1 << 20) && t_opt.hop_cap == 1) ? 4 : 1;
        // (the warp kernel waits on the slab flags: every fast-forward sweep, or >= 8 sigmas)
        const bool polled = slabs == 4 && !weighted && (n_sigma >= 8 || t_opt.kernel == GQC_KERNEL_FASTFWD) &&
                            polled_upload_enabled();
        std::vector<int> bound(slabs + 1, n);
        bound[0] = 0;
        // equal-nnz row slabs; polled: growing (cumulative 10%, 30%, 60%): the
        // first slab lands fast and every later one (the copy engine moves
        // the CSR ~2.7x faster than the kernel consumes it) arrives before
        // the warps reach it
        static const double kGeo[3] = {0.10, 0.30, 0.60};
        for (int k = 1; k < slabs; ++k) {
            const long long at = polled ? static_cast<long long>(nnz * kGeo[k - 1]) : nnz * k / slabs;
            bound[k] = static_cast<int>(std::lower_bound(g->offsets, g->offsets + n + 1, at) - g->offsets);
        }
        const std::size_t cells = static_cast<std::size_t>(n) * n_sigma;
        double* v_nm = C.v_nm.get<double>(cells);
        // Polled upload (unit weights, warp kernel; GQC_POLLED_UPLOAD=0 turns
        // it off): ONE potential launch starts once the offsets are resident;
        // its warps take rows slab-major and wait on a flag per slab that the
        // copy stream sets right after the slab's entries land. Each slab's
        // copy is extended to whole 128 B lines so no line a warp reads can be
        // cached half-written. Otherwise one launch per slab on its own stream.
        if (polled) {
            int* flags = C.slab_sync.get<int>(8);
            if (!C.slab_host) {
                cuda_check(cudaHostAlloc(&C.slab_host, 8 * sizeof(int), cudaHostAllocDefault), "cudaHostAlloc");
                for (int k = 0; k < 8; ++k) C.slab_host[k] = 1;
            }
            C.slab_host[4] = 0;
            cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), cs), "clear flags");
            cuda_check(cudaEventRecord(C.ev[0], cs), "event");  // offsets (and the flags) resident
            for (int k = 0; k < slabs; ++k) {
                const long long a = g->offsets[bound[k]], b = g->offsets[bound[k + 1]];
                const long long a2 = a & ~31ll, b2 = std::min<long long>(nnz, (b + 31) & ~31ll);
                if (b2 > a2)
                    cuda_check(cudaMemcpyAsync(nbr + a2, g->nbr + a2, (b2 - a2) * sizeof(std::int32_t),
                                               cudaMemcpyHostToDevice, cs),
                               "copy nbr");
                set_slab_flag(flags + k, C.slab_host + k, cs);
            }
            cuda_check(cudaStreamWaitEvent(st, C.ev[0], 0), "wait");
            SlabSync sync;
            sync.flags = flags;
            for (int k = 0; k <= slabs; ++k) sync.bound[k] = bound[k];
            sync.err = flags + 4;
            run_potentials(C, d, sigmas, n_sigma, 0, n, v_nm, nullptr, st, g->offsets, 0, 0, &sync);
            cuda_check(cudaMemcpyAsync(C.slab_host + 4, flags + 4, sizeof(int), cudaMemcpyDeviceToHost, st),
                       "copy upload status");
        }
        for (int k = 0; k < slabs && !polled; ++k) {
            const long long a = g->offsets[bound[k]], b = g->offsets[bound[k + 1]];
            if (b > a) {
                cuda_check(cudaMemcpyAsync(nbr + a, g->nbr + a, (b - a) * sizeof(std::int32_t), cudaMemcpyHostToDevice, cs),
                           "copy nbr");
                if (weighted)
                    cuda_check(cudaMemcpyAsync(w + a, g->w + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice, cs),
                               "copy weights");
            }
            // each slab's potentials on its own stream: slabs run concurrently
            // (a slab holding a hub row does not hold back the others)
            cuda_check(cudaEventRecord(C.ev[k], cs), "event");
            cudaStream_t ss = C.slab[k];
            cuda_check(cudaStreamWaitEvent(ss, C.ev[k], 0), "wait");
            if (bound[k + 1] > bound[k])
                run_potentials(C, d, sigmas, n_sigma, bound[k], bound[k + 1], v_nm + static_cast<std::size_t>(bound[k]) * n_sigma,
                               weighted ? g->w : nullptr, ss, g->offsets);
            cuda_check(cudaEventRecord(C.slab_done[k], ss), "event");
        }
        for (int k = 0; k < slabs && !polled; ++k) cuda_check(cudaStreamWaitEvent(st, C.slab_done[k], 0), "wait");
        tr.mark("potentials");
        double* v_src = v_nm;
        const bool v_early = v_out && host_pinned(v_out);  // pageable: copied after the GGD launches
        if (v_out) {  // sigma-major copy of the field
            if (n_sigma > 1) {
                v_src = C.v_sm.get<double>(cells);
                cuda_check(launch_transpose(v_nm, n, n_sigma, v_src, st), "transpose");
            }
            if (v_early) {
                cuda_check(cudaEventRecord(C.ev[8], st), "event");
                cuda_check(cudaStreamWaitEvent(cs, C.ev[8], 0), "wait");
                cuda_check(cudaMemcpyAsync(v_out, v_src, cells * sizeof(double), cudaMemcpyDeviceToHost, cs), "copy V");
            }
        }
        int* ds = C.succ.get<int>(cells);
        int* dc = C.center.get<int>(cells);
        int* dci = C.ci.get<int>(cells);
        int* dnc = C.nc.get<int>(n_sigma);
        long long* d_intra = intra_out ? C.intra.get<long long>(n_sigma) : nullptr;
        const std::size_t wsb = labels_workspace_bytes(n, n_sigma);
        void* ws = C.ws.get<char>(wsb);
        // GGD chunk boundaries: equal chunks of GQC_GGD_CHUNK sigmas (16), or
        // with GQC_GGD_CHUNK=0 growing ones (S = 32: 4, 8, 8, 12) so the
        // downloads start after a small first chunk. Measured on LFR 1M x 32:
        // e2e 8.54 ms (16) vs 8.84 ms (growing); R-MAT 25.7 vs 27.4 ms.
        // GQC_GGD_CHUNK=-1: shrinking chunks (S = 32: 16, 8, 4, 4), so the one
        // download left exposed after the last GGD launch is small.
        std::vector<int> cuts{0};
        if (const char* e = std::getenv("GQC_GGD_CUTS"); e && *e && n_sigma >= 2) {
            // measurement knob: chunk sizes as a comma list, e.g. "4,8,8,12"
            for (const char* p = e; *p;) {
                char* q = nullptr;
                const long c = std::strtol(p, &q, 10);
                if (q == p) break;
                if (c > 0 && cuts.back() + c < n_sigma) cuts.push_back(cuts.back() + static_cast<int>(c));
                p = *q ? q + 1 : q;
            }
        } else if (kGgdChunk > 0 && n >= kSmallFirstChunkRows && n_sigma > kGgdChunk) {
            // large label volumes (R-MAT 22: 537 MB at 32 sigmas) keep the
            // copy engine busy for longer than the GGD: a half-size first
            // chunk (and second) starts the downloads sooner. Measured e2e
            // R-MAT 22: 25.40 (16/16) -> 24.41 ms (8/8/16); LFR 1M (n below
            // the threshold) keeps 16/16: 7.94 vs 8.00 ms
            const int half = kGgdChunk / 2;
            cuts.push_back(half);
            if (2 * half < n_sigma) cuts.push_back(2 * half);
            for (int s0 = 2 * half + kGgdChunk; s0 < n_sigma; s0 += kGgdChunk) cuts.push_back(s0);
        } else if (kGgdChunk > 0) {
            for (int s0 = kGgdChunk; s0 < n_sigma; s0 += kGgdChunk) cuts.push_back(s0);
        } else if (kGgdChunk == 0 && n_sigma >= 16) {
            for (int f : {1, 3, 5}) cuts.push_back((n_sigma * f + 7) / 8);
        } else if (kGgdChunk < 0 && n_sigma >= 16) {
            for (int f : {4, 6, 7}) cuts.push_back((n_sigma * f + 7) / 8);
        }
        cuts.push_back(n_sigma);
        // labels of a chunk go down while the next chunk computes; into
        // pageable buffers every copy blocks the host, so then all chunks are
        // launched first and the copies queued after them
        const bool overlap = host_pinned(cluster_index_out) && (!center_out || host_pinned(center_out)) &&
                             (!succ_out || host_pinned(succ_out));
        int* nc_stage = pinned_counts(C, n_sigma);
        int* d_err = ggd_err_word(C.err, C.err_host, st);
        int ev_i = 9;
        auto download = [&](int s0, int Sc) {
            const std::size_t o = static_cast<std::size_t>(s0) * n, c = static_cast<std::size_t>(Sc) * n;
            if (succ_out)
                cuda_check(cudaMemcpyAsync(succ_out + o, ds + o, c * sizeof(int), cudaMemcpyDeviceToHost, cs), "copy succ");
            if (center_out)
                cuda_check(cudaMemcpyAsync(center_out + o, dc + o, c * sizeof(int), cudaMemcpyDeviceToHost, cs), "copy center");
            cuda_check(cudaMemcpyAsync(cluster_index_out + o, dci + o, c * sizeof(int), cudaMemcpyDeviceToHost, cs),
                       "copy cluster index");
            cuda_check(cudaMemcpyAsync(nc_stage + s0, dnc + s0, Sc * sizeof(int), cudaMemcpyDeviceToHost, cs),
                       "copy counts");
        };
        ClassOrderScope order;
        make_class_order(C, d, v_nm, n_sigma, n_sigma, st, order);
        // the degree sample reads the host CSR while the potentials run
        const int sub = light_row_sigmas_host(g->offsets, n);
        for (std::size_t q = 0; q + 1 < cuts.size(); ++q) {
            const int s0 = cuts[q], Sc = cuts[q + 1] - cuts[q];
            const std::size_t o = static_cast<std::size_t>(s0) * n;
            cuda_check(launch_successors(n, d.offsets, d.nbr, v_nm, n_sigma, s0, Sc, 0, n, ds + o, 1, n, nnz, C.pool, st,
                                         order.get(), sub),
                       "successor kernel");
            cuda_check(launch_labels(n, Sc, ds + o, dc + o, dci + o, dnc + s0, ws, wsb, st, d_err), "label kernels");
            if (intra_out)
                cuda_check(launch_intra_counts(n, Sc, d.offsets, d.nbr, dci + o, d_intra + s0, st), "intra counts");
            tr.mark("ggd_chunk");
            if (overlap) {
                cudaEvent_t e = C.ev[ev_i];
                ev_i = ev_i == 15 ? 9 : ev_i + 1;
                cuda_check(cudaEventRecord(e, st), "event");
                cuda_check(cudaStreamWaitEvent(cs, e, 0), "wait");
                download(s0, Sc);
            }
        }
        if (!overlap || (v_out && !v_early)) {
            cuda_check(cudaEventRecord(C.ev[9], st), "event");
            cuda_check(cudaStreamWaitEvent(cs, C.ev[9], 0), "wait");
        }
        if (!overlap)
            for (std::size_t q = 0; q + 1 < cuts.size(); ++q) download(cuts[q], cuts[q + 1] - cuts[q]);
        if (v_out && !v_early)
            cuda_check(cudaMemcpyAsync(v_out, v_src, cells * sizeof(double), cudaMemcpyDeviceToHost, cs), "copy V");
        cuda_check(cudaEventRecord(C.ev[8], cs), "event");
        cuda_check(cudaStreamWaitEvent(st, C.ev[8], 0), "wait");
        tr.mark("downloads");
        if (intra_out)
            cuda_check(cudaMemcpyAsync(intra_out, d_intra, n_sigma * sizeof(long long), cudaMemcpyDeviceToHost, st),
                       "copy intra counts");
        cuda_check(cudaMemcpyAsync(C.err_host, d_err, sizeof(int), cudaMemcpyDeviceToHost, st), "copy error word");
        cuda_check(cudaStreamSynchronize(cs), "cluster sweep (copies)");
        cuda_check(cudaStreamSynchronize(st), "cluster sweep");
        if (polled && C.slab_host[4]) fail(GQC_ECUDA, "CSR upload did not arrive (polled slab flag timeout)");
        if (*C.err_host) fail(GQC_ECYCLE, "successor map contains a cycle");  // ggd.cpp:41
        std::copy(nc_stage, nc_stage + n_sigma, num_clusters_out);
    }
}

// ------------------------------------------------------------ multi-device
// Row shards of a multi-device sweep (gqc_row_shards): contiguous row blocks
// balanced by the fast-forward kernel's cost, ~ deg(i) + kRowCost per row.
// The reference's equal blocks (potential.cpp:70-74) balance its O(N) rows
// only; they are kept for the dense replay, whose rows all cost N.
constexpr long long kRowCost = 4;

static std::vector<int> row_shards(const std::int64_t* off, int n, int shards, int kernel) {
    std::vector<int> b(shards + 1, n);
    b[0] = 0;
    const long long total = off[n] + kRowCost * n;
    for (int r = 1; r < shards; ++r) {
        if (kernel == GQC_KERNEL_REPLAY) {  // potential.cpp:70-74
            b[r] = static_cast<int>(static_cast<long long>(n / shards) * r + std::min(r, n % shards));
            continue;
        }
        const long long target = total / shards * r + (total % shards) * r / shards;
        int lo = b[r - 1], hi = n;  // first row i with off[i] + kRowCost * i >= target
        while (lo < hi) {
            const int mid = lo + (hi - lo) / 2;
            if (off[mid] + kRowCost * mid < target) lo = mid + 1;
            else hi = mid;
        }
        b[r] = lo;
    }
    return b;
}

// The sweep over `shards` shards on devices[0..shards) (repeats allowed: a
// device then hosts several shards). Shard r computes the potentials of rows
// [rb[r], rb[r+1]) for every sigma; the potential kernel writes sigma chunk
// q (chunk = ceil(S / shards) sigmas) of those rows straight into shard q's
// node-major field V_q[n][chunk] on shard q's device (peer stores over
// NVLink: the kernel IS the exchange; without peer access the chunk is
// staged locally and copied peer-to-peer). Once every shard's potentials are
// done (cross-device event waits), shard q runs GGD for its sigma chunk and
// its labels go straight to the caller's sigma-major output. Bit-identical
// to the single-device sweep for any shard count: rows and sigmas are
// independent (potential.cpp:18-37, ggd.cpp:7-57).
static void sweep_multi_impl(const gqc_csr* g, const double* sigmas, int S, const int* devices, int shards, double* v_out,
                      int* succ_out, int* center_out, int* ci_out, int* nc_out, std::int64_t* intra_out,
                      bool potentials_only) {
    check_sigmas(sigmas, S);
    check_csr_shape(g);
    if (shards < 1 || shards > kMaxShards) fail(GQC_EINVAL, "shard count must be in 1..32");
    if (!devices) fail(GQC_EINVAL, "null device list");
    const int count = visible_devices();
    if (count == 0) fail(GQC_ECUDA, "no CUDA device available (libgqc has no CPU path)");
    for (int r = 0; r < shards; ++r)
        if (devices[r] < 0 || devices[r] >= count) fail(GQC_EINVAL, "device ordinal out of range");
    if (potentials_only ? !v_out : (!ci_out || !nc_out)) fail(GQC_EINVAL, "null output");
    if (g->offsets[0] != 0 || g->offsets[g->n] != g->nnz) fail(GQC_EINVAL, "CSR offsets do not match nnz");
    const int n = g->n;
    const long long nnz = g->nnz;
    const bool weighted = g->w && !all_unit(g->w, nnz);
    if (t_opt.hop_cap > 1 && weighted) fail(GQC_EINVAL, "k-hop distances need unit weights");
    if (intra_out && weighted) fail(GQC_EINVAL, "intra counts need unit weights");

    // devices locked in ascending order: concurrent multi-device calls cannot deadlock
    std::vector<int> uniq(devices, devices + shards);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    std::map<int, DeviceCtx*> C;
    for (int d : uniq) C[d] = &ctx_of(d);
    std::map<std::pair<int, int>, bool> direct;  // (writer, owner): peer stores possible
    for (int a : uniq)
        for (int b : uniq) {
            if (a == b) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess) can = 0;
            if (can) {
                cuda_check(cudaSetDevice(a), "cudaSetDevice");
                cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
                if (e != cudaSuccess) can = 0;
                cudaGetLastError();
            }
            direct[{a, b}] = can != 0;
        }

    // the CSR on every device (its copy stream); potentials wait on it
    std::map<int, gqc_csr> dcsr;
    for (int d : uniq) {
        DeviceCtx& X = *C[d];
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        gqc_csr dg = *g;
        auto* off = X.off.get<std::int64_t>(n + 1);
        auto* nbr = X.nbr.get<std::int32_t>(std::max<long long>(nnz, 1));
        cuda_check(cudaMemcpyAsync(off, g->offsets, (n + 1) * sizeof(std::int64_t), cudaMemcpyHostToDevice, X.copy),
                   "copy offsets");
        if (nnz)
            cuda_check(cudaMemcpyAsync(nbr, g->nbr, nnz * sizeof(std::int32_t), cudaMemcpyHostToDevice, X.copy),
                       "copy nbr");
        dg.offsets = off;
        dg.nbr = nbr;
        dg.w = nullptr;
        if (weighted) {
            auto* w = X.w.get<double>(std::max<long long>(nnz, 1));
            cuda_check(cudaMemcpyAsync(w, g->w, nnz * sizeof(double), cudaMemcpyHostToDevice, X.copy), "copy weights");
            dg.w = w;
        }
        cuda_check(cudaEventRecord(X.ev[0], X.copy), "event");
        dcsr[d] = dg;
    }

    const std::vector<int> rb = row_shards(g->offsets, n, shards, t_opt.kernel);
    const int chunk = (S + shards - 1) / shards;
    const int nchunks = (S + chunk - 1) / chunk;
    auto s_begin = [&](int q) { return std::min(S, q * chunk); };
    auto s_count = [&](int q) { return std::min(S, (q + 1) * chunk) - s_begin(q); };
    std::vector<ShardBufs*> B(shards);
    {
        std::map<int, std::size_t> slot;
        for (int r = 0; r < shards; ++r) B[r] = &shard_bufs(*C[devices[r]], slot[devices[r]]++);
    }
    std::vector<double*> V(shards, nullptr);
    for (int q = 0; q < nchunks; ++q) {
        cuda_check(cudaSetDevice(devices[q]), "cudaSetDevice");
        V[q] = B[q]->v.get<double>(static_cast<std::size_t>(n) * chunk);
    }

    // potentials: shard r's rows for every sigma, each chunk into its owner's V
    for (int r = 0; r < shards; ++r) {
        const int d = devices[r];
        DeviceCtx& X = *C[d];
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        cudaStream_t st = B[r]->stream;
        cuda_check(cudaStreamWaitEvent(st, X.ev[0], 0), "wait");
        const int rows = rb[r + 1] - rb[r];
        double* ptr[kMaxShards] = {};
        std::vector<int> staged;
        for (int q = 0; q < nchunks; ++q) {
            if (devices[q] == d || direct[{d, devices[q]}]) ptr[q] = V[q] + static_cast<std::size_t>(rb[r]) * chunk;
            else staged.push_back(q);
        }
        if (!staged.empty()) {
            double* send = B[r]->send.get<double>(std::max<std::size_t>(1, static_cast<std::size_t>(rows) * chunk * nchunks));
            for (int q : staged) ptr[q] = send + static_cast<std::size_t>(q) * rows * chunk;
        }
        if (rows > 0) {
            run_potentials(X, dcsr[d], sigmas, S, rb[r], rb[r + 1], nullptr, weighted ? g->w : nullptr, st, g->offsets,
                           chunk, 0, nullptr, ptr, &B[r]->scr);
            for (int q : staged)
                cuda_check(cudaMemcpyPeerAsync(V[q] + static_cast<std::size_t>(rb[r]) * chunk, devices[q], ptr[q], d,
                                               static_cast<std::size_t>(rows) * chunk * sizeof(double), st),
                           "peer copy");
        }
        cuda_check(cudaEventRecord(B[r]->ev_pot, st), "event");
    }

    // GGD of every sigma chunk on its owner once all potentials are in
    int sub_multi = 0;
    for (int q = 0; q < nchunks; ++q) {
        const int d = devices[q], Sq = s_count(q), s0 = s_begin(q);
        DeviceCtx& X = *C[d];
        ShardBufs& Bq = *B[q];
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        cudaStream_t st = Bq.stream;
        for (int r = 0; r < shards; ++r)
            if (r != q) cuda_check(cudaStreamWaitEvent(st, B[r]->ev_pot, 0), "wait");
        const std::size_t cells = static_cast<std::size_t>(Sq) * n;
        if (v_out) {
            double* vsm = Bq.v_sm.get<double>(static_cast<std::size_t>(chunk) * n);
            cuda_check(launch_transpose(V[q], n, chunk, vsm, st), "transpose");
        }
        if (potentials_only) continue;
        const gqc_csr& dg = dcsr[d];
        int* ds = Bq.succ.get<int>(cells);
        int* dc = Bq.center.get<int>(cells);
        int* dci = Bq.ci.get<int>(cells);
        int* dnc = Bq.nc.get<int>(Sq);
        const std::size_t wsb = labels_workspace_bytes(n, Sq);
        void* ws = Bq.ws.get<char>(wsb);
        ClassOrderScope order;
        make_class_order(X, dg, V[q], chunk, Sq, st, order);
        if (sub_multi == 0) sub_multi = light_row_sigmas_host(g->offsets, n);  // while the potentials run
        cuda_check(launch_successors(n, dg.offsets, dg.nbr, V[q], chunk, 0, Sq, 0, n, ds, 1, n, nnz, X.pool, st,
                                     order.get(), sub_multi),
                   "successor kernel");
        int* d_err = ggd_err_word(Bq.err, Bq.err_host, st);
        cuda_check(launch_labels(n, Sq, ds, dc, dci, dnc, ws, wsb, st, d_err), "label kernels");
        cuda_check(cudaMemcpyAsync(Bq.err_host, d_err, sizeof(int), cudaMemcpyDeviceToHost, st), "copy error word");
        if (intra_out)
            cuda_check(launch_intra_counts(n, Sq, dg.offsets, dg.nbr, dci, Bq.intra.get<long long>(Sq), st),
                       "intra counts");
        (void)s0;
    }
    // downloads (queued after every launch: a pageable copy blocks the host)
    for (int q = 0; q < nchunks; ++q) {
        const int d = devices[q], Sq = s_count(q), s0 = s_begin(q);
        ShardBufs& Bq = *B[q];
        cuda_check(cudaSetDevice(d), "cudaSetDevice");
        cudaStream_t st = Bq.stream;
        const std::size_t o = static_cast<std::size_t>(s0) * n, cells = static_cast<std::size_t>(Sq) * n;
        if (v_out)
            cuda_check(cudaMemcpyAsync(v_out + o, Bq.v_sm.get<double>(static_cast<std::size_t>(chunk) * n),
                                       cells * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "copy V");
        if (potentials_only) continue;
        if (succ_out)
            cuda_check(cudaMemcpyAsync(succ_out + o, Bq.succ.get<int>(cells), cells * sizeof(int), cudaMemcpyDeviceToHost, st),
                       "copy succ");
        if (center_out)
            cuda_check(cudaMemcpyAsync(center_out + o, Bq.center.get<int>(cells), cells * sizeof(int),
                                       cudaMemcpyDeviceToHost, st),
                       "copy center");
        cuda_check(cudaMemcpyAsync(ci_out + o, Bq.ci.get<int>(cells), cells * sizeof(int), cudaMemcpyDeviceToHost, st),
                   "copy cluster index");
        int* stage = pinned_counts_buf(Bq.nc_host, Bq.nc_host_cap, Sq);
        cuda_check(cudaMemcpyAsync(stage, Bq.nc.get<int>(Sq), Sq * sizeof(int), cudaMemcpyDeviceToHost, st),
                   "copy counts");
        if (intra_out)
            cuda_check(cudaMemcpyAsync(intra_out + s0, Bq.intra.get<long long>(Sq), Sq * sizeof(long long),
                                       cudaMemcpyDeviceToHost, st),
                       "copy intra counts");
    }
    for (int r = 0; r < shards; ++r) {
        cuda_check(cudaSetDevice(devices[r]), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(B[r]->stream), "multi-device sweep");
    }
    if (!potentials_only) {
        for (int q = 0; q < nchunks; ++q)
            if (*B[q]->err_host) fail(GQC_ECYCLE, "successor map contains a cycle");  // ggd.cpp:41
        for (int q = 0; q < nchunks; ++q) std::copy(B[q]->nc_host, B[q]->nc_host + s_count(q), nc_out + s_begin(q));
    }
}

// Devices of the host-buffer entry points: GQC_OPT_DEVICE .. + GQC_OPT_GPUS - 1.
static std::vector<int> option_devices() {
    std::vector<int> d(t_opt.gpus);
    const int count = visible_devices();
    for (int k = 0; k < t_opt.gpus; ++k) {
        d[k] = t_opt.device + k;
        if (d[k] >= count) fail(GQC_EINVAL, "GQC_OPT_GPUS exceeds the visible devices");
    }
    return d;
}

gqc_status gqc_cluster_sweep(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out,
                             int32_t* succ_out, int32_t* center_out, int32_t* cluster_index_out,
                             int32_t* num_clusters_out) {
    return gqc_cluster_sweep_intra(g, sigmas, n_sigma, v_out, succ_out, center_out, cluster_index_out,
                                   num_clusters_out, nullptr);
}

gqc_status gqc_cluster_sweep_intra(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out,
                                   int32_t* succ_out, int32_t* center_out, int32_t* cluster_index_out,
                                   int32_t* num_clusters_out, int64_t* intra_out) {
    return guarded([&] {
        if (t_opt.gpus > 1) {
            const std::vector<int> d = option_devices();
            sweep_multi_impl(g, sigmas, n_sigma, d.data(), static_cast<int>(d.size()), v_out, succ_out, center_out,
                             cluster_index_out, num_clusters_out, intra_out, false);
            return;
        }
        cluster_sweep_impl(g, sigmas, n_sigma, v_out, succ_out, center_out, cluster_index_out, num_clusters_out,
                           intra_out);
    });
}

gqc_status gqc_cluster_sweep_multi(const gqc_csr* g, const double* sigmas, int32_t n_sigma, const int32_t* devices,
                                   int32_t n_shards, double* v_out, int32_t* succ_out, int32_t* center_out,
                                   int32_t* cluster_index_out, int32_t* num_clusters_out, int64_t* intra_out) {
    return guarded([&] {
        if (n_shards == 1 && devices) {  // one shard: the single-device pipeline on that device
            if (devices[0] < 0 || devices[0] >= visible_devices()) fail(GQC_EINVAL, "device ordinal out of range");
            t_opt.device = devices[0];
            cluster_sweep_impl(g, sigmas, n_sigma, v_out, succ_out, center_out, cluster_index_out, num_clusters_out,
                               intra_out);
            return;
        }
        sweep_multi_impl(g, sigmas, n_sigma, devices, n_shards, v_out, succ_out, center_out, cluster_index_out,
                         num_clusters_out, intra_out, false);
    });
}

gqc_status gqc_potentials_multi(const gqc_csr* g, const double* sigmas, int32_t n_sigma, const int32_t* devices,
                                int32_t n_shards, double* v_out) {
    return guarded([&] {
        sweep_multi_impl(g, sigmas, n_sigma, devices, n_shards, v_out, nullptr, nullptr, nullptr, nullptr, nullptr, true);
    });
}

gqc_status gqc_build_csr(int32_t n, int64_t m, const gqc_edge* edges, int64_t* offsets, int32_t* nbr, double* w_out,
                         int64_t* nnz_out, int32_t* unit_out, int64_t* dup_out, int64_t dup_cap, int64_t* n_dup_out) {
    static_assert(sizeof(gqc_edge) == sizeof(GqcEdge), "edge layout");
    return guarded([&] {
        if (n < 1) fail(GQC_EINVAL, "graph needs at least one node");  // graph.cpp:28
        if (m < 0 || m >= (1ll << 32)) fail(GQC_EINVAL, "edge count out of range");
        if (!offsets || !nnz_out || (m > 0 && (!edges || !nbr))) fail(GQC_EINVAL, "null buffer");
        DeviceCtx& C = ctx();
        long long nnz = 0, first = -1;
        int unit = 1;
        std::vector<long long> conf;
        cuda_check(build_csr_device(n, m, reinterpret_cast<const GqcEdge*>(edges), offsets, nbr, w_out, &nnz,
                                    n_dup_out ? &conf : nullptr, &unit, &first, C.pool, C.stream),
                   "CSR build");
        if (first >= 0) {  // graph.cpp:33-39: the first offending edge, endpoint before weight
            if (first & 1) fail(GQC_EINVAL, "edge weight must be positive");
            fail(GQC_ERANGE, "edge endpoint out of range");
        }
        *nnz_out = nnz;
        if (unit_out) *unit_out = unit;
        if (n_dup_out) {
            if (!conf.empty() && conf.back() == -1) fail(GQC_ENOMEM, "too many conflicting duplicate edges");
            std::vector<std::pair<long long, long long>> pairs(conf.size() / 2);
            for (std::size_t j = 0; j < pairs.size(); ++j) pairs[j] = {conf[2 * j], conf[2 * j + 1]};
            std::sort(pairs.begin(), pairs.end());
            *n_dup_out = static_cast<int64_t>(pairs.size());
            for (std::size_t j = 0; j < pairs.size() && static_cast<int64_t>(j) < dup_cap; ++j) {
                dup_out[2 * j] = pairs[j].first;
                dup_out[2 * j + 1] = pairs[j].second;
            }
        }
    });
}

gqc_status gqc_row_shards(const gqc_csr* g, int32_t n_shards, int32_t* bounds) {
    return guarded([&] {
        check_csr_shape(g);
        if (n_shards < 1 || n_shards > kMaxShards) fail(GQC_EINVAL, "shard count must be in 1..32");
        if (!bounds) fail(GQC_EINVAL, "null output");
        if (g->offsets[0] != 0 || g->offsets[g->n] != g->nnz) fail(GQC_EINVAL, "CSR offsets do not match nnz");
        const std::vector<int> b = row_shards(g->offsets, g->n, n_shards, t_opt.kernel);
        std::copy(b.begin(), b.end(), bounds);
    });
}

gqc_status gqc_dev_potentials(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                              int32_t row_end, double* v_rows, void* stream) {
    return guarded([&] {
        check_sigmas(sigmas, n_sigma);
        check_csr_shape(g);
        if (row_begin < 0 || row_end > g->n || row_begin > row_end) fail(GQC_ERANGE, "row range out of range");
        if (!v_rows && row_end > row_begin) fail(GQC_EINVAL, "null output");
        DeviceCtx& C = ctx(static_cast<cudaStream_t>(stream), g->offsets);
        run_potentials(C, *g, sigmas, n_sigma, row_begin, row_end, v_rows, nullptr, static_cast<cudaStream_t>(stream));
    });
}

gqc_status gqc_dev_potentials_packed(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                                     int32_t row_end, double* v_out, int32_t chunk, int64_t chunk_stride,
                                     void* stream) {
    return guarded([&] {
        check_sigmas(sigmas, n_sigma);
        check_csr_shape(g);
        if (row_begin < 0 || row_end > g->n || row_begin > row_end) fail(GQC_ERANGE, "row range out of range");
        if (!v_out && row_end > row_begin) fail(GQC_EINVAL, "null output");
        if (chunk < 1) fail(GQC_EINVAL, "sigma chunk must be positive");
        const int chunks = (n_sigma + chunk - 1) / chunk;
        if (chunks > 1 && chunk_stride < static_cast<int64_t>(row_end - row_begin) * chunk)
            fail(GQC_EINVAL, "chunk stride smaller than one chunk");
        DeviceCtx& C = ctx(static_cast<cudaStream_t>(stream), g->offsets);
        run_potentials(C, *g, sigmas, n_sigma, row_begin, row_end, v_out, nullptr, static_cast<cudaStream_t>(stream),
                       nullptr, chunk, chunk_stride);
    });
}

gqc_status gqc_dev_potentials_peer(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                                   int32_t row_end, double* const* chunk_ptrs, int32_t n_chunks, int32_t chunk,
                                   void* stream) {
    return guarded([&] {
        check_sigmas(sigmas, n_sigma);
        check_csr_shape(g);
        if (row_begin < 0 || row_end > g->n || row_begin > row_end) fail(GQC_ERANGE, "row range out of range");
        if (chunk < 1) fail(GQC_EINVAL, "sigma chunk must be positive");
        if (n_chunks != (n_sigma + chunk - 1) / chunk || n_chunks > kMaxShards)
            fail(GQC_EINVAL, "chunk pointer count does not match the sigma chunks");
        if (!chunk_ptrs) fail(GQC_EINVAL, "null output");
        for (int q = 0; q < n_chunks; ++q)
            if (!chunk_ptrs[q] && row_end > row_begin) fail(GQC_EINVAL, "null output");
        DeviceCtx& C = ctx(static_cast<cudaStream_t>(stream), g->offsets);
        double* ptr[kMaxShards] = {};
        for (int q = 0; q < n_chunks; ++q) ptr[q] = chunk_ptrs[q];
        if (row_end > row_begin)
            run_potentials(C, *g, sigmas, n_sigma, row_begin, row_end, nullptr, nullptr,
                           static_cast<cudaStream_t>(stream), nullptr, chunk, 0, nullptr, ptr);
    });
}

gqc_status gqc_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
    return guarded([&] {
        if (!dev_ptr || !handle_out) fail(GQC_EINVAL, "null output");
        ctx();
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc");
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            cuda_check(e, "cudaIpcGetMemHandle");
        }
        static_assert(sizeof(h) == GQC_IPC_HANDLE_BYTES, "IPC handle size");
        std::memcpy(handle_out, &h, sizeof h);
        *dev_ptr = p;
    });
}

gqc_status gqc_ipc_open(const void* handle, void** dev_ptr) {
    return guarded([&] {
        if (!handle || !dev_ptr) fail(GQC_EINVAL, "null buffer");
        ctx();
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* p = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        *dev_ptr = p;
    });
}

gqc_status gqc_ipc_close(void* dev_ptr) {
    return guarded([&] {
        ctx();
        cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    });
}

gqc_status gqc_ipc_free(void* dev_ptr) {
    return guarded([&] {
        ctx();
        cuda_check(cudaFree(dev_ptr), "cudaFree");
    });
}

size_t gqc_dev_ggd_workspace(int32_t n, int32_t n_sigma) {
    if (n < 1 || n_sigma < 1) return 0;
    return labels_workspace_bytes(n, n_sigma);
}

gqc_status gqc_dev_ggd(const gqc_csr* g, const double* v, int32_t n_sigma, int32_t* succ, int32_t* center,
                       int32_t* cluster_index, int32_t* num_clusters, void* workspace, size_t workspace_bytes,
                       void* stream) {
    return guarded([&] {
        check_csr_shape(g);
        if (n_sigma < 1) fail(GQC_EINVAL, "sigma grid is empty");
        if (!v || !center || !cluster_index || !num_clusters || !workspace) fail(GQC_EINVAL, "null buffer");
        if (workspace_bytes < labels_workspace_bytes(g->n, n_sigma)) fail(GQC_EINVAL, "workspace too small");
        auto st = static_cast<cudaStream_t>(stream);
        DeviceCtx& C = ctx(st, g->offsets);
        int* s = succ ? succ : center;  // the chase runs in place on center
        ClassOrderScope order;
        make_class_order(C, *g, v, n_sigma, n_sigma, st, order);
        cuda_check(launch_successors(g->n, g->offsets, g->nbr, v, n_sigma, 0, n_sigma, 0, g->n, s, 1, g->n, g->nnz, C.pool,
                                     st, order.get(), light_row_sigmas_device(g->offsets, g->n, g->nnz, st)),
                   "successor kernel");
        cuda_check(launch_labels(g->n, n_sigma, s, center, cluster_index, num_clusters, workspace, workspace_bytes, st),
                   "label kernels");
    });
}

gqc_status gqc_dev_successors(const gqc_csr* g, const double* v, int32_t n_sigma, int32_t row_begin, int32_t row_end,
                              int32_t* succ_rows, void* stream) {
    return guarded([&] {
        check_csr_shape(g);
        if (n_sigma < 1) fail(GQC_EINVAL, "sigma grid is empty");
        if (row_begin < 0 || row_end > g->n || row_begin > row_end) fail(GQC_ERANGE, "row range out of range");
        if (!v || (!succ_rows && row_end > row_begin)) fail(GQC_EINVAL, "null buffer");
        auto st = static_cast<cudaStream_t>(stream);
        DeviceCtx& C = ctx(st, g->offsets);
        ClassOrderScope order;
        make_class_order(C, *g, v, n_sigma, n_sigma, st, order);
        cuda_check(launch_successors(g->n, g->offsets, g->nbr, v, n_sigma, 0, n_sigma, row_begin, row_end, succ_rows,
                                     n_sigma, 1, g->nnz, C.pool, st, order.get(),
                                     light_row_sigmas_device(g->offsets, g->n, g->nnz, st)),
                   "successor kernel");
    });
}

size_t gqc_dev_resolve_workspace(int32_t n, int32_t n_sigma) {
    if (n < 1 || n_sigma < 1) return 0;
    return labels_workspace_bytes(n, n_sigma);
}

gqc_status gqc_dev_resolve(int32_t n, int32_t n_sigma, const int32_t* succ_nm, int32_t* center, int32_t* cluster_index,
                           int32_t* num_clusters, void* workspace, size_t workspace_bytes, void* stream) {
    return guarded([&] {
        if (n < 1 || n_sigma < 1) fail(GQC_EINVAL, "empty input");
        if (!succ_nm || !center || !cluster_index || !num_clusters || !workspace) fail(GQC_EINVAL, "null buffer");
        if (workspace_bytes < labels_workspace_bytes(n, n_sigma)) fail(GQC_EINVAL, "workspace too small");
        auto st = static_cast<cudaStream_t>(stream);
        bind_device(st, succ_nm);
        cuda_check(launch_transpose_i32(succ_nm, n, n_sigma, center, st), "transpose");
        cuda_check(launch_labels(n, n_sigma, center, center, cluster_index, num_clusters, workspace, workspace_bytes, st),
                   "label kernels");
    });
}

gqc_status gqc_dev_transpose(const double* v_nm, int32_t n, int32_t n_sigma, double* v_sm, void* stream) {
    return guarded([&] {
        if (n < 0 || n_sigma < 1 || !v_nm || !v_sm) fail(GQC_EINVAL, "bad transpose arguments");
        bind_device(static_cast<cudaStream_t>(stream), v_nm);
        cuda_check(launch_transpose(v_nm, n, n_sigma, v_sm, stream), "transpose");
    });
}

}  // extern "C"
