// sm_100a kernels of the QC potential sweep and Graph Gradient Descent.
//
// Parity contract: the reference accumulates, for every
// row i, num += d2[j]*g[j] and den += g[j] strictly in ascending j in fp64
// (potential.cpp:30-35), and ties between equal-degree nodes are decided by
// the rounding noise of that order. No reduction tree or reassociation is
// allowed inside a row, so each (row, sigma) pair is one sequential chain
// here too, and every add is an explicit round-to-nearest __dadd_rn (the
// library is also built with -fmad=false).
//
// The row is a sequence of runs of identical terms: non-adjacent columns all
// add (W^2 e_W, e_W); the self column adds (0, 1); each neighbour adds
// (w^2 e, e). K1 (REPLAY) performs every add. K2 (FASTFWD) replaces a run of
// L identical adds by an exact closed form per binade of the partial sum
// (ff_chain below), which reproduces the sequential result bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>
#include <utility>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gqc_internal.h"

#ifndef GQC_CONST_SMEM
#define GQC_CONST_SMEM 1
#endif
#ifndef GQC_WALK2
#define GQC_WALK2 1
#endif
// GQC_WALK_EVENTS2=1: the batched walk advances both accumulators in one loop
#ifndef GQC_WALK_EVENTS2
#define GQC_WALK_EVENTS2 0
#endif

#ifndef GQC_LANE_OUT_SMEM
#define GQC_LANE_OUT_SMEM 1
#endif

namespace cg = cooperative_groups;

namespace gqc {
namespace {

constexpr int kBlock = 256;
#ifndef GQC_WARP_MIN_SIGMA
#define GQC_WARP_MIN_SIGMA 8
#endif
constexpr int kWarpKernelMinSigma = GQC_WARP_MIN_SIGMA;  // below this, thread-per-(row, sigma)
// 4 x 256 threads per SM (<= 64 registers): measured best on B200 (vs 3 or 5)
constexpr int kWarpKernelBlocksPerSM = 4;



#include "ff_chain.cuh"

using namespace gqc::ffc;

// K1: the dense in-order replay, two independent chains per thread.
__device__ __forceinline__ void replay(double& num, double& den, const double p, const double e, int L) {
    double a = num, b = den;
#pragma unroll 4
    for (int t = 0; t < L; ++t) {
        a = __dadd_rn(a, p);
        b = __dadd_rn(b, e);
    }
    num = a;
    den = b;
}

// A run of L identical (p, e) neighbour terms (consecutive columns with the
// same weight). Rare outside dense rows; kept out of line (by value, so the
// caller's chains stay in registers).
template <bool kFF>
__device__ __noinline__ double2 term_run_long(const double ns, const double ds, const double p, const double e,
                                              const int L) {
    if constexpr (kFF) {
        Chain a = make_chain(ns, p), b = make_chain(ds, e);
        ff_run(a, p, L);
        ff_run(b, e, L);
        return make_double2(a.s, b.s);
    } else {
        double a = ns, b = ds;
        replay(a, b, p, e, L);
        return make_double2(a, b);
    }
}

// Eigen 3.4 pexp_double restated with explicit IEEE roundings (no FMA): the
// same operation sequence as gqc::host_pexp (host_exp.cpp) and as one SSE2
// lane of the reference build. Used per entry for weighted graphs.
__device__ __noinline__ double pexp_dev(const double x0) {
    double x = fmax(fmin(x0, 709.784), -709.784);
    const double fx = floor(__dadd_rn(__dmul_rn(1.4426950408889634073599, x), 0.5));
    x = __dsub_rn(x, __dmul_rn(fx, 0.693145751953125));
    x = __dsub_rn(x, __dmul_rn(fx, 1.42860682030941723212e-6));
    const double x2 = __dmul_rn(x, x);
    double px = __dadd_rn(__dmul_rn(1.26177193074810590878e-4, x2), 3.02994407707441961300e-2);
    px = __dadd_rn(__dmul_rn(px, x2), 9.99999999999999999910e-1);
    px = __dmul_rn(px, x);
    double qx = __dadd_rn(__dmul_rn(3.00198505138664455042e-6, x2), 2.52448340349684104192e-3);
    qx = __dadd_rn(__dmul_rn(qx, x2), 2.27265548208155028766e-1);
    qx = __dadd_rn(__dmul_rn(qx, x2), 2.00000000000000000009e0);
    double r = __ddiv_rn(px, __dsub_rn(qx, px));
    r = __dadd_rn(__dmul_rn(2.0, r), 1.0);
    const int ei = static_cast<int>(fmin(fmax(fx, -2099.0), 2099.0));
    const int b = ei >> 2;
    const double c = __hiloint2double((b + 1023) << 20, 0);
    double out = __dmul_rn(__dmul_rn(__dmul_rn(r, c), c), c);
    out = __dmul_rn(out, __hiloint2double((ei - 3 * b + 1023) << 20, 0));
    return out > x0 ? out : x0;
}

// ---------------------------------------------------------------------------
// Prefix builder: one thread per (sigma, chain) records the pure trajectory of
// the non-adjacent constant from 0 (ff_chain.cuh, build_prefix). Layout per
// (sigma, chain) q = 2*s + {0 num, 1 den}: kPrefixCap entries of t / s0 / inc.
// ---------------------------------------------------------------------------
struct PrefixTable {
    int* t;
    double* s0;
    double* inc;
    int* count;
    int* t_end;
    double* s_end;
    // numerator of an isolated row (no neighbours): its own column adds 0,
    // so it is n - 1 pure adds of pW (iso_last, also the row n - 1 under a
    // tail) or, under an odd-n tail, n - 2 pure adds then the tail constant
    double* iso;
    double* iso_last;
};

// Longest-first dynamic row scheduling of the warp kernel: rows in
// descending-degree order (one radix sort per launch), handed out to warps
// through an atomic counter, so hub rows of skewed graphs start first and
// no warp idles while another still owns a backlog.
struct RowSched {
    const int* order;  // row ids, heaviest first
    int* counter;      // next position in `order`
    const int* limit;  // rows to take (device), or nullptr for the whole range
};

// Hub rows: a row so long that, walked by one warp sharing its scheduler with
// seven others, it would outlast the rest of the sweep (R-MAT's hub has ~10^5
// neighbours) gets an SM to itself: a companion launch on a side stream runs
// one warp per block with enough dynamic shared memory that no other block
// fits on that SM. The main launch skips those rows.
constexpr int kMaxHubs = 16;
constexpr int kHubSmemBytes = 196 * 1024;

// deg_mask: the polled upload's sort keys carry the slab in bits 24+ (see
// row_degree_kernel); only the degree bits are compared with the threshold.
__global__ void hub_split_kernel(const int* __restrict__ deg_sorted, int rows, long long threshold, int deg_mask,
                                 int* __restrict__ hub_count, int* __restrict__ main_counter,
                                 int* __restrict__ hub_counter) {
    int h = 0;
    while (h < kMaxHubs && h < rows && (deg_sorted[h] & deg_mask) > threshold) ++h;
    *hub_count = h;
    *main_counter = h;
    *hub_counter = 0;
}
constexpr int kRowsPerGrab = 2;
constexpr int kHeavyDegree = 256;  // GGD argmin: rows above this degree use a block each

// Sort keys of the longest-first schedule: the degree capped at 2^bits - 1
// (bits = 24 where the hub split compares degrees; 11 for the unit-weight
// fast-forward, whose order only needs "long rows first": 2 radix passes
// instead of 4), and under the polled upload the slab above it.
__global__ void row_degree_kernel(const long long* __restrict__ off, int row_begin, int rows, int* __restrict__ deg,
                                  int* __restrict__ id, const int* __restrict__ slab_flags, int b1, int b2, int b3,
                                  int bits) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= rows) return;
    const int i = row_begin + k;
    deg[k] = min(static_cast<int>(min(off[i + 1] - off[i], 0x7fffffffll)), (1 << bits) - 1);
    if (slab_flags) {  // polled upload: slab-major (earlier slabs first), heaviest first inside a slab
        const int slab = (i >= b1) + (i >= b2) + (i >= b3);
        deg[k] |= (3 - slab) << bits;
    }
    id[k] = i;
}

__global__ void prefix_kernel(const __grid_constant__ PotentialLaunch P, PrefixTable T) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= 2 * P.n_sigma) return;
    const SigmaConsts& c = P.c[q >> 1];
    const double cst = (q & 1) ? c.eW : c.pW;
    build_prefix(cst, P.n, T.t + q * kPrefixCap, T.s0 + q * kPrefixCap, T.inc + q * kPrefixCap, T.count + q,
                 T.t_end + q, T.s_end + q);
    if (q & 1) return;
    auto pure = [&](const int L) {  // L pure adds of pW from 0
        if (L <= 0) return 0.0;
        if (L < T.t_end[q])
            return prefix_value(T.t + q * kPrefixCap, T.s0 + q * kPrefixCap, T.inc + q * kPrefixCap, T.count[q], L);
        Chain ch = make_chain(T.s_end[q], cst);
        ff_run(ch, cst, L - T.t_end[q]);
        return ch.s;
    };
    T.iso_last[q >> 1] = pure(P.n - 1);
    T.iso[q >> 1] = P.tail ? __dadd_rn(pure(P.n - 2), c.pWt) : T.iso_last[q >> 1];
}

// Value of the first run (L pure adds from 0) for chain q, then the chain's
// binade cache is invalidated so the next run refreshes it.
__device__ __forceinline__ void first_run(Chain& ch, const double c, const PrefixTable& T, const int q, const int L) {
    const int t_end = T.t_end[q];
    if (L < t_end) {
        ch.s = prefix_value(T.t + q * kPrefixCap, T.s0 + q * kPrefixCap, T.inc + q * kPrefixCap, T.count[q], L);
    } else {
        ch.s = T.s_end[q];
        ff_run(ch, c, L - t_end);
    }
    ch.top = 0.0;
}

// ---------------------------------------------------------------------------
// Potential kernel: thread = (row, sigma), sigma fastest, so the lanes of a
// warp share one CSR row (broadcast loads) and write one contiguous node-major
// slice of V. Grid: ceil(rows * n_sigma / 256) blocks of 256 threads.
// Row walk: runs of non-adjacent columns between the ascending breakpoints
// (neighbours and the row itself); K2 takes the first run from the prefix
// table and every later run through the two-chain fast-forward.
// ---------------------------------------------------------------------------
// Thread-per-(row, sigma) launches of at least this many rows take their rows
// in descending-degree order (order[r] = row of slot r).
#ifndef GQC_SORT_ROWS_MIN
#define GQC_SORT_ROWS_MIN 4096
#endif
constexpr int kSortRowsMin = GQC_SORT_ROWS_MIN;

template <bool kFF, int kW>
__global__ void __launch_bounds__(kBlock) potential_kernel(const __grid_constant__ PotentialLaunch P,
                                                           const PrefixTable T, const int* __restrict__ order) {
    __shared__ double sc[kSigmaFields][kMaxSigmaPerLaunch];
    for (int idx = threadIdx.x; idx < kSigmaFields * kMaxSigmaPerLaunch; idx += blockDim.x) {
        const int ss = idx % kMaxSigmaPerLaunch, f = idx / kMaxSigmaPerLaunch;
        if (ss < P.n_sigma) sc[f][ss] = reinterpret_cast<const double*>(&P.c[ss])[f];
    }
    __syncthreads();

    const int S = P.n_sigma;
    const long long tid = static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x;
    const int s = static_cast<int>(tid % S);
    const long long r64 = tid / S;
    if (r64 >= P.row_end - P.row_begin) return;
    const int i = order ? __ldg(order + r64) : P.row_begin + static_cast<int>(r64);

    const double e1 = sc[4][s], p1 = sc[5][s];
    const int n = P.n;
    const bool tail = P.tail != 0;
    const long long kend = P.offsets[i + 1];
    long long k = P.offsets[i];
    const double pW = sc[3][s], eW = sc[2][s];
    Chain num = make_chain(0.0, pW), den = make_chain(0.0, eW);
    int pos = 0;
    bool self_pending = true;

    for (;;) {
        const int nb = (k < kend) ? __ldg(P.nbr + k) : n;
        int col, kind;  // kind: 0 end of row, 1 self, 2 neighbour
        if (self_pending && i < nb) {
            col = i;
            kind = 1;
        } else if (k < kend) {
            col = nb;
            kind = 2;
        } else {
            col = n;
            kind = 0;
        }
        // non-adjacent run over [pos, col); the first run never reaches the
        // tail column (it stops at or before the row's own column)
        const int L = col - pos;
        if (L > 0) {
            const bool at_end = tail && col == n;
            const int Lw = at_end ? L - 1 : L;
            if constexpr (kFF) {
                if (pos == 0) {
                    first_run(num, pW, T, 2 * s, Lw);
                    first_run(den, eW, T, 2 * s + 1, Lw);
                } else if (Lw > 0) {
                    ff_run2(num, pW, den, eW, Lw);
                }
            } else {
                replay(num.s, den.s, pW, eW, Lw);
            }
            if (at_end) {
                num.s = __dadd_rn(num.s, sc[7][s]);
                den.s = __dadd_rn(den.s, sc[6][s]);
            }
        }
        if (kind == 0) break;
        if (kind == 1) {  // self: d2 = 0, exp(-0) = 1 -> num += 0, den += 1
            den.s = __dadd_rn(den.s, 1.0);
            self_pending = false;
            pos = col + 1;
            continue;
        }
        // neighbour(s): coalesce consecutive columns with identical weight
        const bool at_tail = tail && col == n - 1;
        double wk = 1.0;
        if constexpr (kW != kUnit) wk = __ldg(P.w + k);
        long long kk = k + 1;
        int end = col + 1;
        if (!at_tail) {
            while (kk < kend) {
                const int nx = __ldg(P.nbr + kk);
                if (nx != end || (tail && end == n - 1)) break;
                if constexpr (kW != kUnit) {
                    if (__ldg(P.w + kk) != wk) break;
                }
                ++kk;
                ++end;
            }
        }
        double e, p;
        if constexpr (kW == kUnit) {
            e = at_tail ? sc[8][s] : e1;
            p = at_tail ? sc[9][s] : p1;
        } else {
            const double d2 = __dmul_rn(wk, wk);
            if constexpr (kW == kEntryTable) {
                e = __ldg(P.entry_exp + k * P.entry_ld + P.entry_col0 + s);
            } else {
                if (at_tail) {
                    // glibc value of this edge, stored in row n-1's entry order
                    long long lo = P.offsets[n - 1], hi = P.offsets[n];
                    const long long b0 = lo;
                    while (lo < hi) {
                        const long long mid = (lo + hi) >> 1;
                        if (__ldg(P.nbr + mid) < i) lo = mid + 1; else hi = mid;
                    }
                    e = __ldg(P.tail_exp + (lo - b0) * S + s);
                } else {
                    e = pexp_dev(__dmul_rn(sc[1][s], d2));
                }
            }
            p = __dmul_rn(d2, e);
        }
        const int cnt = end - col;
        if (cnt == 1) {
            num.s = __dadd_rn(num.s, p);
            den.s = __dadd_rn(den.s, e);
        } else {
            const double2 r = term_run_long<kFF>(num.s, den.s, p, e, cnt);
            num.s = r.x;
            den.s = r.y;
        }
        k = kk;
        pos = end;
    }
    *out_slot_ptr(P, i, s) = __dmul_rn(sc[0][s], __ddiv_rn(num.s, den.s));
    if (P.out_peer) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Warp-per-row potential kernel (n_sigma >= 8): lane s of a warp is sigma s of
// one row, so the whole walk (breakpoints, run lengths, neighbour terms) is
// warp-uniform and only the fast-forward arithmetic differs between lanes.
// The row's neighbour ids are loaded 32 at a time with one coalesced load and
// read back with shuffles; the prefix search keys live in shared memory.
// Persistent: each warp strides over rows.
// ---------------------------------------------------------------------------
constexpr int kPrefixStride = kPrefixCap + 1;
// Rows with at least this many neighbours take the batched walk (unit weights).
#ifndef GQC_BATCH_MIN_DEGREE
#define GQC_BATCH_MIN_DEGREE 32
#endif
constexpr int kBatchMinDegree = GQC_BATCH_MIN_DEGREE;  // padded: no bank conflicts across lanes
// Rows with at least this many neighbours walk the whole row at once (0: never).
#ifndef GQC_LONG_ROW
#define GQC_LONG_ROW 1024
#endif
constexpr int kLongRow = GQC_LONG_ROW;

// Polled CSR upload: lane 0 waits (acquire) until the copy stream has set
// the flag of row i's slab; a flag that never arrives sets *slab_err after
// ~5 s instead of hanging the GPU.
__device__ __noinline__ void wait_slab(const int* flags, const int b1, const int b2, const int b3, int* err,
                                       const int i, const unsigned long long timeout_ns) {
    const int slab = (i >= b1) + (i >= b2) + (i >= b3);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            int f;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flags + slab) : "memory");
            if (f || *static_cast<volatile int*>(err)) break;  // arrived, or another warp timed out
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                atomicExch(err, 1);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncwarp();
    __threadfence();
}

// CSR neighbour load of the warp kernel. Under the polled upload the copy
// engine is still writing nbr while the kernel runs, so those loads are
// coherent (ld.relaxed.gpu, ordered after the slab flag's acquire) instead of
// the read-only path (ld.global.nc requires data constant for the kernel's
// lifetime).
__device__ __forceinline__ int load_nbr(const PotentialLaunch& P, const long long k) {
    if (P.slab_flags) {
        int v;
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(P.nbr + k) : "memory");
        return v;
    }
    return __ldg(P.nbr + k);
}

// kLong: rows of >= kLongRow neighbours walk the whole row at once (used for
// row-range launches, i.e. shards of a multi-device sweep, where the longest
// row is the critical path; a whole-graph launch keeps the chunked walk, which
// measured faster for throughput and does not carry the extra code).
// kIso: isolated rows take a shortcut (their numerator is a per-sigma
// constant, only the denominator is walked); a separate instantiation,
// chosen from the degree sample, because the branch costs the other rows
// registers (LFR 4.451 -> 4.474 ms with it compiled in).
template <bool kFF, int kW, bool kLong = false, bool kIso = false>
__global__ void __launch_bounds__(kBlock, kWarpKernelBlocksPerSM) potential_warp_kernel(const __grid_constant__ PotentialLaunch P,
                                                                const PrefixTable T, const RowSched R) {
    __shared__ double sc[kSigmaFields][kMaxSigmaPerLaunch];
    __shared__ int pt[kFF ? 2 * kMaxSigmaPerLaunch * kPrefixStride : 1];
    __shared__ int pcount[2 * kMaxSigmaPerLaunch], pend[2 * kMaxSigmaPerLaunch];
    __shared__ int batch_cols[(kFF && kW == kUnit) ? kBlock : 1];  // per-warp neighbour chunk (batched rows)
    // pstart[q][e]: last prefix segment of chain q whose start t <= 2^e (the
    // segments double in length, so a lookup plus a step or two finds a run's)
    __shared__ unsigned char pstart[kFF ? 2 * kMaxSigmaPerLaunch : 1][32];
    const int S = P.n_sigma;
    for (int idx = threadIdx.x; idx < kSigmaFields * kMaxSigmaPerLaunch; idx += blockDim.x) {
        const int ss = idx % kMaxSigmaPerLaunch, f = idx / kMaxSigmaPerLaunch;
        if (ss < S) sc[f][ss] = reinterpret_cast<const double*>(&P.c[ss])[f];
    }
    if constexpr (kFF) {
        for (int idx = threadIdx.x; idx < 2 * S * kPrefixCap; idx += blockDim.x) {
            const int q = idx / kPrefixCap, j = idx % kPrefixCap;
            pt[q * kPrefixStride + j] = T.t[idx];
        }
        for (int q = threadIdx.x; q < 2 * S; q += blockDim.x) {
            pcount[q] = T.count[q];
            pend[q] = T.t_end[q];
        }
        for (int idx = threadIdx.x; idx < 2 * S * 32; idx += blockDim.x) {
            const int q = idx >> 5, e = idx & 31;
            const long long lim = 1ll << e;
            int k = 0;
            const int cnt = T.count[q];
            while (k + 1 < cnt && T.t[q * kPrefixCap + k + 1] <= lim) ++k;
            pstart[q][e] = static_cast<unsigned char>(k);
        }
    }
    __syncthreads();

    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int s = min(lane, S - 1);  // lanes >= S shadow the last sigma (uniform walk)
#if GQC_CONST_SMEM
    // per-sigma constants re-read from shared memory at each use (volatile:
    // not hoisted into registers; the unit kernel is register-bound)
    const volatile double* vsc = &sc[0][0];
#define pW (vsc[3 * kMaxSigmaPerLaunch + s])
#define eW (vsc[2 * kMaxSigmaPerLaunch + s])
#define e1 (vsc[4 * kMaxSigmaPerLaunch + s])
#define p1 (vsc[5 * kMaxSigmaPerLaunch + s])
#else
    const double pW = sc[3][s], eW = sc[2][s], e1 = sc[4][s], p1 = sc[5][s];
#endif
    const int tie_num = tie_binade(pW), tie_den = tie_binade(eW);
    const int n = P.n;
    const bool tail = P.tail != 0;
    // W run of L columns starting at column pos (the first run, pos == 0,
    // comes from the prefix table).
    auto w_run = [&](Chain& num, Chain& den, const int pos, const int L) {
        if (L <= 0) return;
        if constexpr (kFF) {
            if (pos == 0) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int q = 2 * s + c;
                    Chain& ch = c ? den : num;
                    if (L < pend[q]) {
                        const int* tq = pt + q * kPrefixStride;
                        int lo = pstart[q][31 - __clz(L)];  // t[lo] <= 2^floor(log2 L) <= L
                        const int last = pcount[q] - 1;
                        while (lo < last && tq[lo + 1] <= L) ++lo;
                        ch.s = __fma_rn(static_cast<double>(L - tq[lo]), T.inc[q * kPrefixCap + lo],
                                        T.s0[q * kPrefixCap + lo]);
                    } else {
                        ch.s = T.s_end[q];
                        ff_run(ch, c ? eW : pW, L - pend[q]);
                    }
                    ch.top = 0.0;
                }
            } else {
#if GQC_WALK2
                ff_walk2(num, pW, den, eW, L);
#else
                ff_run2(num, pW, den, eW, L);
#endif
            }
        } else {
            replay(num.s, den.s, pW, eW, L);
        }
    };

#if GQC_LANE_OUT_SMEM
    __shared__ double* lane_out_s[32];
    if (threadIdx.x < 32) lane_out_s[threadIdx.x] = out_slot_ptr(P, P.row_begin, min(static_cast<int>(threadIdx.x), S - 1));
    __syncthreads();
#define lane_out (lane_out_s[lane])
#else
    double* const lane_out = out_slot_ptr(P, P.row_begin, s);  // this lane's sigma slot of row_begin
#endif
    const int nrows = R.limit ? *R.limit : P.row_end - P.row_begin;
    int grab = 0, left = 0;
    for (;;) {
        if (left == 0) {  // next batch of rows, heaviest first
            const int take = R.limit ? 1 : kRowsPerGrab;  // hub rows: one per warp
            int g0 = 0;
            if (lane == 0) g0 = atomicAdd(R.counter, take);
            grab = __shfl_sync(kFull, g0, 0);
            if (grab >= nrows) break;
            left = min(take, nrows - grab);
        }
        const int i = R.order[grab];
        ++grab;
        --left;
        if (P.slab_flags)
            wait_slab(P.slab_flags, P.slab_bound[1], P.slab_bound[2], P.slab_bound[3], P.slab_err, i,
                      static_cast<unsigned long long>(P.slab_timeout_ns));
        const long long kbeg = P.offsets[i], kend = P.offsets[i + 1];
        Chain num, den;
        num.s = 0.0; num.top = 0.0; num.inc = 0.0; num.f_tie = tie_num; num.flags = 0;
        den.s = 0.0; den.top = 0.0; den.inc = 0.0; den.f_tie = tie_den; den.flags = 0;
        if constexpr (kFF && kW == kUnit && kIso) {
            if (kbeg == kend) {  // isolated row: the numerator is a per-sigma constant
                if (i > 0) w_run(num, den, 0, i);  // (the numerator's prefix is unused)
                den.s = __dadd_rn(den.s, 1.0);
                const int L = n - 1 - i;  // columns after the row's own
                if (L > 0) {
                    den.top = 0.0;
                    if (tail) {
                        ff_run(den, eW, L - 1);
                        den.s = __dadd_rn(den.s, sc[6][s]);
                    } else {
                        ff_run(den, eW, L);
                    }
                }
                const double nv = (tail && i == n - 1) ? T.iso_last[s] : T.iso[s];
                if (lane < S)
                    lane_out[static_cast<long long>(i - P.row_begin) * P.out_ld] =
                        __dmul_rn(sc[0][s], __ddiv_rn(nv, den.s));
                continue;
            }
        }
        int pos = 0;              // first column not yet added
        bool self_pending = true;
        // one neighbour event: the W run up to col (and the row's own column if
        // it comes first), then the neighbour term of CSR entry k (weight wk)
        auto event = [&](const int col, const long long k, const double wk) {
            if (self_pending && i < col) {  // the row's own column precedes this neighbour
                w_run(num, den, pos, i - pos);
                den.s = __dadd_rn(den.s, 1.0);  // self: num += 0, den += 1
                pos = i + 1;
                self_pending = false;
            }
            w_run(num, den, pos, col - pos);
            const bool at_tail = tail && col == n - 1;
            double e, p;
            if constexpr (kW == kUnit) {
                e = at_tail ? sc[8][s] : e1;
                p = at_tail ? sc[9][s] : p1;
            } else {
                const double d2 = __dmul_rn(wk, wk);
                if constexpr (kW == kEntryTable) {
                    e = __ldg(P.entry_exp + k * P.entry_ld + P.entry_col0 + s);
                } else {
                    if (at_tail) {  // glibc value, stored in row n-1's entry order
                        long long lo = P.offsets[n - 1], hi = P.offsets[n];
                        const long long b0 = lo;
                        while (lo < hi) {
                            const long long mid = (lo + hi) >> 1;
                            if (__ldg(P.nbr + mid) < i) lo = mid + 1;
                            else hi = mid;
                        }
                        e = __ldg(P.tail_exp + (lo - b0) * S + s);
                    } else {
                        e = pexp_dev(__dmul_rn(sc[1][s], d2));
                    }
                }
                p = __dmul_rn(d2, e);
            }
            num.s = __dadd_rn(num.s, p);
            den.s = __dadd_rn(den.s, e);
            pos = col + 1;
        };
        bool batched = false;
        if constexpr (kFF && kW == kUnit) batched = kend - kbeg >= kBatchMinDegree;
        if (batched) {
            // High-degree rows: each 32-neighbour chunk is staged in shared
            // memory and every accumulator walks it with walk_events (batched
            // exact in-binade jumps, ff_chain.cuh). The row's first event
            // (prefix-table run), its own column and a tail neighbour (column
            // n-1 of an odd-N graph) keep the per-event path.
            int* cols = batch_cols + (threadIdx.x >> 5) * 32;
            const struct {
                const int* c;
                __device__ int operator()(int q) const { return c[q]; }
            } colf{cols};
            const int tie_p1 = tie_binade(p1), tie_e1 = tie_binade(e1);
            auto walk = [&](const int j0, const int j1) {
#if GQC_WALK_EVENTS2
                walk_events2(num.s, pW, p1, tie_num, tie_p1, den.s, eW, e1, tie_den, tie_e1, colf, j0, j1, pos);
#else
                num.s = walk_events(num.s, pW, p1, tie_num, tie_p1, colf, j0, j1, pos);
                den.s = walk_events(den.s, eW, e1, tie_den, tie_e1, colf, j0, j1, pos);
#endif
                num.top = 0.0;  // the chains' binade caches are stale now
                den.top = 0.0;
                pos = cols[j1 - 1] + 1;
            };
            if constexpr (kLong) if (kLongRow > 0 && kend - kbeg >= kLongRow) {
                // Long rows (R-MAT's hubs): one walk over the whole row, its
                // binary searches reading the CSR row directly (cached), so a
                // row costs O(crossings x log deg) instead of one staged
                // 32-event chunk after another — a hub of 10^5 neighbours was
                // a ~3-4 ms sequential chain for its warp, the critical path of
                // a sharded R-MAT sweep.
                const int deg = static_cast<int>(kend - kbeg);
                const struct {
                    const PotentialLaunch* P;
                    long long b;
                    __device__ int operator()(int q) const { return load_nbr(*P, b + q); }
                } colg{&P, kbeg};
                auto walkg = [&](const int j0, const int j1) {
                    num.s = walk_events(num.s, pW, p1, tie_num, tie_p1, colg, j0, j1, pos);
                    den.s = walk_events(den.s, eW, e1, tie_den, tie_e1, colg, j0, j1, pos);
                    num.top = 0.0;
                    den.top = 0.0;
                    pos = colg(j1 - 1) + 1;
                };
                const int jend = (tail && colg(deg - 1) == n - 1) ? deg - 1 : deg;
                int before_self = 0;  // neighbours below the row's own column
                {
                    int hi = deg;
                    while (before_self < hi) {
                        const int mid = (before_self + hi) >> 1;
                        if (colg(mid) < i) before_self = mid + 1;
                        else hi = mid;
                    }
                }
                int j = 0;
                while (j < deg) {  // warp-uniform
                    if (pos == 0 || j >= jend) {  // first event of the row, or the tail neighbour
                        event(colg(j), kbeg + j, 1.0);
                        ++j;
                        continue;
                    }
                    int r = jend;
                    if (self_pending) r = min(max(before_self, j), jend);
                    if (r > j) {
                        walkg(j, r);
                        j = r;
                    }
                    if (self_pending && j < jend) {
                        w_run(num, den, pos, i - pos);
                        den.s = __dadd_rn(den.s, 1.0);
                        pos = i + 1;
                        self_pending = false;
                    }
                }
            }
            for (long long base = kbeg; base < kend && !(kLong && kLongRow > 0 && kend - kbeg >= kLongRow);
                 base += 32) {
                const int cnt = static_cast<int>(min(32ll, kend - base));
                const int my = lane < cnt ? load_nbr(P, base + lane) : n;
                __syncwarp();
                cols[lane] = my;
                __syncwarp();
                const int jend = (tail && cols[cnt - 1] == n - 1) ? cnt - 1 : cnt;
                const int before_self = __popc(__ballot_sync(kFull, lane < cnt && my < i));
                int j = 0;
                while (j < cnt) {  // warp-uniform
                    if (pos == 0 || j >= jend) {  // first event of the row, or the tail neighbour
                        event(cols[j], base + j, 1.0);
                        ++j;
                        continue;
                    }
                    int r = jend;
                    if (self_pending) r = min(max(before_self, j), jend);
                    if (r > j) {
                        walk(j, r);
                        j = r;
                    }
                    if (self_pending && j < jend) {  // the row's own column comes before event j
                        w_run(num, den, pos, i - pos);
                        den.s = __dadd_rn(den.s, 1.0);
                        pos = i + 1;
                        self_pending = false;
                    }
                }
            }
        } else {
            // neighbours in chunks of 32: one coalesced load, then shuffles
            for (long long base = kbeg; base < kend; base += 32) {
                const int cnt = static_cast<int>(min(32ll, kend - base));
                const int my = lane < cnt ? load_nbr(P, base + lane) : n;
                double myw = 1.0;
                if constexpr (kW != kUnit) myw = lane < cnt ? __ldg(P.w + base + lane) : 1.0;
                for (int j = 0; j < cnt; ++j) {
                    const int col = __shfl_sync(kFull, my, j);
                    double wk = 1.0;
                    if constexpr (kW != kUnit) wk = __shfl_sync(kFull, myw, j);
                    event(col, base + j, wk);
                }
            }
        }
        if (self_pending) {
            w_run(num, den, pos, i - pos);
            den.s = __dadd_rn(den.s, 1.0);
            pos = i + 1;
        }
        // final run [pos, n); the Eigen scalar tail column n-1 uses glibc constants
        const int L = n - pos;
        if (L > 0) {
            if (tail) {
                w_run(num, den, pos, L - 1);
                num.s = __dadd_rn(num.s, sc[7][s]);
                den.s = __dadd_rn(den.s, sc[6][s]);
            } else {
                w_run(num, den, pos, L);
            }
        }
        if (lane < S)
            lane_out[static_cast<long long>(i - P.row_begin) * P.out_ld] =
                __dmul_rn(sc[0][s], __ddiv_rn(num.s, den.s));
    }
    // peer / IPC outputs: the stores are performed system-wide before the
    // kernel is seen complete by the next operation in stream order
    if (P.out_peer) __threadfence_system();
}
#undef pW
#undef eW
#undef e1
#undef p1
#undef lane_out

// ---------------------------------------------------------------------------
// K3: successor = lexicographic (v, id) argmin over the closed neighbourhood
// (ggd.cpp:7-24). Thread = (row, sigma), sigma fastest: a neighbour's
// potentials for all sigmas are one contiguous node-major line.
// ---------------------------------------------------------------------------
// Output addressing of the GGD argmin: element (row r of the range, sigma q of
// the chunk) is written at out[r * out_row + q * out_col] (sigma-major:
// out_row = 1, out_col = n; node-major row shard: out_row = ld, out_col = 1).
struct SuccOut {
    int* out;
    long long out_row, out_col;
};

#ifndef GQC_SUCC_UNROLL
#define GQC_SUCC_UNROLL 4
#endif
#ifndef GQC_HEAVY_UNROLL
#define GQC_HEAVY_UNROLL 4
#endif
constexpr int kSuccUnroll = GQC_SUCC_UNROLL;    // gathers in flight per thread (light rows)
#ifndef GQC_SUCC_SUB
#define GQC_SUCC_SUB 32
#endif
constexpr int kSuccSub = GQC_SUCC_SUB;  // sigmas per light-row argmin launch (L2-resident V slice)
#ifndef GQC_TINY_DEGREE
#define GQC_TINY_DEGREE 0
#endif
constexpr int kTinyDegree = GQC_TINY_DEGREE;  // light rows up to this degree: 16-sigma launches
constexpr int kHeavyUnroll = GQC_HEAVY_UNROLL;  // gathers in flight per warp (heavy rows)

__device__ __forceinline__ bool lex_less(double va, int ia, double vb, int ib) {
    return va < vb || (va == vb && ia < ib);
}

// Rows of degree in [deg_lo, deg_hi] only (heavy rows: successors_heavy_kernel).
__global__ void __launch_bounds__(kBlock) successors_kernel(const long long* __restrict__ off,
                                                            const int* __restrict__ nbr,
                                                            const double* __restrict__ v, int ld, int s0, int Sc,
                                                            int row_begin, int rows, SuccOut O, int deg_lo,
                                                            int deg_hi) {
    // rows * Sc < 2^31 (launch_successors checks): 32-bit index math
    const unsigned tid = blockIdx.x * static_cast<unsigned>(kBlock) + threadIdx.x;
    const unsigned r = tid / static_cast<unsigned>(Sc);
    const int q = static_cast<int>(tid - r * static_cast<unsigned>(Sc));
    if (r >= static_cast<unsigned>(rows)) return;
    const int s = s0 + q;
    const int i = row_begin + static_cast<int>(r);
    long long k = off[i];
    const long long kend = off[i + 1];
    if (kend - k > deg_hi || kend - k < deg_lo) return;
    double vb = __ldg(v + static_cast<long long>(i) * ld + s);  // an isolated row keeps best = i
    int best = i;
    // kSuccUnroll independent gathers in flight, compared in ascending k
    for (; k + kSuccUnroll <= kend; k += kSuccUnroll) {
        int j[kSuccUnroll];
        double vj[kSuccUnroll];
#pragma unroll
        for (int u = 0; u < kSuccUnroll; ++u) j[u] = __ldg(nbr + k + u);
#pragma unroll
        for (int u = 0; u < kSuccUnroll; ++u) vj[u] = __ldg(v + static_cast<long long>(j[u]) * ld + s);
#pragma unroll
        for (int u = 0; u < kSuccUnroll; ++u)
            if (vj[u] < vb || (vj[u] == vb && j[u] < best)) {
                best = j[u];
                vb = vj[u];
            }
    }
    for (; k < kend; ++k) {
        const int j = __ldg(nbr + k);
        const double vj = __ldg(v + static_cast<long long>(j) * ld + s);
        if (vj < vb || (vj == vb && j < best)) {
            best = j;
            vb = vj;
        }
    }
    O.out[static_cast<long long>(r) * O.out_row + q * O.out_col] = best;
}

// Tiny rows (at most kTinyDegree neighbours, listed by mark_heavy_kernel):
// a half-warp per row, each thread two sigmas (q and q + 16), so a warp
// keeps two rows' gathers in flight where one tiny row per warp would leave
// the memory system idle (R-MAT's 1-4-neighbour rows). Grid-stride over the
// list; same lexicographic (v, id) argmin (ggd.cpp:17-19).
__global__ void __launch_bounds__(kBlock) successors_tiny_kernel(const long long* __restrict__ off,
                                                                 const int* __restrict__ nbr,
                                                                 const double* __restrict__ v, int ld, int s0, int Sc,
                                                                 int row_begin, const int* __restrict__ tiny,
                                                                 const int* __restrict__ counts, SuccOut O) {
    const int n_t = counts[3];
    const int h = threadIdx.x & 15;
    const long long step = (static_cast<long long>(gridDim.x) * blockDim.x) >> 4;
    for (long long t = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 4; t < n_t; t += step) {
        const int i = __ldg(tiny + t);
        const long long kb = off[i], ke = off[i + 1];
        const int qa = h, qb = h + 16;
        const bool hb = qb < Sc;
        if (qa >= Sc) continue;
        const double* vi = v + static_cast<long long>(i) * ld + s0;
        double va = __ldg(vi + qa), vb = hb ? __ldg(vi + qb) : 0.0;
        int ba = i, bb = i;
        for (long long k = kb; k < ke; ++k) {
            const int j = __ldg(nbr + k);
            const double* vj = v + static_cast<long long>(j) * ld + s0;
            const double xa = __ldg(vj + qa);
            const double xb = hb ? __ldg(vj + qb) : 0.0;
            if (lex_less(xa, j, va, ba)) {
                va = xa;
                ba = j;
            }
            if (hb && lex_less(xb, j, vb, bb)) {
                vb = xb;
                bb = j;
            }
        }
        O.out[static_cast<long long>(i - row_begin) * O.out_row + qa * O.out_col] = ba;
        if (hb) O.out[static_cast<long long>(i - row_begin) * O.out_row + qb * O.out_col] = bb;
    }
}

// Degree-class fast path of K3 (ClassOrder verified by launch_class_order):
// a node of a better degree class beats every node of a worse one, so the
// lexicographic (v, id) minimum of a closed neighbourhood lies in its best
// class. Warp per light row: lanes take neighbour slots for the class phase
// (ids and class ids for up to kHeavyDegree neighbours in one round of
// loads, warp min / max), then lanes are sigmas and only the best-class
// candidates' potentials are gathered (one 256 B line each). Per row that is
// ~4 dependent memory levels instead of one gather level per neighbour.
// Sigmas without a verified order (dir 0) scan every neighbour.
__global__ void __launch_bounds__(kBlock) successors_class_kernel(const long long* __restrict__ off,
                                                                  const int* __restrict__ nbr,
                                                                  const double* __restrict__ v, int ld, int s0,
                                                                  int Sc, int row_begin, int rows, SuccOut O,
                                                                  ClassOrder co) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr int kChunks = kHeavyDegree / 32;
    const int lane = threadIdx.x & 31;
    const int r = static_cast<int>((blockIdx.x * static_cast<unsigned>(kBlock) + threadIdx.x) >> 5);
    if (r >= rows) return;
    const int i = row_begin + r;
    const long long kb = off[i], ke = off[i + 1];
    if (ke - kb > kHeavyDegree) return;  // heavy rows: successors_heavy_kernel
    const int s = s0 + min(lane, Sc - 1);
    const int dir = __ldg(co.dir + s);
    const int ci = __ldg(co.cls + i);
    double vb = __ldg(v + static_cast<long long>(i) * ld + s);
    int jr[kChunks], cr[kChunks];
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
        const long long k = kb + 32 * q + lane;
        jr[q] = k < ke ? __ldg(nbr + k) : -1;
    }
#pragma unroll
    for (int q = 0; q < kChunks; ++q) cr[q] = jr[q] >= 0 ? __ldg(co.cls + jr[q]) : ci;
    int cmin = ci, cmax = ci;
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
        cmin = min(cmin, cr[q]);
        cmax = max(cmax, cr[q]);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        cmin = min(cmin, __shfl_xor_sync(kFull, cmin, d));
        cmax = max(cmax, __shfl_xor_sync(kFull, cmax, d));
    }
    const int bc = dir > 0 ? cmin : cmax;
    int best = i;
    if (dir != 0 && ci != bc) {
        best = 0x7fffffff;
        vb = __longlong_as_double(0x7ff0000000000000ll);
    }
#pragma unroll
    for (int q = 0; q < kChunks; ++q) {
        if (kb + 32 * q >= ke) break;  // warp-uniform
        const bool valid = jr[q] >= 0;
        const unsigned m_lo = __ballot_sync(kFull, valid && cr[q] == cmin);
        const unsigned m_hi = __ballot_sync(kFull, valid && cr[q] == cmax);
        const unsigned m_all = __ballot_sync(kFull, valid);
        const unsigned mine = dir > 0 ? m_lo : (dir < 0 ? m_hi : m_all);
        unsigned u = __reduce_or_sync(kFull, mine);
        while (u) {
            const int t = __ffs(u) - 1;
            u &= u - 1;
            const int j = __shfl_sync(kFull, jr[q], t);
            if ((mine >> t) & 1u) {
                const double vj = __ldg(v + static_cast<long long>(j) * ld + s);
                if (lex_less(vj, j, vb, best)) {
                    best = j;
                    vb = vj;
                }
            }
        }
    }
    if (lane < Sc) O.out[static_cast<long long>(r) * O.out_row + lane * O.out_col] = best;
}

// Heavy rows (degree > kHeavyDegree, e.g. R-MAT hubs with ~10^5 neighbours)
// are cut into segments of at most kHeavySegment neighbours by a marking
// pass and every segment is reduced by one block: the lexicographic (v, id)
// minimum is a total-order minimum (potentials are never NaN: den >= 1), so
// partial minima combine in any order to the same successor, and a hub no
// longer serialises on one block. Single-segment rows write their successor
// directly; longer rows write per-segment partials that a warp per row
// combines.
constexpr int kHeavySegment = 1024;

struct HeavyItem {
    int row, seg, slot;  // slot: partial-minimum slot, -1 for single-segment rows
};
struct HeavyRow {
    int row, slot0, nseg;
};

// Also lists the tiny rows (at most kTinyDegree neighbours, counts[3]) for
// successors_tiny_kernel; list order does not matter (rows are independent).
__global__ void mark_heavy_kernel(const long long* __restrict__ off, int row_begin, int rows,
                                  HeavyItem* __restrict__ items, int* __restrict__ counts, HeavyRow* __restrict__ multi,
                                  int* __restrict__ tiny) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = row_begin + r;
    const long long deg = r < rows ? off[i + 1] - off[i] : kHeavyDegree + 1;
    if (tiny) {  // warp-aggregated append
        const bool t = r < rows && deg <= kTinyDegree;
        const unsigned m = __ballot_sync(0xffffffffu, t);
        int base = 0;
        if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(&counts[3], __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (t) tiny[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1))] = i;
    }
    if (r >= rows || deg <= kHeavyDegree) return;
    const int nseg = static_cast<int>((deg + kHeavySegment - 1) / kHeavySegment);
    const int base = atomicAdd(&counts[0], nseg);
    int slot0 = -1;
    if (nseg > 1) {
        slot0 = atomicAdd(&counts[1], nseg);
        multi[atomicAdd(&counts[2], 1)] = HeavyRow{i, slot0, nseg};
    }
    for (int q = 0; q < nseg; ++q) items[base + q] = HeavyItem{i, q, nseg > 1 ? slot0 + q : -1};
}

__global__ void __launch_bounds__(kBlock) successors_heavy_kernel(const long long* __restrict__ off,
                                                                  const int* __restrict__ nbr,
                                                                  const double* __restrict__ v, int ld, int s0, int Sc,
                                                                  int row_begin, const HeavyItem* __restrict__ items,
                                                                  const int* __restrict__ counts,
                                                                  double* __restrict__ part_v, int* __restrict__ part_i,
                                                                  SuccOut O) {
    // one block per segment: lane = sigma, the 8 warps split the segment
    // (each neighbour's potentials are one coalesced node-major line), then
    // the per-warp minima are combined per sigma in shared memory
    constexpr int kWarps = kBlock / 32;
    __shared__ double sv[kWarps][32];
    __shared__ int si[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = s0 + min(lane, Sc - 1);
    const int total = counts[0];
    for (int h = blockIdx.x; h < total; h += gridDim.x) {
        const HeavyItem it = items[h];
        const int i = it.row;
        const long long kb = off[i] + static_cast<long long>(it.seg) * kHeavySegment;
        const long long kend = min(off[i + 1], kb + kHeavySegment);
        double vb = __longlong_as_double(0x7ff0000000000000ll);  // +inf: any neighbour beats it
        int best = 0x7fffffff;
        if (it.seg == 0) {  // the row itself is the initial candidate (ggd.cpp:15)
            vb = __ldg(v + static_cast<long long>(i) * ld + s);
            best = i;
        }
        long long k = kb + warp;
        for (; k + (kHeavyUnroll - 1) * kWarps < kend; k += kHeavyUnroll * kWarps) {  // gathers in flight per warp
            int j[kHeavyUnroll];
            double vj[kHeavyUnroll];
#pragma unroll
            for (int u = 0; u < kHeavyUnroll; ++u) j[u] = __ldg(nbr + k + u * kWarps);
#pragma unroll
            for (int u = 0; u < kHeavyUnroll; ++u) vj[u] = __ldg(v + static_cast<long long>(j[u]) * ld + s);
#pragma unroll
            for (int u = 0; u < kHeavyUnroll; ++u)
                if (lex_less(vj[u], j[u], vb, best)) {
                    vb = vj[u];
                    best = j[u];
                }
        }
        for (; k < kend; k += kWarps) {
            const int j = __ldg(nbr + k);
            const double vj = __ldg(v + static_cast<long long>(j) * ld + s);
            if (lex_less(vj, j, vb, best)) {
                vb = vj;
                best = j;
            }
        }
        sv[warp][lane] = vb;
        si[warp][lane] = best;
        __syncthreads();
        if (warp == 0) {
            for (int w = 1; w < kWarps; ++w)
                if (lex_less(sv[w][lane], si[w][lane], vb, best)) {
                    vb = sv[w][lane];
                    best = si[w][lane];
                }
            if (it.slot < 0) {
                if (lane < Sc) O.out[static_cast<long long>(i - row_begin) * O.out_row + lane * O.out_col] = best;
            } else {
                part_v[static_cast<long long>(it.slot) * 32 + lane] = vb;
                part_i[static_cast<long long>(it.slot) * 32 + lane] = best;
            }
        }
        __syncthreads();
    }
}

// Successor of every multi-segment heavy row from its segments' partial minima
// (warp per row, lane = sigma).
__global__ void __launch_bounds__(kBlock) successors_combine_kernel(const HeavyRow* __restrict__ multi,
                                                                    const int* __restrict__ counts,
                                                                    const double* __restrict__ part_v,
                                                                    const int* __restrict__ part_i, int Sc,
                                                                    int row_begin, SuccOut O) {
    const int lane = threadIdx.x & 31;
    const int nrows = counts[2];
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows; w += (gridDim.x * blockDim.x) >> 5) {
        const HeavyRow r = multi[w];
        double vb = part_v[static_cast<long long>(r.slot0) * 32 + lane];
        int best = part_i[static_cast<long long>(r.slot0) * 32 + lane];
        for (int q = 1; q < r.nseg; ++q) {
            const double vq = part_v[static_cast<long long>(r.slot0 + q) * 32 + lane];
            const int iq = part_i[static_cast<long long>(r.slot0 + q) * 32 + lane];
            if (lex_less(vq, iq, vb, best)) {
                vb = vq;
                best = iq;
            }
        }
        if (lane < Sc) O.out[static_cast<long long>(r.row - row_begin) * O.out_row + lane * O.out_col] = best;
    }
}

// int32 node-major [n][S] -> sigma-major [S][n] (successor shards gathered
// node-major across ranks are chased sigma-major).
__global__ void transpose_i32_kernel(const int* __restrict__ in, int n, int S, int* __restrict__ out) {
    __shared__ int tile[32][33];
    const int i0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, s = s0 + threadIdx.x;
        if (i < n && s < S) tile[r][threadIdx.x] = in[static_cast<long long>(i) * S + s];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int s = s0 + r, i = i0 + threadIdx.x;
        if (i < n && s < S) out[static_cast<long long>(s) * n + i] = tile[threadIdx.x][r];
    }
}

// K4/K5: successor chase and labels (ggd.cpp:26-57).
// roots_kernel reads succ once: it copies it into center[] (unless in place)
// and writes, per sigma, a bitmap of the roots (succ[i] == i: every root is
// known before any chasing) with one 32-bit word per 32 nodes and the word's
// popcount; one exclusive scan over the popcounts then gives every root its
// rank among the ascending roots of its sigma, rank(x) = pre[x/32] -
// pre[0] + popc(word[x/32] below bit x%32), which is cluster_index
// (ggd.cpp:48-55), and the scan's per-sigma totals are the cluster counts.
// The roots' entries of center[] are then replaced by -1 - rank, so
// chase_kernel, following pointers through center[] (which other threads
// overwrite with root ids as they finish: any value read is an ancestor, so
// the result is exact; finished neighbours shorten the walk), reads its
// label at the end of the walk with no further lookup and writes center and
// cluster_index together; the root entries are restored afterwards. Maps
// built by K3 strictly decrease (v, id) along a chain, so every walk
// terminates -- but a long monotone chain would cost one thread O(depth)
// dependent loads, so a walk stops after kChaseSteps, leaves the ancestor it
// reached and counts itself pending; jump_kernel then finishes by pointer
// jumping in at most ceil(log2 n) + 2 synchronous rounds (or reports a
// cycle, ggd.cpp:41) and rewrites the labels. No N x S flag or scan arrays
// (LFR 1M x 32: label passes 0.43 -> 0.29 ms with the succ copy; R-MAT 22:
// 1.45 -> 1.10 ms).
constexpr int kChaseSteps = 256;

// Root bitmap of one sigma slice: W = ceil(n / 32) words per sigma.
struct RootRank {
    const unsigned* word;  // [S][W]
    const int* pre;        // [S * W + 1]: exclusive scan of the words' popcounts
    int W;
    __device__ __forceinline__ int operator()(int sigma, int x) const {
        const long long k = static_cast<long long>(sigma) * W + (x >> 5);
        return __ldg(pre + k) - __ldg(pre + static_cast<long long>(sigma) * W) +
               __popc(__ldg(word + k) & ((1u << (x & 31)) - 1u));
    }
};

// Four nodes per thread (16 B loads / stores); a lane's 4-bit nibble of
// roots is merged with its 7 neighbours' into the 32-node word.
__global__ void __launch_bounds__(kBlock) roots_kernel(int n, int W, const int* __restrict__ succ,
                                                       int* __restrict__ center, unsigned* __restrict__ word,
                                                       int* __restrict__ pop, int S, bool aligned) {
    const long long b = static_cast<long long>(blockIdx.y) * n;
    const int i0 = (blockIdx.x * kBlock + threadIdx.x) * 4;
    int x[4];
    const bool vec = aligned && i0 + 3 < n;  // 16 B aligned buffers, n % 4 == 0: every slice aligned
    if (vec) {
        const int4 q = __ldg(reinterpret_cast<const int4*>(succ + b + i0));
        x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
        if (center != succ) *reinterpret_cast<int4*>(center + b + i0) = q;
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            x[u] = i0 + u < n ? succ[b + i0 + u] : -1;
            if (i0 + u < n && center != succ) center[b + i0 + u] = x[u];
        }
    }
    unsigned m = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) m |= (x[u] == i0 + u ? 1u : 0u) << u;
    const int lane = threadIdx.x & 31;
    m <<= 4 * (lane & 7);
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) m |= __shfl_xor_sync(0xffffffffu, m, d);
    const int k = i0 >> 5;
    if ((lane & 7) == 0 && k < W) {
        const long long o = static_cast<long long>(blockIdx.y) * W + k;
        word[o] = m;
        pop[o] = __popc(m);
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) pop[static_cast<long long>(S) * W] = 0;
}

// Roots carry their label through the chase: center[r] = -1 - rank(r) for
// every root r (encode), restored to r afterwards (decode). Four nodes of
// one word per thread: coalesced, and nothing to do where the word is 0.
template <bool kEncode>
__global__ void __launch_bounds__(kBlock) root_code_kernel(int n, int* __restrict__ center, const RootRank rank) {
    const int i0 = (blockIdx.x * kBlock + threadIdx.x) * 4;
    if (i0 >= n) return;
    const int sigma = blockIdx.y;
    const long long k = static_cast<long long>(sigma) * rank.W + (i0 >> 5);
    const unsigned word = __ldg(rank.word + k);
    const unsigned m = (word >> (i0 & 31)) & 0xfu;
    if (!m) return;
    int r = __ldg(rank.pre + k) - __ldg(rank.pre + static_cast<long long>(sigma) * rank.W) +
            __popc(word & ((1u << (i0 & 31)) - 1u));
    int* c = center + static_cast<long long>(sigma) * n;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if ((m >> u) & 1u) {
            c[i0 + u] = kEncode ? -1 - r : i0 + u;
            ++r;
        }
}

// center[] holds parent pointers with the roots encoded as -1 - rank: a walk
// ends at the first negative value, which is its root's label, and writes
// the root's id (the one a later walk reads is then one step from the code).
__global__ void __launch_bounds__(kBlock) chase_kernel(int n, int* __restrict__ center, int* __restrict__ ci,
                                                       int* __restrict__ pending) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const long long b = static_cast<long long>(blockIdx.y) * n;
    int* c = center + b;
    int x = c[i];
    if (x < 0) {  // i is a root
        ci[b + i] = -1 - x;
        return;
    }
    for (int step = 0;; ++step) {
        const int y = c[x];
        if (y < 0) {
            ci[b + i] = -1 - y;
            break;
        }
        x = y;
        if (step == kChaseSteps) {
            atomicAdd(pending, 1);
            break;
        }
    }
    c[i] = x;
}

// Pointer jumping over every (sigma, node) of center[] until all point at
// roots, then the labels of every node again; does nothing more than the
// per-sigma cluster counts (one launch, all blocks return at once) when no
// chase hit its step bound. Cooperative launch: rounds are separated by grid
// syncs, so each round at least halves every remaining distance (in-place
// updates only jump further). A map still unresolved after `rounds` rounds
// has a cycle: *err = 1.
__global__ void __launch_bounds__(kBlock) jump_kernel(int n, int S, int* __restrict__ center, int* __restrict__ ci,
                                                      const RootRank rank, int* __restrict__ num_clusters,
                                                      int* __restrict__ status, int rounds, int* __restrict__ err) {
    const long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t0 < S)
        num_clusters[t0] = rank.pre[(t0 + 1) * rank.W] - rank.pre[t0 * rank.W];
    if (*reinterpret_cast<volatile int*>(status) == 0) return;  // no pending chase (uniform across the grid)
    cg::grid_group grid = cg::this_grid();
    const long long total = static_cast<long long>(n) * S;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    bool done = false;
    for (int r = 0; r < rounds && !done; ++r) {
        int* cnt = status + 1 + (r % 3);
        if (t0 == 0) status[1 + ((r + 1) % 3)] = 0;  // last read before the previous round's sync
        int changed = 0;
        for (long long t = t0; t < total; t += stride) {
            const long long b = t - t % n;
            const int x = center[t];
            const int y = center[b + x];
            if (y != x) {
                center[t] = y;
                ++changed;
            }
        }
        if (changed) atomicAdd(cnt, changed);
        grid.sync();
        done = *reinterpret_cast<volatile int*>(cnt) == 0;
    }
    if (!done) {
        if (t0 == 0 && err) atomicExch(err, 1);
        return;
    }
    for (long long t = t0; t < total; t += stride) ci[t] = rank(static_cast<int>(t / n), center[t]);
}

// Node-major [n][S] -> sigma-major [S][n].
__global__ void transpose_kernel(const double* __restrict__ in, int n, int S, double* __restrict__ out) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r, s = s0 + threadIdx.x;
        if (i < n && s < S) tile[r][threadIdx.x] = in[static_cast<long long>(i) * S + s];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int s = s0 + r, i = i0 + threadIdx.x;
        if (i < n && s < S) out[static_cast<long long>(s) * n + i] = tile[threadIdx.x][r];
    }
}

// Checked resolve (arbitrary successor maps): pointer jumping that carries
// the terminal kind of each chain: 0 pending, 1 root, 2 out-of-range node.
__global__ void resolve_init_kernel(int n, const int* __restrict__ succ, int* __restrict__ ptr,
                                    int* __restrict__ term) {
    const int x = blockIdx.x * kBlock + threadIdx.x;
    if (x >= n) return;
    const int sx = succ[x];
    if (sx < 0 || sx >= n) {
        ptr[x] = x;
        term[x] = 2;
    } else if (sx == x) {
        ptr[x] = x;
        term[x] = 1;
    } else {
        ptr[x] = sx;
        term[x] = 0;
    }
}

__global__ void resolve_round_kernel(int n, const int* __restrict__ pin, const int* __restrict__ tin,
                                     int* __restrict__ pout, int* __restrict__ tout) {
    const int x = blockIdx.x * kBlock + threadIdx.x;
    if (x >= n) return;
    const int t = tin[x];
    if (t != 0) {
        pout[x] = pin[x];
        tout[x] = t;
        return;
    }
    const int p = pin[x];
    pout[x] = pin[p];
    tout[x] = tin[p];
}

// First failing start node in ascending order decides the reference's error
// (ggd.cpp:30-46): out-of-range (2) or cycle (still pending after the rounds).
__global__ void resolve_error_kernel(int n, const int* __restrict__ term, unsigned long long* __restrict__ first) {
    const int x = blockIdx.x * kBlock + threadIdx.x;
    if (x >= n) return;
    const int t = term[x];
    if (t != 1) {
        const unsigned long long kind = t == 2 ? 1ull : 2ull;
        atomicMin(first, (static_cast<unsigned long long>(x) << 2) | kind);
    }
}

int grid_for(long long threads) { return static_cast<int>((threads + kBlock - 1) / kBlock); }

// Side stream and fork/join events for companion launches, one set per parent
// stream (calls on different devices run concurrently: the map is locked; a
// parent stream belongs to one device, whose calls are serialized).
struct SideStream {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_for(cudaStream_t parent) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, SideStream> all;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    SideStream& c = all[{dev, parent}];
    if (!c.stream) {
        cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming);
    }
    return c;
}

}  // namespace

int launch_potentials(const PotentialLaunch& p, int kernel, void* pool, void* stream) {
    const long long threads = static_cast<long long>(p.row_end - p.row_begin) * p.n_sigma;
    if (threads <= 0) return cudaSuccess;
    auto st = static_cast<cudaStream_t>(stream);
    const dim3 grid(grid_for(threads));
    const bool ff = kernel == 0;
    PrefixTable T{};
    void* mem = nullptr;
    if (ff) {
        // stream-ordered scratch: safe for concurrent calls on other streams
        const int q = 2 * p.n_sigma;
        const std::size_t bytes = static_cast<std::size_t>(q) * kPrefixCap * (sizeof(int) + 2 * sizeof(double)) +
                                  static_cast<std::size_t>(q) * (2 * sizeof(int) + 2 * sizeof(double)) + 64;
        cudaError_t e = cudaMallocFromPoolAsync(&mem, bytes, static_cast<cudaMemPool_t>(pool), st);
        if (e != cudaSuccess) return e;
        char* b = static_cast<char*>(mem);
        T.s0 = reinterpret_cast<double*>(b);
        T.inc = T.s0 + q * kPrefixCap;
        T.s_end = T.inc + q * kPrefixCap;
        T.iso = T.s_end + q;
        T.iso_last = T.iso + q / 2;
        T.t = reinterpret_cast<int*>(T.iso_last + q / 2);
        T.count = T.t + q * kPrefixCap;
        T.t_end = T.count + q;
        prefix_kernel<<<1, 64, 0, st>>>(p, T);
        count_launch();
    }
    // the fast-forward always runs warp per row (a single sigma leaves 31
    // lanes idle, but hub rows take the batched walk: R-MAT 22 at one sigma
    // 7.1 ms against 188 ms thread per row; LFR 1M 2.6 vs 2.4 ms); the dense
    // replay below kWarpKernelMinSigma sigmas fills the lanes with rows
    if (ff || p.n_sigma >= kWarpKernelMinSigma) {
        // persistent warp-per-row kernel: one resident wave, rows scheduled
        // longest first through an atomic counter
        const int num_sms = sm_count();
        const int rows = p.row_end - p.row_begin;
        auto pl = static_cast<cudaMemPool_t>(pool);
        std::size_t sort_bytes = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, static_cast<const int*>(nullptr),
                                                  static_cast<int*>(nullptr), static_cast<const int*>(nullptr),
                                                  static_cast<int*>(nullptr), rows);
        const std::size_t arr = ((static_cast<std::size_t>(rows) * sizeof(int)) + 255) & ~static_cast<std::size_t>(255);
        void* sched = nullptr;
        cudaError_t e = cudaMallocFromPoolAsync(&sched, 4 * arr + sort_bytes + 256, pl, st);
        if (e != cudaSuccess) {
            if (mem) cudaFreeAsync(mem, st);
            return e;
        }
        char* b = static_cast<char*>(sched);
        int* deg_in = reinterpret_cast<int*>(b);
        int* deg_out = reinterpret_cast<int*>(b + arr);
        int* id_in = reinterpret_cast<int*>(b + 2 * arr);
        int* id_out = reinterpret_cast<int*>(b + 3 * arr);
        int* counter = reinterpret_cast<int*>(b + 4 * arr);
        void* temp = b + 4 * arr + 256;
        // hub rows (see hub_split_kernel) need the degree itself; otherwise
        // capped keys (11 bits + 2 slab bits) sort in 2 passes
        const bool hubs = !(ff && p.weight_mode == kUnit);
        const int key_bits = hubs ? 24 : 11;
        row_degree_kernel<<<grid_for(rows), kBlock, 0, st>>>(reinterpret_cast<const long long*>(p.offsets),
                                                              p.row_begin, rows, deg_in, id_in, p.slab_flags,
                                                              p.slab_bound[1], p.slab_bound[2], p.slab_bound[3],
                                                              key_bits);
        count_launch();
        e = cub::DeviceRadixSort::SortPairsDescending(temp, sort_bytes, deg_in, deg_out, id_in, id_out, rows, 0,
                                                      key_bits + 2, st);
        count_launch(2);
        if (e != cudaSuccess) {  // no scratch leaks on the error path
            cudaFreeAsync(sched, st);
            if (mem) cudaFreeAsync(mem, st);
            return e;
        }
        // hub rows (see hub_split_kernel): longer than ~1/4096 of the entries.
        // The unit-weight fast-forward walks long rows with batched in-binade
        // jumps (walk_events), so a hub costs it ~10^2 steps and no hub gets
        // an SM of its own there.
        int* hub_count = counter + 1;
        int* hub_counter = counter + 2;
        const long long threshold = hubs ? std::max<long long>(4096, p.nnz / 4096) : (1ll << 62);
        hub_split_kernel<<<1, 1, 0, st>>>(deg_out, rows, threshold, p.slab_flags ? (1 << key_bits) - 1 : -1, hub_count,
                                          counter, hub_counter);
        count_launch();
        const RowSched R{id_out, counter, nullptr};
        const RowSched Rh{id_out, hub_counter, hub_count};
        const long long want = (static_cast<long long>(rows) + kBlock / 32 - 1) / (kBlock / 32);
        const dim3 wgrid(static_cast<unsigned>(
            std::min<long long>(want, static_cast<long long>(num_sms) * kWarpKernelBlocksPerSM)));
        SideStream& side = side_for(st);
        if (hubs) {
            cudaEventRecord(side.fork, st);
            cudaStreamWaitEvent(side.stream, side.fork, 0);
        }
        auto launch = [&](auto kernel) {
            if (hubs) {
                cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHubSmemBytes);
                kernel<<<kMaxHubs, 32, kHubSmemBytes, side.stream>>>(p, T, Rh);  // first: hub blocks claim SMs
                count_launch();
            }
            kernel<<<wgrid, kBlock, 0, st>>>(p, T, R);
            count_launch();
        };
        switch (p.weight_mode) {
            case kUnit:
                // a row range short of the whole graph is a shard of a
                // multi-device sweep: hub rows walk whole (kLong)
                if (ff && p.row_end - p.row_begin < p.n)
                    p.iso ? launch(potential_warp_kernel<true, kUnit, true, true>)
                          : launch(potential_warp_kernel<true, kUnit, true>);
                else if (ff)
                    p.iso ? launch(potential_warp_kernel<true, kUnit, false, true>)
                          : launch(potential_warp_kernel<true, kUnit>);
                else launch(potential_warp_kernel<false, kUnit>);
                break;
            case kDevicePexp:
                if (ff) launch(potential_warp_kernel<true, kDevicePexp>);
                else launch(potential_warp_kernel<false, kDevicePexp>);
                break;
            default:
                if (ff) launch(potential_warp_kernel<true, kEntryTable>);
                else launch(potential_warp_kernel<false, kEntryTable>);
                break;
        }
        if (hubs) {
            cudaEventRecord(side.join, side.stream);
            cudaStreamWaitEvent(st, side.join, 0);
        }
        cudaFreeAsync(sched, st);
    } else {
        // thread per (row, sigma): rows in descending-degree order, so the
        // lanes of a warp walk rows with the same number of events (one sort
        // per launch; small launches keep the natural order)
        const int rows = p.row_end - p.row_begin;
        const int* order = nullptr;
        void* sched = nullptr;
        if (rows >= kSortRowsMin) {
            std::size_t sort_bytes = 0;
            cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, static_cast<const int*>(nullptr),
                                                      static_cast<int*>(nullptr), static_cast<const int*>(nullptr),
                                                      static_cast<int*>(nullptr), rows);
            const std::size_t arr = ((static_cast<std::size_t>(rows) * sizeof(int)) + 255) & ~static_cast<std::size_t>(255);
            cudaError_t e = cudaMallocFromPoolAsync(&sched, 4 * arr + sort_bytes, static_cast<cudaMemPool_t>(pool), st);
            if (e != cudaSuccess) {
                if (mem) cudaFreeAsync(mem, st);
                return e;
            }
            char* b = static_cast<char*>(sched);
            int* deg_in = reinterpret_cast<int*>(b);
            int* deg_out = reinterpret_cast<int*>(b + arr);
            int* id_in = reinterpret_cast<int*>(b + 2 * arr);
            int* id_out = reinterpret_cast<int*>(b + 3 * arr);
            row_degree_kernel<<<grid_for(rows), kBlock, 0, st>>>(reinterpret_cast<const long long*>(p.offsets),
                                                                  p.row_begin, rows, deg_in, id_in, nullptr, 0, 0, 0,
                                                                  24);
            e = cub::DeviceRadixSort::SortPairsDescending(b + 4 * arr, sort_bytes, deg_in, deg_out, id_in, id_out, rows,
                                                          0, 32, st);
            count_launch(3);
            if (e != cudaSuccess) {
                cudaFreeAsync(sched, st);
                if (mem) cudaFreeAsync(mem, st);
                return e;
            }
            order = id_out;
        }
        switch (p.weight_mode) {
            case kUnit:
                if (ff) potential_kernel<true, kUnit><<<grid, kBlock, 0, st>>>(p, T, order);
                else potential_kernel<false, kUnit><<<grid, kBlock, 0, st>>>(p, T, order);
                break;
            case kDevicePexp:
                if (ff) potential_kernel<true, kDevicePexp><<<grid, kBlock, 0, st>>>(p, T, order);
                else potential_kernel<false, kDevicePexp><<<grid, kBlock, 0, st>>>(p, T, order);
                break;
            default:
                if (ff) potential_kernel<true, kEntryTable><<<grid, kBlock, 0, st>>>(p, T, order);
                else potential_kernel<false, kEntryTable><<<grid, kBlock, 0, st>>>(p, T, order);
                break;
        }
        if (sched) cudaFreeAsync(sched, st);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (mem) cudaFreeAsync(mem, st);
    return e;
}

namespace {

// ---------------------------------------------------------------------------
// Degree-class order (ClassOrder, gqc_internal.h). On a unit-weight graph a
// row's potential is mathematically a Moebius function of its degree d
// (num and den are affine in d, potential.cpp:18-37), hence monotone in d;
// rounding noise separates equal-degree nodes only. Whether the field at
// hand really orders its degree classes strictly is VERIFIED per sigma:
// nodes are sorted by degree, each class's [min, max] potential is reduced,
// and consecutive classes must not overlap (in one direction). A sigma that
// fails (weighted graphs, k-hop fields, saturated regimes) keeps the plain
// argmin. Potentials are >= +0, so their bit patterns order like the values.
// ---------------------------------------------------------------------------
__global__ void class_key_kernel(const long long* __restrict__ off, int n, int* __restrict__ key,
                                 int* __restrict__ id) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        key[i] = static_cast<int>(off[i + 1] - off[i]);
        id[i] = i;
    }
}

__global__ void class_flag_kernel(const int* __restrict__ sdeg, int n, int* __restrict__ flag) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) flag[k] = (k == 0 || sdeg[k] != sdeg[k - 1]) ? 1 : 0;
}

// cls[node] = class index (inclusive scan - 1); clear the min / max tables
__global__ void class_scatter_kernel(const int* __restrict__ sid, const int* __restrict__ cidx, int n, int S,
                                     int* __restrict__ cls, unsigned long long* __restrict__ mn,
                                     unsigned long long* __restrict__ mx) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) cls[sid[k]] = cidx[k] - 1;
    const int C = cidx[n - 1];
    for (long long t = k; t < static_cast<long long>(C) * S; t += static_cast<long long>(gridDim.x) * blockDim.x) {
        mn[t] = ~0ull;
        mx[t] = 0ull;
    }
}

// warp per run of kClassRun sorted positions, lane = sigma: running min / max
// of the class, flushed with 64-bit atomics when the class changes
constexpr int kClassRun = 64;
__global__ void class_minmax_kernel(const int* __restrict__ sid, const int* __restrict__ cls,
                                    const double* __restrict__ v, int ld, int S, int n,
                                    unsigned long long* __restrict__ mn, unsigned long long* __restrict__ mx) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int k0 = w * kClassRun;
    if (k0 >= n) return;
    const int k1 = min(n, k0 + kClassRun);
    for (int sb = 0; sb < S; sb += 32) {
        const int s = sb + lane;
        int cur = -1;
        unsigned long long lo = ~0ull, hi = 0ull;
        for (int k = k0; k < k1; ++k) {
            const int i = __ldg(sid + k);
            const int c = __ldg(cls + i);
            if (c != cur) {
                if (cur >= 0 && s < S) {
                    atomicMin(mn + static_cast<long long>(cur) * S + s, lo);
                    atomicMax(mx + static_cast<long long>(cur) * S + s, hi);
                }
                cur = c;
                lo = ~0ull;
                hi = 0ull;
            }
            if (s < S) {
                const unsigned long long b =
                    static_cast<unsigned long long>(__double_as_longlong(__ldg(v + static_cast<long long>(i) * ld + s)));
                lo = min(lo, b);
                hi = max(hi, b);
            }
        }
        if (s < S) {
            atomicMin(mn + static_cast<long long>(cur) * S + s, lo);
            atomicMax(mx + static_cast<long long>(cur) * S + s, hi);
        }
    }
}

// viol[s] bit 0: some consecutive classes not strictly ascending; bit 1: not
// strictly descending
__global__ void class_check_kernel(const unsigned long long* __restrict__ mn, const unsigned long long* __restrict__ mx,
                                   const int* __restrict__ cidx, int n, int S, int* __restrict__ viol) {
    const long long pairs = static_cast<long long>(cidx[n - 1] - 1) * S;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < pairs;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long c = t / S;
        const int s = static_cast<int>(t - c * S);
        const long long a = c * S + s, b = (c + 1) * S + s;
        int f = 0;
        if (!(mx[a] < mn[b])) f |= 1;
        if (!(mn[a] > mx[b])) f |= 2;
        if (f) atomicOr(viol + s, f);
    }
}

__global__ void class_dir_kernel(const int* __restrict__ viol, int S, signed char* __restrict__ dir) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < S) dir[s] = !(viol[s] & 1) ? 1 : (!(viol[s] & 2) ? -1 : 0);
}

}  // namespace

int launch_class_order(int n, const std::int64_t* offsets, long long nnz, const double* v, int ld, int S, void* pool_,
                       void* stream, ClassOrder* out, void** mem) {
    auto st = static_cast<cudaStream_t>(stream);
    auto pool = static_cast<cudaMemPool_t>(pool_);
    *mem = nullptr;
    if (n < 1 || S < 1) return cudaSuccess;
    // distinct degrees d_1 < ... < d_C sum to at most nnz: C <= sqrt(2 nnz) + 1
    const long long cmax = std::min<long long>(n, static_cast<long long>(std::sqrt(2.0 * static_cast<double>(nnz))) + 2);
    int end_bit = 1;
    while (end_bit < 31 && (1ll << end_bit) <= nnz) ++end_bit;
    std::size_t sort_bytes = 0, scan_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<const int*>(nullptr), static_cast<int*>(nullptr), n, 0, end_bit);
    cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, static_cast<const int*>(nullptr), static_cast<int*>(nullptr), n);
    auto al = [](std::size_t b) { return (b + 255) & ~static_cast<std::size_t>(255); };
    const std::size_t b_n = al(static_cast<std::size_t>(n) * sizeof(int));
    const std::size_t b_t = al(static_cast<std::size_t>(cmax) * S * sizeof(unsigned long long));
    const std::size_t b_s = al(static_cast<std::size_t>(S) * sizeof(int));
    const std::size_t total = 6 * b_n + 2 * b_t + 2 * b_s + al(std::max(sort_bytes, scan_bytes));
    cudaError_t e = cudaMallocFromPoolAsync(mem, total, pool, st);
    if (e != cudaSuccess) return e;
    char* m = static_cast<char*>(*mem);
    int* key = reinterpret_cast<int*>(m);
    int* id = reinterpret_cast<int*>(m + b_n);
    int* sdeg = reinterpret_cast<int*>(m + 2 * b_n);
    int* sid = reinterpret_cast<int*>(m + 3 * b_n);
    int* cidx = reinterpret_cast<int*>(m + 4 * b_n);
    int* cls = reinterpret_cast<int*>(m + 5 * b_n);
    auto* mn = reinterpret_cast<unsigned long long*>(m + 6 * b_n);
    auto* mx = reinterpret_cast<unsigned long long*>(m + 6 * b_n + b_t);
    int* viol = reinterpret_cast<int*>(m + 6 * b_n + 2 * b_t);
    auto* dir = reinterpret_cast<signed char*>(m + 6 * b_n + 2 * b_t + b_s);
    void* tmp = m + 6 * b_n + 2 * b_t + 2 * b_s;
    auto off = reinterpret_cast<const long long*>(offsets);
    const int g = grid_for(n);
    class_key_kernel<<<g, kBlock, 0, st>>>(off, n, key, id);
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, key, sdeg, id, sid, n, 0, end_bit, st)) != cudaSuccess)
        return e;
    class_flag_kernel<<<g, kBlock, 0, st>>>(sdeg, n, key);
    if ((e = cub::DeviceScan::InclusiveSum(tmp, scan_bytes, key, cidx, n, st)) != cudaSuccess) return e;
    class_scatter_kernel<<<g, kBlock, 0, st>>>(sid, cidx, n, S, cls, mn, mx);
    const long long warps = (n + kClassRun - 1) / kClassRun;
    class_minmax_kernel<<<static_cast<unsigned>((warps * 32 + kBlock - 1) / kBlock), kBlock, 0, st>>>(sid, cls, v, ld,
                                                                                                     S, n, mn, mx);
    cudaMemsetAsync(viol, 0, S * sizeof(int), st);
    class_check_kernel<<<512, kBlock, 0, st>>>(mn, mx, cidx, n, S, viol);
    class_dir_kernel<<<(S + kBlock - 1) / kBlock, kBlock, 0, st>>>(viol, S, dir);
    count_launch(10);
    out->cls = cls;
    out->dir = dir;
    if (const char* t = std::getenv("GQC_TRACE"); t && *t && *t != '0') {  // which sigmas verified
        std::vector<signed char> h(S);
        int C = 0;
        cudaMemcpyAsync(h.data(), dir, S, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&C, cidx + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        std::string line = "[gqc trace] class order: " + std::to_string(C) + " degree classes, dir =";
        for (int q = 0; q < S; ++q) line += " " + std::to_string(static_cast<int>(h[q]));
        std::fprintf(stderr, "%s\n", line.c_str());
    }
    return cudaGetLastError();
}

namespace {
// Modularity's intra-cluster weight for unit weights (metrics.cpp:37-44):
// out[s] += #{CSR entries (i, j) with ci[s][i] == ci[s][j]}, an exact integer
// (the reference sums 1.0s, also exact). Thread per row, blockIdx.y = sigma.
__global__ void __launch_bounds__(kBlock) intra_count_kernel(const long long* __restrict__ off,
                                                             const int* __restrict__ nbr,
                                                             const int* __restrict__ ci, int n,
                                                             unsigned long long* __restrict__ out) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const int* c = ci + static_cast<long long>(blockIdx.y) * n;
    unsigned long long cnt = 0;
    if (i < n) {
        const int ci_i = c[i];
        for (long long k = off[i]; k < off[i + 1]; ++k) cnt += __ldg(c + __ldg(nbr + k)) == ci_i;
    }
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out + blockIdx.y, cnt);
}
}  // namespace

int launch_intra_counts(int n, int n_sigma, const std::int64_t* offsets, const std::int32_t* nbr,
                        const std::int32_t* ci_sm, long long* out, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(out, 0, n_sigma * sizeof(long long), st);
    intra_count_kernel<<<dim3(grid_for(n), n_sigma), kBlock, 0, st>>>(
        reinterpret_cast<const long long*>(offsets), nbr, ci_sm, n, reinterpret_cast<unsigned long long*>(out));
    count_launch();
    return cudaGetLastError();
}

namespace {
// Degree sample of the GGD argmin's launch shape: kTinySample pseudo-random
// rows (multiplicative hashing: evenly spaced ids would follow R-MAT's id
// structure, where ids with many trailing zero bits are hubs).
constexpr int kTinySample = 8192;
constexpr int kTinyRowDegree = 4;
__host__ __device__ inline long long sample_row(int k, long long n) {
    unsigned long long h = static_cast<unsigned long long>(k) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    return static_cast<long long>(h % static_cast<unsigned long long>(n));
}
// count[0]: sampled rows with <= kTinyRowDegree neighbours, count[1]: with none
__global__ void tiny_sample_kernel(const long long* __restrict__ off, int n, int* __restrict__ count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const long long d = k < kTinySample ? off[sample_row(k, n) + 1] - off[sample_row(k, n)] : 1 << 30;
    const unsigned m = __ballot_sync(0xffffffffu, d <= kTinyRowDegree);
    const unsigned z = __ballot_sync(0xffffffffu, d == 0);
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicAdd(count, __popc(m));
        if (z) atomicAdd(count + 1, __popc(z));
    }
}
int sub_from_count(int tiny) { return 5 * tiny > kTinySample ? 16 : 32; }  // > 20% of rows tiny

// The degree sample of a device CSR, cached per device and CSR pointer /
// shape (one stream synchronisation the first time; only the speed depends
// on it): {rows with <= 4 neighbours, isolated rows} among kTinySample.
std::pair<int, int> degree_sample_device(const std::int64_t* offsets, int n, long long nnz, void* stream) {
    if (n < 1) return {0, 0};
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, long long>, std::pair<int, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, static_cast<const void*>(offsets), n, nnz);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    auto st = static_cast<cudaStream_t>(stream);
    int* d = nullptr;
    int h[2] = {0, 0};
    if (cudaMallocAsync(reinterpret_cast<void**>(&d), 2 * sizeof(int), st) != cudaSuccess) {
        cudaGetLastError();
        return {0, 0};
    }
    cudaMemsetAsync(d, 0, 2 * sizeof(int), st);
    tiny_sample_kernel<<<kTinySample / kBlock, kBlock, 0, st>>>(reinterpret_cast<const long long*>(offsets), n, d);
    count_launch();
    cudaMemcpyAsync(h, d, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return {0, 0};
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = {h[0], h[1]};
    return {h[0], h[1]};
}
}  // namespace

int isolated_rows_device(const std::int64_t* offsets, int n, long long nnz, void* stream) {
    return 100 * degree_sample_device(offsets, n, nnz, stream).second > kTinySample ? 1 : 0;  // > 1% of rows
}

int light_row_sigmas_host(const std::int64_t* offsets, int n) {
    if (n < 1) return 32;
    int tiny = 0;
    for (int k = 0; k < kTinySample; ++k) {
        const long long i = sample_row(k, n);
        tiny += offsets[i + 1] - offsets[i] <= kTinyRowDegree;
    }
    return sub_from_count(tiny);
}

int light_row_sigmas_device(const std::int64_t* offsets, int n, long long nnz, void* stream) {
    return sub_from_count(degree_sample_device(offsets, n, nnz, stream).first);
}

int launch_successors(int n, const std::int64_t* offsets, const std::int32_t* nbr, const double* v, int ld, int s0,
                      int n_sigma, int row_begin, int row_end, std::int32_t* out, long long out_row, long long out_col,
                      long long nnz, void* pool, void* stream, const ClassOrder* co, int sub) {
    if (sub < 1 || sub > 32) sub = kSuccSub;
    (void)n;
    auto st = static_cast<cudaStream_t>(stream);
    auto off = reinterpret_cast<const long long*>(offsets);
    const int rows = row_end - row_begin;
    if (rows <= 0) return cudaSuccess;
    // heavy rows have > kHeavyDegree entries each and multi-segment rows >
    // kHeavySegment, so nnz bounds the items, partial slots and row lists
    const long long heavy_max = std::min<long long>(rows, nnz / (kHeavyDegree + 1) + 1);
    const long long seg_max = heavy_max + nnz / kHeavySegment + 1;
    const long long multi_max = nnz / (kHeavySegment + 1) + 1;
    const long long slot_max = 2 * multi_max + nnz / kHeavySegment + 1;
    const std::size_t bytes_items = sizeof(HeavyItem) * seg_max, bytes_multi = sizeof(HeavyRow) * multi_max;
    const std::size_t bytes_pv = sizeof(double) * 32 * slot_max, bytes_pi = sizeof(int) * 32 * slot_max;
    const std::size_t head = 256;
    const bool tiny_rows = kTinyDegree > 0 && !(co && co->dir);
    const std::size_t bytes_tiny = tiny_rows ? sizeof(int) * static_cast<std::size_t>(rows) : 0;
    void* scratch = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&scratch, head + bytes_pv + bytes_items + bytes_multi + bytes_pi + bytes_tiny,
                                            static_cast<cudaMemPool_t>(pool), st);
    if (e != cudaSuccess) return e;
    char* p = static_cast<char*>(scratch);
    int* counts = reinterpret_cast<int*>(p);
    double* part_v = reinterpret_cast<double*>(p + head);
    auto* items = reinterpret_cast<HeavyItem*>(p + head + bytes_pv);
    auto* multi = reinterpret_cast<HeavyRow*>(p + head + bytes_pv + bytes_items);
    int* part_i = reinterpret_cast<int*>(p + head + bytes_pv + bytes_items + bytes_multi);
    int* tiny = tiny_rows ? reinterpret_cast<int*>(p + head + bytes_pv + bytes_items + bytes_multi + bytes_pi) : nullptr;
    cudaMemsetAsync(counts, 0, 4 * sizeof(int), st);
    mark_heavy_kernel<<<grid_for(rows), kBlock, 0, st>>>(off, row_begin, rows, items, counts, multi, tiny);
    count_launch(2);
    const int num_sms = sm_count();
    // thread = (row, sigma), sigma fastest: a neighbour's potentials for the
    // chunk's sigmas are one contiguous node-major line
    for (int c0 = 0; c0 < n_sigma; c0 += 32) {
        const int Sc = std::min(32, n_sigma - c0);
        const SuccOut O{out + c0 * out_col, out_row, out_col};
        // light rows: the kernels index threads in 32 bits, so the row range
        // goes in sub-launches of fewer than 2^31 threads (graphs of ~67M+
        // nodes at 32 sigmas), each with its output moved to its first row.
        // sub < 32 runs the plain argmin in launches of that many sigmas
        // over all rows (a warp then takes 32 / sub rows), so each launch
        // gathers one slice of every node's V line. Measured (32 sigmas, GGD
        // ms, 32 / 16 / 8 / 4 per launch): LFR 1M 1.33 / 1.43 / 1.87 / 2.58,
        // R-MAT 22 5.94 / 4.52 / 5.00 / 6.13: graphs made mostly of rows
        // with a handful of neighbours (R-MAT: 79% of rows have <= 4) gain
        // from two rows per warp, the others do not; the callers pick it
        // from a degree sample (light_row_sigmas).
        const long long per = ((1ll << 31) - 2 * kBlock) / 32;
        for (long long r0 = 0; r0 < rows; r0 += per) {
            const int rr = static_cast<int>(std::min<long long>(per, rows - r0));
            const int rb = row_begin + static_cast<int>(r0);
            if (co && co->dir) {
                const SuccOut Or{O.out + r0 * out_row, out_row, out_col};
                successors_class_kernel<<<grid_for(static_cast<long long>(rr) * 32), kBlock, 0, st>>>(
                    off, nbr, v, ld, s0 + c0, Sc, rb, rr, Or, *co);
                count_launch();
            } else {  // rows of more than kTinyDegree neighbours (tiny ones: successors_tiny_kernel)
                const int lo = tiny_rows ? kTinyDegree + 1 : 0;
                for (int q0 = 0; q0 < Sc; q0 += sub) {
                    const int Sq = std::min(sub, Sc - q0);
                    const SuccOut Or{O.out + r0 * out_row + q0 * out_col, out_row, out_col};
                    successors_kernel<<<grid_for(static_cast<long long>(rr) * Sq), kBlock, 0, st>>>(
                        off, nbr, v, ld, s0 + c0 + q0, Sq, rb, rr, Or, lo, kHeavyDegree);
                    count_launch();
                }
            }
        }
        if (tiny_rows) {
            successors_tiny_kernel<<<num_sms * 8, kBlock, 0, st>>>(off, nbr, v, ld, s0 + c0, Sc, row_begin, tiny, counts,
                                                                    O);
            count_launch();
        }
        successors_heavy_kernel<<<num_sms * 8, kBlock, 0, st>>>(off, nbr, v, ld, s0 + c0, Sc, row_begin, items, counts,
                                                                 part_v, part_i, O);
        successors_combine_kernel<<<num_sms * 2, kBlock, 0, st>>>(multi, counts, part_v, part_i, Sc, row_begin, O);
        count_launch(2);
    }
    cudaFreeAsync(scratch, st);
    return cudaGetLastError();
}

int launch_transpose_i32(const std::int32_t* in, int n, int n_sigma, std::int32_t* out, void* stream) {
    const dim3 grid((n + 31) / 32, (n_sigma + 31) / 32);
    transpose_i32_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(in, n, n_sigma, out);
    count_launch();
    return cudaGetLastError();
}

namespace {
// launch_labels' workspace: [status 256 B][root words S*W][popcounts /
// their scan S*W + 1][CUB temp], W = ceil(n / 32). status[0]: chases that
// hit their step bound; status[1..3]: jump_kernel's round counters.
struct LabelsWs {
    int* status;
    unsigned* word;
    int* pop;
    int* pre;
    void* temp;
    std::size_t temp_bytes;
    int W;
};
std::size_t align256(std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); }
std::size_t scan_temp_bytes(long long items) {
    std::size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<const int*>(nullptr), static_cast<int*>(nullptr), items);
    return temp;
}
LabelsWs labels_ws(void* workspace, int n, int n_sigma) {
    const int W = (n + 31) / 32;
    const long long words = static_cast<long long>(W) * n_sigma;
    char* w = static_cast<char*>(workspace);
    LabelsWs L;
    L.W = W;
    L.status = reinterpret_cast<int*>(w);
    L.word = reinterpret_cast<unsigned*>(w + 256);
    L.pop = reinterpret_cast<int*>(w + 256 + align256(sizeof(unsigned) * words));
    L.pre = reinterpret_cast<int*>(w + 256 + align256(sizeof(unsigned) * words) + align256(sizeof(int) * (words + 1)));
    L.temp = w + 256 + align256(sizeof(unsigned) * words) + 2 * align256(sizeof(int) * (words + 1));
    L.temp_bytes = align256(scan_temp_bytes(words + 1));
    return L;
}
int jump_grid() {  // co-resident blocks of jump_kernel (cooperative launch), per device
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cache[dev].load();
    if (!v) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jump_kernel, kBlock, 0);
        v = std::max(1, per_sm) * sm_count();
        cache[dev].store(v);
    }
    return v;
}
}  // namespace

std::size_t labels_workspace_bytes(int n, int n_sigma) {
    const long long words = static_cast<long long>((n + 31) / 32) * n_sigma;
    return 256 + align256(sizeof(unsigned) * words) + 2 * align256(sizeof(int) * (words + 1)) +
           align256(scan_temp_bytes(words + 1));
}

int launch_labels(int n, int n_sigma, const std::int32_t* succ_sm, std::int32_t* center_sm, std::int32_t* ci_sm,
                  std::int32_t* num_clusters, void* workspace, std::size_t ws_bytes, void* stream, std::int32_t* err) {
    auto st = static_cast<cudaStream_t>(stream);
    if (!workspace || ws_bytes < labels_workspace_bytes(n, n_sigma)) return cudaErrorInvalidValue;
    if (n < 1 || n_sigma < 1) return cudaSuccess;
    const LabelsWs L = labels_ws(workspace, n, n_sigma);
    cudaError_t e = cudaMemsetAsync(L.status, 0, 4 * sizeof(int), st);
    if (e != cudaSuccess) return e;
    roots_kernel<<<dim3(static_cast<unsigned>((n + 4 * kBlock - 1) / (4 * kBlock)), n_sigma), kBlock, 0, st>>>(
        n, L.W, succ_sm, center_sm, L.word, L.pop, n_sigma,
        (n & 3) == 0 && ((reinterpret_cast<std::uintptr_t>(succ_sm) | reinterpret_cast<std::uintptr_t>(center_sm)) & 15) == 0);
    std::size_t temp_bytes = L.temp_bytes;
    const long long words = static_cast<long long>(L.W) * n_sigma;
    e = cub::DeviceScan::ExclusiveSum(L.temp, temp_bytes, L.pop, L.pre, words + 1, st);
    count_launch(3);  // roots + CUB init + scan
    if (e != cudaSuccess) return e;
    const RootRank rank{L.word, L.pre, L.W};
    const dim3 g4(static_cast<unsigned>((n + 4 * kBlock - 1) / (4 * kBlock)), n_sigma);
    root_code_kernel<true><<<g4, kBlock, 0, st>>>(n, center_sm, rank);
    chase_kernel<<<dim3(grid_for(n), n_sigma), kBlock, 0, st>>>(n, center_sm, ci_sm, L.status);
    root_code_kernel<false><<<g4, kBlock, 0, st>>>(n, center_sm, rank);
    count_launch(3);
    int rounds = 2;
    while ((1ll << (rounds - 2)) < n) ++rounds;  // ceil(log2 n) + 2
    int* status = L.status;
    void* args[] = {&n, &n_sigma, &center_sm, &ci_sm, const_cast<RootRank*>(&rank), &num_clusters, &status, &rounds,
                    &err};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jump_kernel), dim3(jump_grid()), dim3(kBlock), args, 0, st);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int launch_transpose(const double* v_nm, int n, int n_sigma, double* v_sm, void* stream) {
    const dim3 grid((n + 31) / 32, (n_sigma + 31) / 32);
    transpose_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(v_nm, n, n_sigma, v_sm);
    count_launch();
    return cudaGetLastError();
}

int resolve_checked(int n, const std::int32_t* succ_dev, std::int32_t* center_dev, std::int32_t* ci_dev,
                    std::int32_t* num_clusters_host, int* err_kind, void* pool_, void* stream) {
    auto pool = static_cast<cudaMemPool_t>(pool_);
    auto st = static_cast<cudaStream_t>(stream);
    int *p0, *t0, *p1, *t1, *nc;
    unsigned long long* first;
    const std::size_t bytes = sizeof(int) * static_cast<std::size_t>(n);
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p0), bytes * 4 + 64, pool, st);
    if (e != cudaSuccess) return e;
    int* const alloc = p0;
    t0 = p0 + n;
    p1 = t0 + n;
    t1 = p1 + n;
    first = reinterpret_cast<unsigned long long*>(p0 + 4 * static_cast<std::size_t>(n));  // 16n bytes: 8-aligned
    nc = reinterpret_cast<int*>(first + 1);
    const int g = grid_for(n);
    resolve_init_kernel<<<g, kBlock, 0, st>>>(n, succ_dev, p0, t0);
    count_launch();
    int rounds = 2;
    for (long long span = 1; span < n; span <<= 1) ++rounds;
    for (int r = 0; r < rounds; ++r) {
        resolve_round_kernel<<<g, kBlock, 0, st>>>(n, p0, t0, p1, t1);
        count_launch();
        std::swap(p0, p1);
        std::swap(t0, t1);
    }
    const unsigned long long none = ~0ull;
    cudaMemcpyAsync(first, &none, sizeof none, cudaMemcpyHostToDevice, st);
    resolve_error_kernel<<<g, kBlock, 0, st>>>(n, t0, first);
    count_launch();
    unsigned long long hfirst = none;
    cudaMemcpyAsync(&hfirst, first, sizeof hfirst, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeAsync(alloc, st);
        return e;
    }
    *err_kind = hfirst == none ? 0 : static_cast<int>(hfirst & 3ull);
    if (*err_kind == 0) {
        cudaMemcpyAsync(center_dev, p0, bytes, cudaMemcpyDeviceToDevice, st);
        std::size_t ws = labels_workspace_bytes(n, 1);
        void* wsp = nullptr;
        e = cudaMallocFromPoolAsync(&wsp, ws, pool, st);
        if (e == cudaSuccess) {
            e = static_cast<cudaError_t>(launch_labels(n, 1, center_dev, center_dev, ci_dev, nc, wsp, ws, st));
            cudaMemcpyAsync(num_clusters_host, nc, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaFreeAsync(wsp, st);
        }
    }
    cudaFreeAsync(alloc, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace gqc
