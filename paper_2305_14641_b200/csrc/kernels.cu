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

#include <cub/device/device_scan.cuh>

#include "gqc_internal.h"

namespace gqc {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ int exp_field(double x) { return (__double2hiint(x) >> 20) & 0x7ff; }
// 2^(f - 1023) for a biased exponent f in [1, 2046]
__device__ __forceinline__ double pow2_field(int f) { return __hiloint2double(f << 20, 0); }

// ---------------------------------------------------------------------------
// Exact fast-forward of L sequential adds s <- fl(s + c), s >= 0, c >= 0.
//
// Inside a binade [base, 2 base) of s (unit in the last place u = base*2^-52;
// the subnormals share u = 2^-1074 with [2^-1022, 2^-1021) and are treated as
// that binade), an add whose exact result stays <= 2 base rounds on the
// u-grid, so fl(s + c) = s + inc with inc = round_u(c). round_u(c) can depend
// on the parity of s/u only when c is an exact half-ulp tie, and a tie always
// lands on an even multiple, after which the increment is constant. inc is
// read off an even reference point, inc = fl(base + c) - base; odd s with a
// tie takes one real step first. Then m = floor((2 base - u - s) / inc) steps
// are all exact grid steps (their exact sums stay below 2 base - u/2) and are
// taken at once; the binade crossing itself is always a real add. c >= base/2
// (at most two adds per binade) and inc == 0 (a fixed point after at most one
// real add) are handled by real adds. Work: O(number of binades crossed).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ff_chain(double s, const double c, int L) {
    if (c == 0.0) return s;
    while (L > 0) {
        const int f = max(exp_field(s), 1);
        const double base = pow2_field(f);
        if (!(c < __dmul_rn(base, 0.5))) {
            s = __dadd_rn(s, c);
            --L;
            continue;
        }
        const double inc = __dsub_rn(__dadd_rn(base, c), base);
        if (inc == 0.0) return __dadd_rn(s, c);
        const double u = __dmul_rn(base, 0x1p-52);
        if (__double2loint(s) & 1) {
            const double bo = __dadd_rn(base, u);
            if (__dsub_rn(__dadd_rn(bo, c), bo) != inc) {  // half-ulp tie: settle parity
                s = __dadd_rn(s, c);
                --L;
                continue;
            }
        }
        const double room = __dsub_rn(__dsub_rn(__dadd_rn(base, base), s), u);
        if (room < inc) {  // crossing into the next binade
            s = __dadd_rn(s, c);
            --L;
            continue;
        }
        double m = floor(__ddiv_rn(room, inc));
        m = fmin(m, static_cast<double>(L));
        if (__fma_rn(-m, inc, room) < 0.0) m = m - 1.0;  // exact sign of room - m*inc
        s = __dadd_rn(s, __dmul_rn(m, inc));               // exact: a u-grid point below 2 base
        L -= static_cast<int>(m);
    }
    return s;
}

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

template <bool kFF>
__device__ __forceinline__ void run(double& num, double& den, const double p, const double e, const int L) {
    if (L <= 0) return;
    if constexpr (kFF) {
        num = ff_chain(num, p, L);
        den = ff_chain(den, e, L);
    } else {
        replay(num, den, p, e, L);
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
// Potential kernel: thread = (row, sigma), sigma fastest, so the lanes of a
// warp share one CSR row (broadcast loads) and write one contiguous node-major
// slice of V. Grid: ceil(rows * n_sigma / 256) blocks of 256 threads.
// ---------------------------------------------------------------------------
template <bool kFF, int kW>
__global__ void __launch_bounds__(kBlock) potential_kernel(const __grid_constant__ PotentialLaunch P) {
    __shared__ double sc[kSigmaFields][kMaxSigmaPerLaunch];
    for (int idx = threadIdx.x; idx < kSigmaFields * kMaxSigmaPerLaunch; idx += blockDim.x) {
        const int ss = idx % kMaxSigmaPerLaunch, f = idx / kMaxSigmaPerLaunch;
        if (ss < P.n_sigma) sc[f][ss] = reinterpret_cast<const double*>(&P.c[ss])[f];
    }
    __syncthreads();

    const int S = P.n_sigma;
    const long long tid = static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x;
    const int s = static_cast<int>(tid % S);
    const long long r64 = P.row_begin + tid / S;
    if (r64 >= P.row_end) return;
    const int i = static_cast<int>(r64);

    const double inv = sc[0][s], neg_inv = sc[1][s];
    const double eW = sc[2][s], pW = sc[3][s];
    const double e1 = sc[4][s], p1 = sc[5][s];
    const double eWt = sc[6][s], pWt = sc[7][s];
    const double e1t = sc[8][s], p1t = sc[9][s];

    const int n = P.n;
    const bool tail = P.tail != 0;
    const long long kend = P.offsets[i + 1];
    long long k = P.offsets[i];
    double num = 0.0, den = 0.0;
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
        // non-adjacent run over [pos, col)
        const int L = col - pos;
        if (L > 0) {
            if (tail && col == n) {
                run<kFF>(num, den, pW, eW, L - 1);
                num = __dadd_rn(num, pWt);
                den = __dadd_rn(den, eWt);
            } else {
                run<kFF>(num, den, pW, eW, L);
            }
        }
        if (kind == 0) break;
        if (kind == 1) {  // self: d2 = 0, exp(-0) = 1 -> num += 0, den += 1
            den = __dadd_rn(den, 1.0);
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
            e = at_tail ? e1t : e1;
            p = at_tail ? p1t : p1;
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
                    e = pexp_dev(__dmul_rn(neg_inv, d2));
                }
            }
            p = __dmul_rn(d2, e);
        }
        run<kFF>(num, den, p, e, end - col);
        k = kk;
        pos = end;
    }
    P.out[static_cast<long long>(i - P.row_begin) * P.out_ld + P.out_col0 + s] = __dmul_rn(inv, __ddiv_rn(num, den));
}

// ---------------------------------------------------------------------------
// K3: successor = lexicographic (v, id) argmin over the closed neighbourhood
// (ggd.cpp:7-24). Thread = (row, sigma), sigma fastest: a neighbour's
// potentials for all sigmas are one contiguous node-major line.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) successors_kernel(int n, const long long* __restrict__ off,
                                                            const int* __restrict__ nbr,
                                                            const double* __restrict__ v, int S,
                                                            int* __restrict__ succ_sm) {
    const long long tid = static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x;
    const int s = static_cast<int>(tid % S);
    const long long i64 = tid / S;
    if (i64 >= n) return;
    const int i = static_cast<int>(i64);
    int best = i;
    double vb = __ldg(v + i64 * S + s);
    const long long kend = off[i + 1];
    for (long long k = off[i]; k < kend; ++k) {
        const int j = __ldg(nbr + k);
        const double vj = __ldg(v + static_cast<long long>(j) * S + s);
        if (vj < vb || (vj == vb && j < best)) {
            best = j;
            vb = vj;
        }
    }
    succ_sm[static_cast<long long>(s) * n + i] = best;
}

// K4: chase successors to their fixed point. center[] starts as a copy of
// succ; every thread follows pointers through center[], which other threads
// overwrite with roots as they finish (any value read is an ancestor, so the
// result is exact; finished neighbours shorten the walk). Maps built by K3
// strictly decrease (v, id) along a chain, so every walk terminates.
__global__ void __launch_bounds__(kBlock) chase_kernel(int n, int* __restrict__ center) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    int* c = center + static_cast<long long>(blockIdx.y) * n;
    int x = c[i];
    for (;;) {
        const int y = c[x];
        if (y == x) break;
        x = y;
    }
    c[i] = x;
}

// K5a: center flags for the dense relabel scan (flag[S*n] = 0 terminator).
__global__ void __launch_bounds__(kBlock) center_flags_kernel(int n, int S, const int* __restrict__ center,
                                                              int* __restrict__ flag) {
    const long long t = static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x;
    const long long total = static_cast<long long>(n) * S;
    if (t < total) flag[t] = center[t] == static_cast<int>(t % n) ? 1 : 0;
    else if (t == total) flag[t] = 0;
}

// K5b: cluster_index = rank of the center among ascending centers.
__global__ void __launch_bounds__(kBlock) relabel_kernel(int n, const int* __restrict__ center,
                                                         const int* __restrict__ scan, int* __restrict__ ci,
                                                         int* __restrict__ num_clusters) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const long long b = static_cast<long long>(blockIdx.y) * n;
    if (i < n) ci[b + i] = scan[b + center[b + i]] - scan[b];
    if (i == 0) num_clusters[blockIdx.y] = scan[b + n] - scan[b];
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

}  // namespace

int launch_potentials(const PotentialLaunch& p, int kernel, void* stream) {
    const long long threads = static_cast<long long>(p.row_end - p.row_begin) * p.n_sigma;
    if (threads <= 0) return cudaSuccess;
    auto st = static_cast<cudaStream_t>(stream);
    const dim3 grid(grid_for(threads));
    const bool ff = kernel == 0;
    switch (p.weight_mode) {
        case kUnit:
            if (ff) potential_kernel<true, kUnit><<<grid, kBlock, 0, st>>>(p);
            else potential_kernel<false, kUnit><<<grid, kBlock, 0, st>>>(p);
            break;
        case kDevicePexp:
            if (ff) potential_kernel<true, kDevicePexp><<<grid, kBlock, 0, st>>>(p);
            else potential_kernel<false, kDevicePexp><<<grid, kBlock, 0, st>>>(p);
            break;
        default:
            if (ff) potential_kernel<true, kEntryTable><<<grid, kBlock, 0, st>>>(p);
            else potential_kernel<false, kEntryTable><<<grid, kBlock, 0, st>>>(p);
            break;
    }
    count_launch();
    return cudaGetLastError();
}

int launch_successors(int n, const std::int64_t* offsets, const std::int32_t* nbr, const double* v, int n_sigma,
                      std::int32_t* succ_sm, void* stream) {
    const long long threads = static_cast<long long>(n) * n_sigma;
    successors_kernel<<<grid_for(threads), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
        n, reinterpret_cast<const long long*>(offsets), nbr, v, n_sigma, succ_sm);
    count_launch();
    return cudaGetLastError();
}

int launch_chase(int n, int n_sigma, const std::int32_t* succ_sm, std::int32_t* center_sm, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    if (succ_sm != center_sm)
        e = cudaMemcpyAsync(center_sm, succ_sm, sizeof(int) * static_cast<size_t>(n) * n_sigma,
                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    chase_kernel<<<dim3(grid_for(n), n_sigma), kBlock, 0, st>>>(n, center_sm);
    count_launch();
    return cudaGetLastError();
}

std::size_t labels_workspace_bytes(int n, int n_sigma) {
    const long long items = static_cast<long long>(n) * n_sigma + 1;
    std::size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  items);
    auto align = [](std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); };
    return 2 * align(sizeof(int) * items) + align(temp);
}

int launch_labels(int n, int n_sigma, const std::int32_t* center_sm, std::int32_t* ci_sm, std::int32_t* num_clusters,
                  void* workspace, std::size_t ws_bytes, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    const long long items = static_cast<long long>(n) * n_sigma + 1;
    auto align = [](std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); };
    char* w = static_cast<char*>(workspace);
    int* flag = reinterpret_cast<int*>(w);
    int* scan = reinterpret_cast<int*>(w + align(sizeof(int) * items));
    void* temp = w + 2 * align(sizeof(int) * items);
    std::size_t temp_bytes = ws_bytes - 2 * align(sizeof(int) * items);
    center_flags_kernel<<<grid_for(items), kBlock, 0, st>>>(n, n_sigma, center_sm, flag);
    count_launch();
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flag, scan, items, st);
    count_launch(2);  // CUB: init + scan kernels
    if (e != cudaSuccess) return e;
    relabel_kernel<<<dim3(grid_for(n), n_sigma), kBlock, 0, st>>>(n, center_sm, scan, ci_sm, num_clusters);
    count_launch();
    return cudaGetLastError();
}

int launch_transpose(const double* v_nm, int n, int n_sigma, double* v_sm, void* stream) {
    const dim3 grid((n + 31) / 32, (n_sigma + 31) / 32);
    transpose_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(v_nm, n, n_sigma, v_sm);
    count_launch();
    return cudaGetLastError();
}

int resolve_checked(int n, const std::int32_t* succ_dev, std::int32_t* center_dev, std::int32_t* ci_dev,
                    std::int32_t* num_clusters_host, int* err_kind, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    int *p0, *t0, *p1, *t1, *nc;
    unsigned long long* first;
    const std::size_t bytes = sizeof(int) * static_cast<std::size_t>(n);
    cudaError_t e = cudaMallocAsync(&p0, bytes * 4 + 64, st);
    if (e != cudaSuccess) return e;
    int* const alloc = p0;
    t0 = p0 + n;
    p1 = t0 + n;
    t1 = p1 + n;
    first = reinterpret_cast<unsigned long long*>(t1 + n + (n & 1));
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
        e = cudaMallocAsync(&wsp, ws, st);
        if (e == cudaSuccess) {
            e = static_cast<cudaError_t>(launch_labels(n, 1, center_dev, ci_dev, nc, wsp, ws, st));
            cudaMemcpyAsync(num_clusters_host, nc, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaFreeAsync(wsp, st);
        }
    }
    cudaFreeAsync(alloc, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace gqc
