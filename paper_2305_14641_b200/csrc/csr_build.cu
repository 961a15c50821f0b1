// Device CSR construction for edge-list ingestion: the
// reference builds graphqc::Graph's CSR with a std::map per node
// (graph.cpp:25-71); here the same CSR comes from two radix sorts on the
// device.
//
//   1. validate every edge in input order (first offender decides: endpoint
//      out of range before non-positive weight, graph.cpp:33-39);
//   2. key each non-loop edge by its undirected pair (min, max) and sort
//      stably, so the first edge of every run of equal keys is the input's
//      first occurrence: keep-first dedup (graph.cpp:40-52); a later
//      duplicate with a different weight is reported back (the caller prints
//      the reference's warning in input order);
//   3. emit both directions of every kept edge keyed (row, col) and sort:
//      rows come out with ascending neighbour ids, exactly the order of the
//      reference's std::map iteration (graph.cpp:64-70).
//
// Pure integer / copy work; HBM-bound radix sorts (CUB onesweep).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gqc_internal.h"

namespace gqc {
namespace {

constexpr int kB = 256;

int blocks_for(long long items) { return static_cast<int>(std::max<long long>(1, (items + kB - 1) / kB)); }

// first[0] = min over offending edges of (k << 1 | kind), kind 0 = endpoint
// out of range, 1 = non-positive weight (checked in that order per edge).
__global__ void validate_kernel(const GqcEdge* __restrict__ e, long long m, int n,
                                unsigned long long* __restrict__ first) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= m) return;
    const GqcEdge x = e[k];
    unsigned long long code = ~0ull;
    if (x.u < 0 || x.u >= n || x.v < 0 || x.v >= n) code = static_cast<unsigned long long>(k) << 1;
    else if (x.w <= 0.0) code = (static_cast<unsigned long long>(k) << 1) | 1ull;
    if (code != ~0ull) atomicMin(first, code);
}

// key = min << b | max for non-loop edges, the all-ones sentinel for loops
// (sorts after every real pair); val = input index.
__global__ void pair_key_kernel(const GqcEdge* __restrict__ e, long long m, int b, unsigned long long* __restrict__ key,
                                unsigned* __restrict__ val) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= m) return;
    const GqcEdge x = e[k];
    const unsigned long long lo = static_cast<unsigned>(min(x.u, x.v)), hi = static_cast<unsigned>(max(x.u, x.v));
    key[k] = x.u == x.v ? (1ull << (2 * b)) - 1 : (lo << b) | hi;
    val[k] = static_cast<unsigned>(k);
}

// head[k] = 1 for the first (kept) edge of every run of equal pairs;
// run_head[k] = position of the run's first element (for the conflict check).
__global__ void head_kernel(const unsigned long long* __restrict__ key, long long m, unsigned long long sentinel,
                            int* __restrict__ head, long long* __restrict__ pos) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= m) return;
    const bool h = key[k] != sentinel && (k == 0 || key[k] != key[k - 1]);
    head[k] = h ? 1 : 0;
    pos[k] = h ? k : -1;
}

struct MaxOp {
    __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};

// Dropped duplicates whose weight differs from the kept edge's: (dropped, kept) input indices.
__global__ void conflict_kernel(const unsigned long long* __restrict__ key, const unsigned* __restrict__ val,
                                const long long* __restrict__ run_pos, long long m, unsigned long long sentinel,
                                const GqcEdge* __restrict__ e, long long* __restrict__ out, long long cap,
                                unsigned long long* __restrict__ count) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= m || key[k] == sentinel || run_pos[k] == k) return;
    const unsigned kept = val[run_pos[k]], dropped = val[k];
    if (e[dropped].w != e[kept].w) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if (static_cast<long long>(slot) < cap) {
            out[2 * slot] = dropped;
            out[2 * slot + 1] = kept;
        }
    }
}

// Both directions of every kept edge: (row << b | col, weight); degrees.
__global__ void directed_kernel(const unsigned long long* __restrict__ key, const unsigned* __restrict__ val,
                                const int* __restrict__ head, const int* __restrict__ slot, long long m, int b,
                                const GqcEdge* __restrict__ e, unsigned long long* __restrict__ dkey,
                                double* __restrict__ dw, unsigned long long* __restrict__ deg) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= m || !head[k]) return;
    const unsigned long long mask = (1ull << b) - 1;
    const unsigned long long lo = key[k] >> b, hi = key[k] & mask;
    const double w = e[val[k]].w;
    const long long j = slot[k];
    dkey[2 * j] = (lo << b) | hi;
    dw[2 * j] = w;
    dkey[2 * j + 1] = (hi << b) | lo;
    dw[2 * j + 1] = w;
    atomicAdd(deg + lo, 1ull);
    atomicAdd(deg + hi, 1ull);
}

__global__ void unpack_kernel(const unsigned long long* __restrict__ dkey, long long nnz, int b, int* __restrict__ nbr,
                              const double* __restrict__ dw, int* __restrict__ not_unit) {
    const long long k = static_cast<long long>(blockIdx.x) * kB + threadIdx.x;
    if (k >= nnz) return;
    nbr[k] = static_cast<int>(dkey[k] & ((1ull << b) - 1));
    if (dw[k] != 1.0) *not_unit = 1;
}

}  // namespace

int build_csr_device(int n, long long m, const GqcEdge* host_edges, std::int64_t* offsets, std::int32_t* nbr,
                     double* w_out, long long* nnz_out, std::vector<long long>* conflicts, int* unit_out,
                     long long* first_error, void* pool_, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    auto pool = static_cast<cudaMemPool_t>(pool_);
    int b = 1;
    while ((1ll << b) < n) ++b;  // node ids fit b bits; keys use 2b bits
    const unsigned long long sentinel = (1ull << (2 * b)) - 1;
    cudaError_t e = cudaSuccess;
    std::vector<void*> allocs;
    auto alloc = [&](std::size_t bytes) -> void* {
        void* p = nullptr;
        if (e == cudaSuccess) e = cudaMallocFromPoolAsync(&p, std::max<std::size_t>(bytes, 256), pool, st);
        if (e == cudaSuccess) allocs.push_back(p);
        return p;
    };
    auto release = [&] {
        for (void* p : allocs) cudaFreeAsync(p, st);
        allocs.clear();
    };
    auto* d_e = static_cast<GqcEdge*>(alloc(sizeof(GqcEdge) * m));
    auto* first = static_cast<unsigned long long*>(alloc(4 * sizeof(unsigned long long)));
    auto* key = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * m));
    auto* key2 = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * m));
    auto* val = static_cast<unsigned*>(alloc(sizeof(unsigned) * m));
    auto* val2 = static_cast<unsigned*>(alloc(sizeof(unsigned) * m));
    if (e != cudaSuccess) {
        release();
        return e;
    }
    e = cudaMemcpyAsync(d_e, host_edges, sizeof(GqcEdge) * m, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(first + 1, 0, 3 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) {
        release();
        return e;
    }
    validate_kernel<<<blocks_for(m), kB, 0, st>>>(d_e, m, n, first);
    pair_key_kernel<<<blocks_for(m), kB, 0, st>>>(d_e, m, b, key, val);
    count_launch(2);
    {
        std::size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, val, val2, m, 0, 2 * b, st);
        void* temp = alloc(tb);
        if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(temp, tb, key, key2, val, val2, m, 0, 2 * b, st);
        count_launch(4);
    }
    // heads, kept-edge slots, run heads
    auto* head = static_cast<int*>(alloc(sizeof(int) * (m + 1)));
    auto* slot = static_cast<int*>(alloc(sizeof(int) * (m + 1)));
    auto* pos = static_cast<long long*>(alloc(sizeof(long long) * m));
    auto* run_pos = static_cast<long long*>(alloc(sizeof(long long) * m));
    if (e != cudaSuccess) {
        release();
        return e;
    }
    head_kernel<<<blocks_for(m), kB, 0, st>>>(key2, m, sentinel, head, pos);
    cudaMemsetAsync(head + m, 0, sizeof(int), st);
    count_launch(2);
    {
        std::size_t t1 = 0, t2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, t1, head, slot, m + 1, st);
        cub::DeviceScan::InclusiveScan(nullptr, t2, pos, run_pos, MaxOp{}, m, st);
        void* temp = alloc(std::max(t1, t2));
        if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, t1, head, slot, m + 1, st);
        if (e == cudaSuccess) e = cub::DeviceScan::InclusiveScan(temp, t2, pos, run_pos, MaxOp{}, m, st);
        count_launch(4);
    }
    const long long cap = conflicts ? 1 << 20 : 0;
    auto* conf = static_cast<long long*>(alloc(sizeof(long long) * 2 * std::max<long long>(cap, 1)));
    if (e != cudaSuccess) {
        release();
        return e;
    }
    if (conflicts) {
        conflict_kernel<<<blocks_for(m), kB, 0, st>>>(key2, val2, run_pos, m, sentinel, d_e, conf, cap, first + 1);
        count_launch();
    }
    // unique edge count -> nnz
    int kept = 0;
    unsigned long long hfirst[2] = {0, 0};
    e = cudaMemcpyAsync(&kept, slot + m, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hfirst, first, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        release();
        return e;
    }
    *first_error = hfirst[0] == ~0ull ? -1 : static_cast<long long>(hfirst[0]);
    if (*first_error >= 0) {  // the caller raises the reference's exception for that edge
        release();
        return cudaStreamSynchronize(st);
    }
    const long long nnz = 2ll * kept;
    *nnz_out = nnz;
    auto* dkey = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * std::max<long long>(nnz, 1)));
    auto* dkey2 = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * std::max<long long>(nnz, 1)));
    auto* dw = static_cast<double*>(alloc(sizeof(double) * std::max<long long>(nnz, 1)));
    auto* dw2 = static_cast<double*>(alloc(sizeof(double) * std::max<long long>(nnz, 1)));
    auto* deg = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * (n + 1)));
    auto* off = static_cast<unsigned long long*>(alloc(sizeof(unsigned long long) * (n + 1)));
    auto* d_nbr = static_cast<int*>(alloc(sizeof(int) * std::max<long long>(nnz, 1)));
    auto* not_unit = static_cast<int*>(alloc(sizeof(int)));
    if (e != cudaSuccess) {
        release();
        return e;
    }
    cudaMemsetAsync(deg, 0, sizeof(unsigned long long) * (n + 1), st);
    cudaMemsetAsync(not_unit, 0, sizeof(int), st);
    directed_kernel<<<blocks_for(m), kB, 0, st>>>(key2, val2, head, slot, m, b, d_e, dkey, dw, deg);
    count_launch(3);
    if (nnz > 0) {
        std::size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, dkey, dkey2, dw, dw2, nnz, 0, 2 * b, st);
        void* temp = alloc(tb);
        if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(temp, tb, dkey, dkey2, dw, dw2, nnz, 0, 2 * b, st);
        count_launch(4);
    }
    {
        std::size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, n + 1, st);
        void* temp = alloc(tb);
        if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, tb, deg, off, n + 1, st);
        count_launch(2);
    }
    if (e != cudaSuccess) {
        release();
        return e;
    }
    if (nnz > 0) {
        unpack_kernel<<<blocks_for(nnz), kB, 0, st>>>(dkey2, nnz, b, d_nbr, dw2, not_unit);
        count_launch();
    }
    int h_not_unit = 0;
    unsigned long long n_conf = 0;
    e = cudaMemcpyAsync(offsets, off, sizeof(std::int64_t) * (n + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(nbr, d_nbr, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && nnz > 0 && w_out)
        e = cudaMemcpyAsync(w_out, dw2, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_not_unit, not_unit, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&n_conf, first + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && conflicts) {
        const long long got = std::min<long long>(static_cast<long long>(n_conf), cap);
        conflicts->resize(2 * got);
        if (got > 0)
            e = cudaMemcpy(conflicts->data(), conf, sizeof(long long) * 2 * got, cudaMemcpyDeviceToHost);
        if (static_cast<long long>(n_conf) > cap) conflicts->push_back(-1);  // overflow: the caller falls back
    }
    *unit_out = h_not_unit ? 0 : 1;
    release();
    const cudaError_t e2 = cudaStreamSynchronize(st);
    return e != cudaSuccess ? e : e2;
}

}  // namespace gqc
