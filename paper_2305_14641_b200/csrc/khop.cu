// k-hop distance extension of the potential sweep (opt-in, GQC_OPT_HOP_CAP).
//
// NOT in the reference: its distance is hop-capped at 1 (graph.cpp:258-267,
// SPEC.md:69-77). This is SURVEY §8(f) row 4, the north star's "multi-source
// BFS hop distances over CSR": on a unit-weight graph d(i,j) = 0 for j == i,
// the BFS hop count h for 1 <= h <= K, and W beyond K or when unreachable.
// K = 1 is exactly the reference's distance (and runs the main kernels). The
// per-row sums keep the reference's contract unchanged: ascending j, fp64,
// Eigen packet exp + glibc tail column (oracle.cpp fill_khop is the checker).
//
// Pipeline per launch (rows [row_begin, row_end)):
//   1. K >= 3: khop_expand_kernel<false>: BFS from every source row to depth
//      K with the visited set as a bitset in shared memory (one per block;
//      global memory when N bits do not fit): warp-per-frontier-vertex
//      expansion, each neighbour row read as coalesced 32-wide chunks,
//      atomicOr into the bitset, and warp-ballot compaction of the newly
//      reached columns into the next frontier. Counts the nodes at hops 2..K
//      per row. K = 2: no BFS, the sum of the neighbours' degrees bounds the
//      count (khop_bound_kernel);
//   2. exclusive scan of the counts -> event offsets (int64);
//   3. khop_expand_kernel<true>: the same BFS, writing each row's hop >= 2
//      nodes as events (col << 3 | hop) into its segment, and the count;
//   4. cub segmented sort of the events by column (row segments);
//   5. khop_walk_kernel: warp = one row x 32 sigma lanes, the same exact
//      run fast-forward as the main kernel (ff_chain.cuh) over the merge of
//      the CSR row (hop 1) and the sorted events (hop >= 2), longest rows
//      first. Rows are processed in batches that bound the event memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <vector>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "gqc_internal.h"
#include "ff_chain.cuh"

namespace gqc {
namespace {

using namespace gqc::ffc;

constexpr int kExpandThreads = 512;
constexpr int kWalkBlock = 256;
constexpr int kWalkBlocksPerSM = 4;
constexpr unsigned kFull = 0xffffffffu;
// Shared-memory bitset limit per block (bits of N): N <= 1.6M keeps it on chip.
constexpr std::size_t kSmemBitsetBytes = 200 * 1024;
// Events held in device memory at once (keys + sorted keys): 2 x 4 B each.
constexpr long long kEventBudget = 1ll << 30;
// On-chip sorted emission (hop cap 2): rows with at most kSortCap candidates.
// Two sizes: 128 x 4 (<= 512 candidates) and 256 x 8 (<= 2048).
constexpr long long kSortCap0 = 128 * 4, kSortCap1 = 256 * 8;

struct KhopExpand {
    int n;
    const long long* off;
    const int* nbr;
    int row_begin, rows;  // this pass covers rows [row_begin, row_begin + rows)
    int K;
    int* counter;              // row queue
    long long* count;          // events of each row, hops 1..K (both passes write it)
    const long long* ev_off;   // fill pass: event offset of each row (absolute)
    long long ev_base;         // fill pass: ev_off value of the pass's first row
    unsigned* ev;              // fill pass: events (col << 3 | hop), relative to ev_base
    unsigned* scratch;         // count pass: [gridDim.x][n] per-block level lists
    unsigned* gbits;           // [gridDim.x][words] global bitsets, or nullptr (shared)
    int words;
    const int* list;           // hop cap 2 emission: the pass's rows (pass-relative), or nullptr = all
    const int* list_len;
};

template <bool kFill>
__global__ void __launch_bounds__(kExpandThreads) khop_expand_kernel(const KhopExpand E) {
    extern __shared__ unsigned sbits[];
    __shared__ int s_row, s_pos;
    unsigned* bits = E.gbits ? E.gbits + static_cast<std::size_t>(blockIdx.x) * E.words : sbits;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int w = tid; w < E.words; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    for (;;) {
        if (tid == 0) s_row = atomicAdd(E.counter, 1);
        __syncthreads();
        const int r = s_row;
        if (r >= E.rows) break;
        const int i = E.row_begin + r;
        const long long kb = E.off[i], ke = E.off[i + 1];
        const int deg = static_cast<int>(ke - kb);
        unsigned* dst = kFill ? E.ev + (E.ev_off[r] - E.ev_base)
                              : E.scratch + static_cast<std::size_t>(blockIdx.x) * E.n;
        // hop 0 and 1: the row itself and its CSR neighbours (the hop-1
        // events open the row's list; deeper levels are appended after them)
        if (tid == 0) {
            atomicOr(&bits[i >> 5], 1u << (i & 31));
            s_pos = deg;
        }
        for (long long k = kb + tid; k < ke; k += blockDim.x) {
            const int c = E.nbr[k];
            atomicOr(&bits[c >> 5], 1u << (c & 31));
            dst[k - kb] = (static_cast<unsigned>(c) << 3) | 1u;
        }
        __syncthreads();
        int lvl_b = deg, lvl_e = deg;
        for (int h = 2; h <= E.K; ++h) {
            const long long nf = (h == 2) ? (ke - kb) : (lvl_e - lvl_b);
            // warp per frontier vertex: its row in coalesced 32-wide chunks
            for (long long f = warp; f < nf; f += nwarps) {
                const int u = (h == 2) ? E.nbr[kb + f] : static_cast<int>(dst[lvl_b + f] >> 3);
                const long long ub = E.off[u], ue = E.off[u + 1];
                for (long long k = ub; k < ue; k += 32) {
                    const bool valid = k + lane < ue;
                    const int c = valid ? E.nbr[k + lane] : 0;
                    bool fresh = false;
                    if (valid) {
                        const unsigned bit = 1u << (c & 31);
                        fresh = !(atomicOr(&bits[c >> 5], bit) & bit);
                    }
                    const unsigned m = __ballot_sync(kFull, fresh);
                    if (m) {  // ballot compaction of the newly reached columns
                        int base = 0;
                        if (lane == 0) base = atomicAdd(&s_pos, __popc(m));
                        base = __shfl_sync(kFull, base, 0);
                        if (fresh) dst[base + __popc(m & ((1u << lane) - 1u))] = (static_cast<unsigned>(c) << 3) | h;
                    }
                }
            }
            __syncthreads();
            lvl_b = lvl_e;
            lvl_e = s_pos;
            __syncthreads();  // every thread has read s_pos before the next level appends
        }
        if (tid == 0) E.count[r] = lvl_e;
        // clear the words this row touched
        if (tid == 0) bits[i >> 5] = 0u;
        for (long long k = kb + tid; k < ke; k += blockDim.x) bits[E.nbr[k] >> 5] = 0u;
        for (int q = tid; q < lvl_e; q += blockDim.x) bits[(dst[q] >> 3) >> 5] = 0u;
        __syncthreads();
    }
}

// Hop cap 2, rows whose candidates (the CSR row plus every neighbour's row)
// fit kThreads * kItems: block per row with everything on chip and many rows
// in flight per SM (the bitset kernel below holds one N-bit row per SM). The
// candidates are gathered into shared memory as (col << 1 | 0) for the row's
// own neighbours and (col << 1 | 1) for its neighbours' neighbours (warp per
// neighbour, coalesced), block radix sorted (cub::BlockRadixSort, bits of N
// plus one), and the first entry of every column other than the row itself
// is kept: hop 1 when the row lists it, else hop 2. A block scan places the
// events, already in column order.
template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads) khop2_sort_kernel(const KhopExpand E, int end_bit) {
    constexpr int kCap = kThreads * kItems;
    constexpr int kWarps = kThreads / 32;
    using Sort = cub::BlockRadixSort<unsigned, kThreads, kItems>;
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ unsigned keys[kCap];
    __shared__ int s_row, s_cnt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nrows = *E.list_len;
    for (;;) {
        if (tid == 0) s_row = atomicAdd(E.counter, 1);
        __syncthreads();
        const int idx = s_row;
        if (idx >= nrows) break;
        const int r = E.list[idx];
        const int i = E.row_begin + r;
        const long long kb = E.off[i];
        const int deg = static_cast<int>(E.off[i + 1] - kb);  // deg + sum of their degrees <= kCap
        if (tid == 0) s_cnt = deg;
        for (int k = tid; k < deg; k += kThreads) keys[k] = static_cast<unsigned>(E.nbr[kb + k]) << 1;
        __syncthreads();
        for (int f = warp; f < deg; f += kWarps) {  // warp per neighbour
            const int u = static_cast<int>(keys[f] >> 1);
            const long long ub = E.off[u], ue = E.off[u + 1];
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_cnt, static_cast<int>(ue - ub));
            base = __shfl_sync(kFull, base, 0);
            for (long long k = ub + lane; k < ue; k += 32)
                keys[base + (k - ub)] = (static_cast<unsigned>(E.nbr[k]) << 1) | 1u;
        }
        __syncthreads();
        const int cnt = s_cnt;
        unsigned item[kItems];
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const int p = tid * kItems + q;
            item[q] = p < cnt ? keys[p] : 0xffffffffu;  // padding sorts last (low end_bit bits all ones)
        }
        Sort(tmp.sort).Sort(item, 0, end_bit);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kItems; ++q) keys[tid * kItems + q] = item[q];
        __syncthreads();
        bool keep[kItems];
        int nkeep = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const int p = tid * kItems + q;
            const unsigned c = item[q] >> 1;
            keep[q] = p < cnt && c != static_cast<unsigned>(i) && (p == 0 || (keys[p - 1] >> 1) != c);
            nkeep += keep[q];
        }
        int pos = 0, total = 0;
        Scan(tmp.scan).ExclusiveSum(nkeep, pos, total);
        unsigned* dst = E.ev + (E.ev_off[r] - E.ev_base);
#pragma unroll
        for (int q = 0; q < kItems; ++q)
            if (keep[q]) dst[pos++] = ((item[q] >> 1) << 3) | ((item[q] & 1u) ? 2u : 1u);
        if (tid == 0) E.count[r] = total;
        __syncthreads();
    }
}

// Rows of a pass split by their candidate bound: <= cap0 and <= cap1 to the
// two sort-kernel sizes, the rest to the bitset kernel (warp-aggregated
// appends into lists[0..2], lengths in lens[0..2]).
__global__ void khop_split_kernel(const long long* __restrict__ ev_off, int rows, long long cap0, long long cap1,
                                  int* __restrict__ list0, int* __restrict__ list1, int* __restrict__ list2,
                                  int* __restrict__ lens) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool valid = r < rows;
    const long long b = valid ? ev_off[r + 1] - ev_off[r] : 0;
    const int cls = !valid ? -1 : (b <= cap0 ? 0 : (b <= cap1 ? 1 : 2));
    int* lists[3] = {list0, list1, list2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const unsigned m = __ballot_sync(kFull, cls == c);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(&lens[c], __popc(m));
        base = __shfl_sync(kFull, base, 0);
        if (cls == c) lists[c][base + __popc(m & ((1u << lane) - 1u))] = r;
    }
}

// Hop cap 2 with the bitset on chip: the events are emitted already sorted.
// Block per source row (rows from a queue): the row's own neighbours and
// every neighbour's row are OR-ed into the shared-memory bitset (warp per
// neighbour, coalesced 32-wide chunks; a word that turns non-zero also sets
// its bit in a summary bitset, one bit per word), the row itself is cleared,
// and the summary is walked in column order: thread t owns a contiguous run
// of summary words, counts the columns under them, a block scan gives each
// thread its output position, and it writes its columns ascending (hop 1 when
// the CSR row lists it, by binary search, else hop 2) and zeroes what it
// visited. Work per row is proportional to its events, not to N; no per-row
// sort and no second BFS.
template <int kThreads>
__global__ void __launch_bounds__(kThreads) khop2_emit_kernel(const KhopExpand E) {
    extern __shared__ unsigned bits[];  // [words] bitset, then [swords] summary
    __shared__ int s_row;
    __shared__ int s_warp[kThreads / 32];
    constexpr int kRowCap = 2048;  // the CSR row is staged here for the hop-1 tags (longer rows: global)
    __shared__ int row_s[kRowCap];
    constexpr int kWarps = kThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int swords = (E.words + 31) >> 5;
    unsigned* summ = bits + E.words;
    const int spt = (swords + kThreads - 1) / kThreads;  // summary words per thread
    for (int w = tid; w < E.words + swords; w += kThreads) bits[w] = 0u;
    __syncthreads();
    const int nrows = E.list ? *E.list_len : E.rows;
    for (;;) {
        if (tid == 0) s_row = atomicAdd(E.counter, 1);
        __syncthreads();
        const int idx = s_row;
        if (idx >= nrows) break;
        const int r = E.list ? E.list[idx] : idx;
        const int i = E.row_begin + r;
        const long long kb = E.off[i], ke = E.off[i + 1];
        for (long long f = warp; f < ke - kb; f += kWarps) {  // warp per neighbour
            const int u = E.nbr[kb + f];
            const long long ub = E.off[u], ue = E.off[u + 1];
            for (long long k = ub + lane; k < ue; k += 32) {
                const int c = E.nbr[k];
                const int x = c >> 5;
                if (atomicOr(&bits[x], 1u << (c & 31)) == 0u) atomicOr(&summ[x >> 5], 1u << (x & 31));
            }
        }
        __syncthreads();
        const int deg = static_cast<int>(ke - kb);
        for (long long k = kb + tid; k < ke; k += kThreads) {  // hop 1 (not every neighbour is 2 hops away)
            const int c = E.nbr[k];
            const int x = c >> 5;
            if (atomicOr(&bits[x], 1u << (c & 31)) == 0u) atomicOr(&summ[x >> 5], 1u << (x & 31));
            if (deg <= kRowCap) row_s[k - kb] = c;
        }
        __syncthreads();
        if (tid == 0) atomicAnd(&bits[i >> 5], ~(1u << (i & 31)));
        __syncthreads();
        // count the columns under this thread's summary words
        const int s0 = tid * spt, s1 = min(swords, s0 + spt);
        int cnt = 0;
        for (int sw = s0; sw < s1; ++sw) {
            unsigned m = summ[sw];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                cnt += __popc(bits[(sw << 5) + b]);
            }
        }
        // block exclusive scan of the counts
        int incl = cnt;
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int v = lane < kWarps ? s_warp[lane] : 0;
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(kFull, v, d);
                if (lane >= d) v += t;
            }
            if (lane < kWarps) s_warp[lane] = v;  // inclusive warp totals
        }
        __syncthreads();
        int pos = incl - cnt + (warp ? s_warp[warp - 1] : 0);
        unsigned* dst = E.ev + (E.ev_off[r] - E.ev_base);
        const int* rowp = deg <= kRowCap ? row_s : E.nbr + kb;
        int cur = -1;  // cursor into the CSR row: this thread's columns ascend
        for (int sw = s0; sw < s1; ++sw) {
            unsigned m = summ[sw];
            if (!m) continue;
            summ[sw] = 0u;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int x = (sw << 5) + b;
                unsigned v = bits[x];
                bits[x] = 0u;
                const unsigned col0 = static_cast<unsigned>(x) << 5;
                while (v) {
                    const int c = static_cast<int>(col0) + (__ffs(v) - 1);
                    if (cur < 0) {  // first column of this thread: binary search, then advance
                        int lo = 0, hi = deg;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (rowp[mid] < c) lo = mid + 1;
                            else hi = mid;
                        }
                        cur = lo;
                    }
                    while (cur < deg && rowp[cur] < c) ++cur;
                    dst[pos++] = (static_cast<unsigned>(c) << 3) | ((cur < deg && rowp[cur] == c) ? 1u : 2u);
                    v &= v - 1;
                }
            }
        }
        if (tid == 0) E.count[r] = s_warp[kWarps - 1];
        __syncthreads();
    }
}

// Row segments of a batch relative to its first row: [seg_b, seg_e) = the
// events the fill pass wrote (offsets may be upper bounds, hop cap 2).
__global__ void khop_segments_kernel(const long long* __restrict__ ev_off, const long long* __restrict__ count,
                                     int rows, int* __restrict__ seg_b, int* __restrict__ seg_e) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < rows) {
        seg_b[k] = static_cast<int>(ev_off[k] - ev_off[0]);
        seg_e[k] = seg_b[k] + static_cast<int>(count[k]);
    }
}

// Hop cap 2: an upper bound of each row's event count without a BFS pass,
// its degree plus the sum of its neighbours' degrees (warp per row).
__global__ void khop_bound_kernel(const long long* __restrict__ off, const int* __restrict__ nbr, int row_begin,
                                  int rows, long long* __restrict__ bound) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int i = row_begin + w;
    long long acc = 0;
    for (long long k = off[i] + lane; k < off[i + 1]; k += 32) {
        const int u = nbr[k];
        acc += off[u + 1] - off[u];
    }
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) bound[w] = acc + (off[i + 1] - off[i]);  // + the row's own hop-1 events
}

__global__ void khop_keys_kernel(const long long* __restrict__ off, const long long* __restrict__ count, int row_begin,
                                 int rows, int* __restrict__ key, int* __restrict__ id) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= rows) return;
    const int i = row_begin + k;
    const long long w = count[k];  // events incl. hop 1
    key[k] = static_cast<int>(min(w, static_cast<long long>(INT_MAX)));
    id[k] = k;
}


// Chunk of up to 32 merged events staged per warp for the batched walk:
// classes 0 = hop 1 (CSR), 1 = hop 2; cnt(q, k) from the class ballots.
struct ChunkEvents {
    const int* cols;
    const unsigned char* kls;
    unsigned m0, m1;
    __device__ int col(int q) const { return cols[q]; }
    __device__ int cls(int q) const { return kls[q]; }
    __device__ int cnt(int q, int k) const {
        const unsigned upto = q < 0 ? 0u : (0xffffffffu >> (31 - q));
        return __popc((k ? m1 : m0) & upto);
    }
};

// Walk of rows whose batch-relative index comes from `order` (heaviest
// first): lane s = sigma s; the row's events (hops 1..K in column order, one
// list) are read 32 at a time with one coalesced load, so the walk is
// warp-uniform. kBatch (hop cap 2): each chunk is walked with
// walk_events_multi (batched in-binade jumps, ff_chain.cuh); otherwise one
// event at a time.
template <bool kBatch>
__global__ void __launch_bounds__(kWalkBlock, kWalkBlocksPerSM)
    khop_walk_kernel(const __grid_constant__ PotentialLaunch P, const __grid_constant__ KhopTable T,
                     const unsigned* __restrict__ ev, const int* __restrict__ seg_b,
                     const int* __restrict__ seg_e, int batch_row0,
                     const int* __restrict__ order, int rows, int* __restrict__ counter) {
    // per-sigma constants staged in shared memory (lane-indexed reads of the
    // kernel parameters would serialise on the constant cache)
    __shared__ double sc[6][kMaxSigmaPerLaunch];
    __shared__ double st[4][kMaxHopCap + 1][kMaxSigmaPerLaunch];
    const int S = P.n_sigma;
    for (int idx = threadIdx.x; idx < kMaxSigmaPerLaunch; idx += blockDim.x) {
        const int q = min(idx, S - 1);
        sc[0][idx] = P.c[q].pW;
        sc[1][idx] = P.c[q].eW;
        sc[2][idx] = P.c[q].pWt;
        sc[3][idx] = P.c[q].eWt;
        sc[4][idx] = P.c[q].inv;
    }
    for (int idx = threadIdx.x; idx < (kMaxHopCap + 1) * kMaxSigmaPerLaunch; idx += blockDim.x) {
        const int h = idx / kMaxSigmaPerLaunch, q = idx % kMaxSigmaPerLaunch;
        st[0][h][q] = T.e[h][q];
        st[1][h][q] = T.p[h][q];
        st[2][h][q] = T.et[h][q];
        st[3][h][q] = T.pt[h][q];
    }
    constexpr int kWarps = kWalkBlock / 32;
    __shared__ int s_cols[kBatch ? kWarps : 1][32];
    __shared__ unsigned char s_kls[kBatch ? kWarps : 1][32];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int s = min(lane, S - 1);
    const double pW = sc[0][s], eW = sc[1][s];
    const int n = P.n;
    const bool tail = P.tail != 0;
    for (;;) {
        int g0 = 0;
        if (lane == 0) g0 = atomicAdd(counter, 1);
        const int g = __shfl_sync(kFull, g0, 0);
        if (g >= rows) break;
        const int rb = order[g];                   // batch-relative row
        const int i = P.row_begin + batch_row0 + rb;
        Chain num = make_chain(0.0, pW), den = make_chain(0.0, eW);
        int pos = 0;
        bool self_pending = true;
        auto w_run = [&](const int L) {
            if (L <= 0) return;
            if (pos == 0) {  // first run: from s = 0 (general loop)
                ff_run(num, pW, L);
                ff_run(den, eW, L);
                num.top = 0.0;
                den.top = 0.0;
            } else {
                ff_walk2(num, pW, den, eW, L);
            }
        };
        auto add_self = [&]() {
            w_run(i - pos);
            den.s = __dadd_rn(den.s, 1.0);  // d2 = 0: num += 0, den += exp(0) = 1
            pos = i + 1;
            self_pending = false;
        };
        auto event = [&](const int col, const int h) {
            if (self_pending && i < col) add_self();
            w_run(col - pos);
            const bool at_tail = tail && col == n - 1;
            const double e = st[at_tail ? 2 : 0][h][s];
            const double p = st[at_tail ? 3 : 1][h][s];
            num.s = __dadd_rn(num.s, p);
            den.s = __dadd_rn(den.s, e);
            pos = col + 1;
        };
        // the row's events (hops 1..K), ascending columns
        long long kb = seg_b[rb];
        const long long kb_end = seg_e[rb];
        if constexpr (kBatch) {
            const int wslot = threadIdx.x >> 5;
            int* cols = s_cols[wslot];
            unsigned char* kls = s_kls[wslot];
            const double cn[2] = {st[1][1][s], st[1][2][s]}, cd[2] = {st[0][1][s], st[0][2][s]};
            const int tn[2] = {tie_binade(cn[0]), tie_binade(cn[1])}, td[2] = {tie_binade(cd[0]), tie_binade(cd[1])};
            const int tie_pW = tie_binade(pW), tie_eW = tie_binade(eW);
            for (; kb < kb_end; kb += 32) {  // warp-uniform: 32 events per chunk
                const int cnt = static_cast<int>(min(32ll, kb_end - kb));
                const unsigned evl = lane < cnt ? __ldg(ev + kb + lane) : 0xffffffffu;
                const int my = lane < cnt ? static_cast<int>(evl >> 3) : INT_MAX;
                __syncwarp();
                cols[lane] = my;
                kls[lane] = static_cast<unsigned char>((evl & 7u) - 1u);
                __syncwarp();
                ChunkEvents ce{cols, kls, __ballot_sync(kFull, lane < cnt && (evl & 7u) == 1u),
                               __ballot_sync(kFull, lane < cnt && (evl & 7u) == 2u)};
                const int jend = (tail && cols[cnt - 1] == n - 1) ? cnt - 1 : cnt;
                const int before_self = __popc(__ballot_sync(kFull, my < i));
                int j = 0;
                while (j < jend) {  // warp-uniform
                    int r = jend;
                    if (self_pending) r = min(max(before_self, j), jend);
                    if (r > j) {
                        num.s = walk_events_multi<2>(num.s, pW, tie_pW, cn, tn, ce, j, r, pos);
                        den.s = walk_events_multi<2>(den.s, eW, tie_eW, cd, td, ce, j, r, pos);
                        num.top = 0.0;  // binade caches are stale now
                        den.top = 0.0;
                        pos = cols[r - 1] + 1;
                        j = r;
                    }
                    if (self_pending && j < jend) add_self();
                }
                if (jend < cnt) event(cols[cnt - 1], kls[cnt - 1] + 1);  // the Eigen tail column
                __syncwarp();
            }
        } else {
            for (; kb < kb_end; kb += 32) {  // one event at a time, 32 loaded per chunk
                const int cnt = static_cast<int>(min(32ll, kb_end - kb));
                const unsigned evl = lane < cnt ? __ldg(ev + kb + lane) : 0u;
                for (int q = 0; q < cnt; ++q) {
                    const unsigned e = __shfl_sync(kFull, evl, q);
                    event(static_cast<int>(e >> 3), static_cast<int>(e & 7u));
                }
            }
        }
        if (self_pending) add_self();
        const int L = n - pos;  // final run; the Eigen tail column n-1 uses glibc constants
        if (L > 0) {
            if (tail) {
                w_run(L - 1);
                num.s = __dadd_rn(num.s, sc[2][s]);
                den.s = __dadd_rn(den.s, sc[3][s]);
            } else {
                w_run(L);
            }
        }
        if (lane < S) *out_slot_ptr(P, i, s) = __dmul_rn(sc[4][s], __ddiv_rn(num.s, den.s));
    }
    if (P.out_peer) __threadfence_system();
}

int num_sms() { return sm_count(); }

}  // namespace

int launch_potentials_khop(const PotentialLaunch& p, int hop_cap, const KhopTable& T, void* pool_, void* stream) {
    const int rows = p.row_end - p.row_begin;
    if (rows <= 0) return cudaSuccess;
    auto st = static_cast<cudaStream_t>(stream);
    auto pool = static_cast<cudaMemPool_t>(pool_);
    cudaError_t e;
    const int n = p.n;
    const int words = (n + 31) / 32;
    const std::size_t bitset_bytes = static_cast<std::size_t>(words) * 4;
    const bool smem = bitset_bytes <= kSmemBitsetBytes;
    const int dyn = smem ? static_cast<int>(bitset_bytes) : 0;
    int per_sm = 1;
    cudaFuncSetAttribute(khop_expand_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaFuncSetAttribute(khop_expand_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, khop_expand_kernel<false>, kExpandThreads, dyn);
    const int grid = std::max(1, std::min(num_sms() * std::max(per_sm, 1), rows));

    // scratch: counter, counts/offsets, per-block level lists, global bitsets
    auto bytes_of = [](std::size_t b) { return (b + 255) & ~static_cast<std::size_t>(255); };
    const std::size_t b_cnt = bytes_of(16), b_count = bytes_of((rows + 1) * sizeof(long long));
    const std::size_t b_off = b_count;
    const std::size_t b_scr = hop_cap == 2 ? 0 : bytes_of(static_cast<std::size_t>(grid) * n * sizeof(unsigned));
    const std::size_t b_bits = smem ? 0 : bytes_of(static_cast<std::size_t>(grid) * bitset_bytes);
    std::size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<long long*>(nullptr),
                                  static_cast<long long*>(nullptr), rows + 1);
    void* mem = nullptr;
    if ((e = cudaMallocFromPoolAsync(&mem, b_cnt + b_count + b_off + b_scr + b_bits + bytes_of(scan_bytes), pool,
                                     st)) != cudaSuccess)
        return e;
    char* m = static_cast<char*>(mem);
    int* counter = reinterpret_cast<int*>(m);
    long long* count = reinterpret_cast<long long*>(m + b_cnt);
    long long* ev_off = reinterpret_cast<long long*>(m + b_cnt + b_count);
    unsigned* scratch = reinterpret_cast<unsigned*>(m + b_cnt + b_count + b_off);
    unsigned* gbits = smem ? nullptr : reinterpret_cast<unsigned*>(m + b_cnt + b_count + b_off + b_scr);
    void* scan_tmp = m + b_cnt + b_count + b_off + b_scr + b_bits;

    KhopExpand E{};
    E.n = n;
    E.off = reinterpret_cast<const long long*>(p.offsets);
    E.nbr = p.nbr;
    E.K = hop_cap;
    E.count = count;
    E.scratch = scratch;
    E.gbits = gbits;
    E.words = words;
    E.counter = counter;
    E.row_begin = p.row_begin;
    E.rows = rows;
    cudaMemsetAsync(counter, 0, 16, st);
    cudaMemsetAsync(count + rows, 0, sizeof(long long), st);
    if (hop_cap == 2) {
        // no counting BFS: segments sized by the neighbour-degree bound
        khop_bound_kernel<<<(rows + 7) / 8, 256, 0, st>>>(E.off, E.nbr, p.row_begin, rows, count);
    } else {
        khop_expand_kernel<false><<<grid, kExpandThreads, dyn, st>>>(E);
    }
    count_launch();
    if ((e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, count, ev_off, rows + 1, st)) != cudaSuccess)
        return e;
    count_launch();

    // batches of rows whose events fit the budget
    std::vector<long long> h_off(rows + 1);
    if ((e = cudaMemcpyAsync(h_off.data(), ev_off, (rows + 1) * sizeof(long long), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    std::vector<int> cuts{0};
    while (cuts.back() < rows) {
        const int r0 = cuts.back();
        int r1 = static_cast<int>(std::upper_bound(h_off.begin() + r0 + 1, h_off.end(), h_off[r0] + kEventBudget) -
                                  h_off.begin()) - 1;
        cuts.push_back(std::max(r1, r0 + 1));  // a single row always fits (< N events)
    }

    // hop cap 2 with an on-chip bitset: sorted emission, no sort pass
    const std::size_t emit_bytes = bitset_bytes + static_cast<std::size_t>((words + 31) / 32) * 4;
    const bool emit = hop_cap == 2 && emit_bytes <= kSmemBitsetBytes;
    const bool big_emit = emit_bytes > 96 * 1024;  // one 1024-thread block per SM, else 256-thread blocks
    const int edyn = static_cast<int>(emit_bytes);
    int emit_grid = 1;
    if (emit) {
        int per = 1;
        if (big_emit) {
            cudaFuncSetAttribute(khop2_emit_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, edyn);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, khop2_emit_kernel<1024>, 1024, edyn);
        } else {
            cudaFuncSetAttribute(khop2_emit_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, edyn);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, khop2_emit_kernel<256>, 256, edyn);
        }
        emit_grid = num_sms() * std::max(per, 1);
    }
    int sort_end_bit = 1;  // keys (col << 1 | tag) < 2n: the padding 0xffffffff must sort after every key
    while (sort_end_bit < 32 && (1ll << sort_end_bit) <= 2ll * n) ++sort_end_bit;
    int walk_grid_cap = num_sms() * kWalkBlocksPerSM;
    for (std::size_t b = 0; b + 1 < cuts.size(); ++b) {
        const int r0 = cuts[b], r1 = cuts[b + 1], nr = r1 - r0;
        const long long items = h_off[r1] - h_off[r0];
        std::size_t sort_bytes = 0, key_bytes = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, sort_bytes, static_cast<const unsigned*>(nullptr),
                                           static_cast<unsigned*>(nullptr), static_cast<int>(items), nr,
                                           static_cast<const int*>(nullptr), static_cast<const int*>(nullptr), st);
        cub::DeviceRadixSort::SortPairsDescending(nullptr, key_bytes, static_cast<const int*>(nullptr),
                                                  static_cast<int*>(nullptr), static_cast<const int*>(nullptr),
                                                  static_cast<int*>(nullptr), nr);
        const std::size_t b_ev = bytes_of(std::max<long long>(items, 1) * sizeof(unsigned));
        const std::size_t b_raw = emit ? 0 : b_ev;  // ordered emission writes the final list directly
        const std::size_t b_seg = 2 * bytes_of((nr + 1) * sizeof(int));
        const std::size_t b_key = bytes_of(nr * sizeof(int));
        void* bm = nullptr;
        if ((e = cudaMallocFromPoolAsync(&bm, b_raw + b_ev + b_seg + 7 * b_key + (emit ? 0 : bytes_of(sort_bytes)) +
                                                  bytes_of(key_bytes) + 512,
                                         pool, st)) != cudaSuccess)
            return e;
        char* q = static_cast<char*>(bm);
        unsigned* ev_raw = reinterpret_cast<unsigned*>(q);  // (unused with ordered emission)
        unsigned* ev_sorted = reinterpret_cast<unsigned*>(q + b_raw);
        int* seg_b = reinterpret_cast<int*>(q + b_raw + b_ev);
        int* seg_e = seg_b + b_seg / (2 * sizeof(int));
        int* key_in = reinterpret_cast<int*>(q + b_raw + b_ev + b_seg);
        int* key_out = key_in + b_key / sizeof(int);
        int* id_in = key_out + b_key / sizeof(int);
        int* id_out = id_in + b_key / sizeof(int);
        int* wcounter = reinterpret_cast<int*>(q + b_raw + b_ev + b_seg + 4 * b_key);
        void* sort_tmp = q + b_raw + b_ev + b_seg + 4 * b_key + 256;
        void* key_tmp = static_cast<char*>(sort_tmp) + (emit ? 0 : bytes_of(sort_bytes));
        int* rows0 = reinterpret_cast<int*>(static_cast<char*>(key_tmp) + bytes_of(key_bytes));
        int* rows1 = rows0 + b_key / sizeof(int);
        int* rows2 = rows1 + b_key / sizeof(int);
        int* lens = rows2 + b_key / sizeof(int);  // list lengths

        // fill pass over the batch's rows
        KhopExpand F = E;
        F.row_begin = p.row_begin + r0;
        F.rows = nr;
        F.ev_off = ev_off + r0;
        F.ev_base = h_off[r0];
        F.ev = ev_raw;
        F.count = count + r0;
        cudaMemsetAsync(counter, 0, 16, st);
        const unsigned* ev_walk = ev_sorted;
        if (emit) {
            F.ev = ev_sorted;  // written in column order
            // rows whose candidates fit on chip go to the sort kernel (many rows
            // in flight per SM); the rest to the bitset kernel. With a large
            // bitset (one block per SM) the 2048-candidate sort size is used
            // too; with a small one only the 512 size (padding would dominate).
            cudaMemsetAsync(lens, 0, 4 * sizeof(int), st);
            khop_split_kernel<<<(nr + 255) / 256, 256, 0, st>>>(ev_off + r0, nr, kSortCap0,
                                                                 big_emit ? kSortCap1 : kSortCap0, rows0, rows1,
                                                                 rows2, lens);
            KhopExpand F0 = F, F1 = F, F2 = F;
            F0.list = rows0;
            F0.list_len = lens;
            F1.list = rows1;
            F1.list_len = lens + 1;
            F1.counter = counter + 1;
            F2.list = rows2;
            F2.list_len = lens + 2;
            F2.counter = counter + 2;
            khop2_sort_kernel<128, 4><<<num_sms() * 8, 128, 0, st>>>(F0, sort_end_bit);
            if (big_emit) {
                khop2_sort_kernel<256, 8><<<num_sms() * 4, 256, 0, st>>>(F1, sort_end_bit);
                khop2_emit_kernel<1024><<<std::max(1, std::min(emit_grid, nr)), 1024, edyn, st>>>(F2);
            } else {
                khop2_emit_kernel<256><<<std::max(1, std::min(emit_grid, nr)), 256, edyn, st>>>(F2);
            }
            count_launch(big_emit ? 4 : 3);
        } else {
            khop_expand_kernel<true><<<std::max(1, std::min(grid, nr)), kExpandThreads, dyn, st>>>(F);
            count_launch();
        }
        khop_segments_kernel<<<(nr + 255) / 256, 256, 0, st>>>(ev_off + r0, count + r0, nr, seg_b, seg_e);
        count_launch();
        if (items > 0 && !emit) {
            if ((e = cub::DeviceSegmentedSort::SortKeys(sort_tmp, sort_bytes, ev_raw, ev_sorted,
                                                        static_cast<int>(items), nr, seg_b, seg_e, st)) !=
                cudaSuccess)
                return e;
            count_launch();
        }
        // longest rows first
        khop_keys_kernel<<<(nr + 255) / 256, 256, 0, st>>>(E.off, count + r0, p.row_begin + r0, nr, key_in, id_in);
        count_launch();
        if ((e = cub::DeviceRadixSort::SortPairsDescending(key_tmp, key_bytes, key_in, key_out, id_in, id_out, nr, 0,
                                                           32, st)) != cudaSuccess)
            return e;
        count_launch(2);
        cudaMemsetAsync(wcounter, 0, sizeof(int), st);
        const int wgrid = static_cast<int>(
            std::min<long long>((nr + kWalkBlock / 32 - 1) / (kWalkBlock / 32), walk_grid_cap));
        if (hop_cap == 2)
            khop_walk_kernel<true><<<wgrid, kWalkBlock, 0, st>>>(p, T, ev_walk, seg_b, seg_e, r0, id_out, nr, wcounter);
        else
            khop_walk_kernel<false><<<wgrid, kWalkBlock, 0, st>>>(p, T, ev_walk, seg_b, seg_e, r0, id_out, nr, wcounter);
        count_launch();
        cudaFreeAsync(bm, st);
    }
    cudaFreeAsync(mem, st);
    return cudaGetLastError();
}

}  // namespace gqc
