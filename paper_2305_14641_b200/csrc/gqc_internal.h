// Internal shared definitions of libgqc (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gqc {

// Per-sigma constants handed to the potential kernels. "t" variants are the
// glibc values for the reference's scalar tail column (j = N-1 when N is odd
// in the Eigen build, potential.cpp:26).
struct SigmaConsts {
    double inv, neg_inv;
    double eW, pW;    // non-adjacent pair: exp(-inv*W^2), W^2*exp(...)
    double e1, p1;    // unit-weight neighbour
    double eWt, pWt;  // tail column, non-adjacent
    double e1t, p1t;  // tail column, unit-weight neighbour
};
constexpr int kSigmaFields = 10;
constexpr int kMaxSigmaPerLaunch = 32;
constexpr int kMaxShards = 32;  // shards of a multi-device sweep (one sigma chunk each)

double host_pexp(double x);
double host_glibc_exp(double x);
double inv_two_sigma_sq(double sigma);
SigmaConsts make_sigma_consts(double sigma, double W, int exp_mode);

// Weight handling of a potential launch.
enum WeightMode : int {
    kUnit = 0,        // all neighbour weights 1.0: constants only
    kDevicePexp = 1,  // per-entry device pexp (Eigen mode), tail entries from tail_exp
    kEntryTable = 2,  // per-entry exp values precomputed on the host (glibc mode)
};

struct PotentialLaunch {
    std::int32_t n;
    std::int32_t n_sigma;      // sigmas in this launch (<= kMaxSigmaPerLaunch)
    std::int32_t row_begin, row_end;
    std::int64_t nnz;          // entries of the whole CSR (hub threshold)
    const std::int64_t* offsets;
    const std::int32_t* nbr;
    const double* w;           // nullptr for unit weights
    int tail;                  // column n-1 uses the glibc tail constants
    int weight_mode;
    const double* entry_exp;   // kEntryTable: [nnz][entry_ld] at column entry_col0 + s
    std::int32_t entry_ld, entry_col0;
    const double* tail_exp;    // kDevicePexp && tail: [deg(n-1)][n_sigma] glibc exp of row n-1's entries
    // out[(k / out_chunk) * out_chunk_stride + (i - row_begin) * out_ld + k % out_chunk],
    // k = out_col0 + s the sigma's index in the caller's grid (out_chunk >= that
    // grid's size: plain node-major rows)
    double* out;
    std::int32_t out_ld, out_col0;
    std::int32_t out_chunk;
    long long out_chunk_stride;
    // Multi-device sweep: when out_peer is set, chunk q goes to
    // out_chunk_ptr[q] + (i - row_begin) * out_ld + k % out_chunk instead of
    // out + q * out_chunk_stride + ... — the buffer of the device that owns
    // sigma chunk q, written in place over peer memory (NVLink), so the
    // potential kernel itself performs the V exchange.
    int out_peer;
    double* out_chunk_ptr[kMaxShards];
    // Polled CSR upload (host pipeline, unit weights, warp kernel): rows
    // [slab_bound[k], slab_bound[k+1]) may be read once slab_flags[k] != 0
    // (set by a copy after the slab's data on the copy stream); rows are
    // scheduled slab-major. slab_err: set if a flag never arrives (timeout).
    int iso;  // the graph has isolated rows (degree sample): the fast-forward's isolated-row instantiation
    const int* slab_flags;
    std::int32_t slab_bound[5];
    int* slab_err;
    long long slab_timeout_ns;  // GQC_SLAB_TIMEOUT_MS (default 5000)
    SigmaConsts c[kMaxSigmaPerLaunch];
};

#ifdef __CUDACC__
// Address of (row i, launch sigma s) in the launch's output (see PotentialLaunch::out).
__device__ __forceinline__ double* out_slot_ptr(const PotentialLaunch& P, const int i, const int s) {
    const int k = P.out_col0 + s;
    const int q = k / P.out_chunk;
    double* base = P.out_peer ? P.out_chunk_ptr[q] : P.out + q * P.out_chunk_stride;
    return base + static_cast<long long>(i - P.row_begin) * P.out_ld + (k - q * P.out_chunk);
}
#endif

// Kernel launchers (kernels.cu). Return a cudaError_t as int.
// Stream-ordered scratch comes from `pool` (a cudaMemPool_t that keeps its
// memory, so per-call scratch costs no driver allocation).
int launch_potentials(const PotentialLaunch& p, int kernel, void* pool, void* stream);
// Degree-class order of a potential field (unit-weight fast path of the GGD
// argmin, see kernels.cu): cls[i] = rank of node i's degree among the
// distinct degrees, dir[s] = +1 / -1 when, for sigma s, every node of a lower
// class has a strictly smaller / larger potential than every node of a higher
// class (verified on the field itself, not assumed), 0 otherwise.
struct ClassOrder {
    const std::int32_t* cls = nullptr;
    const signed char* dir = nullptr;  // indexed by the sigma column of V
};
// Builds the order for V (node-major, leading dimension ld, n_sigma columns)
// into pool scratch *mem (release with cudaFreeAsync(*mem, stream) after the
// successor launches that use it).
int launch_class_order(std::int32_t n, const std::int64_t* offsets, long long nnz, const double* v, std::int32_t ld,
                       std::int32_t n_sigma, void* pool, void* stream, ClassOrder* out, void** mem);
// GGD argmin for rows [row_begin, row_end) and the sigma columns
// [s0, s0 + n_sigma) of a node-major V with leading dimension ld. Element
// (row r of the range, sigma q) goes to out[r * out_row + q * out_col]
// (sigma-major: out_row = 1, out_col = n; node-major shard: out_row = ld, out_col = 1).
// co (optional): the field's class order; sigmas with dir != 0 take the
// fast path (only best-class neighbours' potentials are gathered).
// sub: sigmas per light-row launch (32, or 16 for graphs made mostly of rows
// with a handful of neighbours: two rows per warp), see light_row_sigmas_*.
int launch_successors(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* v,
                      std::int32_t ld, std::int32_t s0, std::int32_t n_sigma, std::int32_t row_begin,
                      std::int32_t row_end, std::int32_t* out, long long out_row, long long out_col, long long nnz,
                      void* pool, void* stream, const ClassOrder* co = nullptr, int sub = 32);
// The GGD argmin's light-row launch width for a CSR from a sample of 8192
// pseudo-random rows' degrees: 16 when more than 20% have <= 4 neighbours,
// else 32. Host offsets, or device offsets (cached per device and CSR
// pointer / shape: one stream synchronisation the first time; only the
// speed depends on it).
int light_row_sigmas_host(const std::int64_t* offsets, std::int32_t n);
int light_row_sigmas_device(const std::int64_t* offsets, std::int32_t n, long long nnz, void* stream);
// 1 when more than 1% of the same sample of a device CSR's rows are isolated
// (no neighbours): the unit-weight fast-forward then runs the instantiation
// with the isolated-row shortcut.
int isolated_rows_device(const std::int64_t* offsets, std::int32_t n, long long nnz, void* stream);
// out[s] = CSR entries (i, j) whose cluster_index matches for sigma s (device,
// sigma-major labels [n_sigma][n]); the unit-weight modularity intra term.
int launch_intra_counts(std::int32_t n, std::int32_t n_sigma, const std::int64_t* offsets, const std::int32_t* nbr,
                        const std::int32_t* ci_sm, long long* out, void* stream);
int launch_transpose_i32(const std::int32_t* in, std::int32_t n, std::int32_t n_sigma, std::int32_t* out, void* stream);
// GGD chase + labels (K4/K5, ggd.cpp:26-57) for n_sigma sigma-major slices:
// center = the root of every node's successor chain (succ_sm == center_sm:
// in place), cluster_index = the root's rank among the ascending roots,
// num_clusters (device) per sigma. workspace: labels_workspace_bytes(n,
// n_sigma) bytes (required). err (optional, device): set to 1 if a map has a
// cycle (bounded chase + pointer jumping, see chase_kernel).
int launch_labels(std::int32_t n, std::int32_t n_sigma, const std::int32_t* succ_sm, std::int32_t* center_sm,
                  std::int32_t* cluster_index_sm, std::int32_t* num_clusters, void* workspace, std::size_t ws_bytes,
                  void* stream, std::int32_t* err = nullptr);
std::size_t labels_workspace_bytes(std::int32_t n, std::int32_t n_sigma);
int launch_transpose(const double* v_nm, std::int32_t n, std::int32_t n_sigma, double* v_sm, void* stream);
// Checked resolve for arbitrary successor maps: writes center/cluster_index,
// returns status via *err_kind (0 ok, 1 out of range, 2 cycle) on the host.
int resolve_checked(std::int32_t n, const std::int32_t* succ_dev, std::int32_t* center_dev,
                    std::int32_t* cluster_index_dev, std::int32_t* num_clusters_host, int* err_kind, void* pool,
                    void* stream);

// k-hop extension (khop.cu): per-sigma constants of a hop-h term,
// d2 = h*h: e = exp(-inv*d2) by the exp provider, p = d2*e; "t" = the glibc
// values of the Eigen tail column. Index 0 unused; h = 1 equals (e1, p1).
constexpr int kMaxHopCap = 7;
struct KhopTable {
    double e[kMaxHopCap + 1][kMaxSigmaPerLaunch];
    double p[kMaxHopCap + 1][kMaxSigmaPerLaunch];
    double et[kMaxHopCap + 1][kMaxSigmaPerLaunch];
    double pt[kMaxHopCap + 1][kMaxSigmaPerLaunch];
};
void fill_khop_table(KhopTable& t, int s, double sigma, int hop_cap, int exp_mode);
int launch_potentials_khop(const PotentialLaunch& p, int hop_cap, const KhopTable& t, void* pool, void* stream);

// Edge-list ingestion on the device (csr_build.cu): graphqc::Graph's CSR
// (graph.cpp:25-71) from m input edges. offsets[n+1], nbr / w_out (capacity
// >= 2m, w_out optional) are host outputs; conflicts (optional) receives
// (dropped, kept) input-index pairs of duplicates with a different weight
// (unsorted; a trailing -1 marks an overflow); *first_error = -1 or
// k << 1 | kind of the first offending edge (0 endpoint, 1 weight).
struct GqcEdge {
    std::int32_t u, v;
    double w;
};
int build_csr_device(int n, long long m, const GqcEdge* host_edges, std::int64_t* offsets, std::int32_t* nbr,
                     double* w_out, long long* nnz_out, std::vector<long long>* conflicts, int* unit_out,
                     long long* first_error, void* pool, void* stream);

// SM count of the calling thread's current device (cached per device).
int sm_count();

// Launch accounting (kernels issued by the last C-ABI call).
void count_launch(int k = 1);

}  // namespace gqc
