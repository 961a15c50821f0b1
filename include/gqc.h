/*
 * gqc.h — C-ABI of the B200-native QC potential sweep + Graph Gradient Descent.
 *
 * This is the drop-in boundary for the reference's hot path. Each entry point
 * replaces one graphqc C++ function (paths relative to the reference's proj/):
 *
 *   gqc_potentials          <- graphqc::compute_potentials / compute_potentials_parallel
 *                              (include/graphqc/potential.hpp:33-37, src/potential.cpp:53-87),
 *                              batched over sigma.
 *   gqc_node_potential      <- graphqc::node_potential (potential.hpp:30, potential.cpp:46-51)
 *   gqc_build_successors    <- graphqc::build_successors (ggd.hpp:28, ggd.cpp:7-24)
 *   gqc_resolve_centers     <- graphqc::resolve_centers (ggd.hpp:33, ggd.cpp:26-57)
 *   gqc_cluster_sweep       <- graphqc::cluster (ggd.hpp:37, ggd.cpp:59-62) for every sigma of a
 *                              grid, i.e. the per-sigma loop of graphqc::run_sweep (sweep.cpp:50-57)
 *   gqc_cluster_sweep_multi,
 *   gqc_potentials_multi    <- compute_potentials_parallel(g, sigma, workers) (potential.cpp:62-87)
 *                              with GPUs as the workers, for cluster / run_sweep; the n_gpus
 *                              parameter of the survey's gqc_potentials / gqc_cluster_sweep is
 *                              GQC_OPT_GPUS (same entry points) or the explicit device list here
 *   gqc_build_csr           <- graphqc::Graph(n, edges, W)'s CSR (graph.cpp:25-71), on the device
 *   gqc_dev_*               <- the same operations on device-resident buffers (row-sharded
 *                              potentials for multi-GPU, incl. gqc_dev_potentials_peer whose
 *                              kernel stores each sigma chunk into its owner's buffer)
 *
 * Conventions: plain pointers and sizes, no C++ or torch types. Host-buffer
 * entry points (gqc_potentials, gqc_build_successors, gqc_resolve_centers,
 * gqc_cluster_sweep, gqc_node_potential) copy inputs to the current CUDA
 * device and results back; the caller owns every buffer. Errors are status
 * codes mirroring the reference's exception classes; gqc_last_error() returns
 * the message of the calling thread's last failure (same texts as the
 * reference, e.g. "sigma must be positive"). Each call locks the context of
 * every device it uses for its whole duration (one lock per device, taken in
 * ascending device order): calls on different devices, from different host
 * threads, run concurrently; calls on one device are serialized.
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point fails with GQC_ECUDA.
 */
#ifndef GQC_H
#define GQC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gqc_status {
    GQC_OK = 0,
    GQC_EINVAL = 1, /* std::invalid_argument (bad sigma, size mismatch, successor out of range) */
    GQC_ERANGE = 2, /* std::out_of_range (bad node id) */
    GQC_ECYCLE = 3, /* std::logic_error ("successor map contains a cycle") */
    GQC_EIO = 4,    /* graphqc::IoError */
    GQC_ECUDA = 5,  /* CUDA runtime failure or no device */
    GQC_ENOMEM = 6, /* device or host allocation failure (std::bad_alloc) */
    GQC_ENCCL = 7   /* collective / peer-memory exchange failures */
} gqc_status;

/* Undirected CSR exactly as graphqc::Graph stores it (graph.hpp:66-71):
 * offsets[n+1] (int64), nbr[nnz] ascending within each row (int32),
 * w[nnz] positive distances or NULL for unit weights, W = default distance
 * of non-adjacent pairs. Borrowed for the duration of a call. */
typedef struct gqc_csr {
    int32_t n;
    int64_t nnz;
    const int64_t* offsets;
    const int32_t* nbr;
    const double* w;
    double W;
} gqc_csr;

/* Exp provider: which exp the reference build used for exp(-d^2/2sigma^2)
 * at potential.cpp:26. EIGEN = Eigen 3.4 pexp on SSE2 packets of two plus
 * glibc std::exp for the N mod 2 tail element (the default Release build);
 * GLIBC = std::exp for every element. */
typedef enum gqc_exp_mode { GQC_EXP_EIGEN = 0, GQC_EXP_GLIBC = 1 } gqc_exp_mode;

/* Potential kernel: FASTFWD = exact run fast-forward (default, O(deg + log N)
 * per row); REPLAY = dense in-order replay (O(N) per row, the parity anchor).
 * Both are bit-identical to the reference's ascending-j fp64 sums. */
typedef enum gqc_kernel { GQC_KERNEL_FASTFWD = 0, GQC_KERNEL_REPLAY = 1 } gqc_kernel;

/* GQC_OPT_DEVICE: CUDA device ordinal of the host-buffer entry points
 * (default 0). The gqc_dev_* entry points run on the device of the stream
 * they are given (or, for the legacy default stream, of their buffers):
 * libgqc links its own CUDA runtime, so the caller's current device does not
 * carry over. */
/* GQC_OPT_HOP_CAP (K, default 1): distance model of every potential entry
 * point. 1 = the reference's pairwise_distance (graph.cpp:258-267: 0 / edge
 * weight / W). K in 2..7 = opt-in k-hop extension, NOT in the reference
 * (SURVEY §8(f)): on unit-weight graphs d(i,j) = BFS hop count for hops
 * 1..K and W beyond; the sums keep the reference's order and exp rule.
 * Weighted graphs with K > 1 -> GQC_EINVAL ("k-hop distances need unit
 * weights"). The fast-forward kernel runs either way (GQC_OPT_KERNEL only
 * selects the K = 1 kernel). */
/* GQC_OPT_GPUS (g, default 1): gqc_potentials, gqc_cluster_sweep and
 * gqc_cluster_sweep_intra run on the g devices GQC_OPT_DEVICE ..
 * GQC_OPT_DEVICE + g - 1 (see gqc_cluster_sweep_multi); the results are the
 * same bits for every g. */
typedef enum gqc_option {
    GQC_OPT_EXP_MODE = 1,
    GQC_OPT_KERNEL = 2,
    GQC_OPT_DEVICE = 3,
    GQC_OPT_HOP_CAP = 4,
    GQC_OPT_GPUS = 5
} gqc_option;

const char* gqc_last_error(void);
const char* gqc_version(void);
gqc_status gqc_set_option(gqc_option key, int64_t value);
gqc_status gqc_get_option(gqc_option key, int64_t* value);
/* Number of CUDA devices visible (0 on a machine without a GPU). */
int32_t gqc_device_count(void);
/* Optional: create the current device's context, streams and memory pool and
 * load the sweep kernels now (every entry point otherwise does this on first
 * use). Safe to call from a helper thread while the caller parses its input
 * (it holds the device's lock; other calls on that device wait for it). No
 * reference counterpart
 * (the reference has no device); the CLI uses it to overlap CUDA start-up
 * (~0.5-1.5 s per process) with edge-list parsing. */
gqc_status gqc_init(void);
/* 1 once this process has created the context of GQC_OPT_DEVICE (gqc_init or
 * any call on it), else 0. Never blocks or initializes anything: a host
 * program can pick a device path only when it costs no start-up (the facade's
 * edge-list loader builds the CSR on the device when it is ready). */
int32_t gqc_device_ready(void);

/* ---------------------------------------------------------------- host API */

/* v_out[k*n + i] = potential of node i at sigmas[k] (sigma-major, one
 * PotentialField::values per sigma). sigma <= 0 -> GQC_EINVAL. */
gqc_status gqc_potentials(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out);

/* One node (node_potential). Bad node -> GQC_ERANGE, bad sigma -> GQC_EINVAL. */
gqc_status gqc_node_potential(const gqc_csr* g, int32_t node, double sigma, double* out);

/* succ[i] = lexicographic (v, id) argmin over {i} + neighbors(i). v has n entries. */
gqc_status gqc_build_successors(const gqc_csr* g, const double* v, int32_t* succ);

/* Chase succ to fixed points. Out-of-range successor -> GQC_EINVAL
 * ("successor id out of range"), cycle -> GQC_ECYCLE ("successor map contains
 * a cycle"), reporting whichever the reference's ascending chase meets first.
 * cluster_index numbers centers densely by ascending center id. */
gqc_status gqc_resolve_centers(int32_t n, const int32_t* succ, int32_t* center, int32_t* cluster_index,
                               int32_t* num_clusters);

/* Full pipeline per sigma (potentials -> successors -> centers). Outputs are
 * sigma-major [n_sigma][n]; v_out, succ_out and center_out may be NULL (a
 * sweep needs only cluster_index and the counts). num_clusters_out has
 * n_sigma entries. The CSR upload is pipelined under the potential launches
 * and the label downloads under the GGD of the next sigma chunk. */
gqc_status gqc_cluster_sweep(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out,
                             int32_t* succ_out, int32_t* center_out, int32_t* cluster_index_out,
                             int32_t* num_clusters_out);

/* gqc_cluster_sweep plus, per sigma, intra_out[k] = the number of CSR
 * entries (i, j) with cluster_index[k][i] == cluster_index[k][j]: the
 * intra-cluster weight of modularity (metrics.cpp:37-44) for a unit-weight
 * graph, exact, so the host evaluates modularity in O(N + K) instead of
 * O(nnz). Weighted graphs -> GQC_EINVAL ("intra counts need unit weights").
 * intra_out may be NULL (then identical to gqc_cluster_sweep). */
gqc_status gqc_cluster_sweep_intra(const gqc_csr* g, const double* sigmas, int32_t n_sigma, double* v_out,
                                   int32_t* succ_out, int32_t* center_out, int32_t* cluster_index_out,
                                   int32_t* num_clusters_out, int64_t* intra_out);

/* ------------------------------------------------------------- ingestion */
/* One input edge, laid out like graphqc::Edge (graph.hpp:20-24). */
typedef struct gqc_edge {
    int32_t u, v;
    double w;
} gqc_edge;

/* The CSR of graphqc::Graph(n, edges, W) (graph.cpp:25-71), built on the
 * device by two radix sorts: validation in input order (the first edge with
 * an endpoint outside [0, n) -> GQC_ERANGE "edge endpoint out of range", or
 * with weight <= 0 -> GQC_EINVAL "edge weight must be positive"), self loops
 * dropped, duplicate undirected pairs keep their first occurrence, rows
 * ascending. Host outputs: offsets[n+1]; nbr and w_out (optional) with room
 * for 2*m entries; *nnz_out; *unit_out = 1 when every kept weight is 1.0.
 * Dropped duplicates whose weight differs from the kept one (the reference
 * warns about each, in input order): dup_out[2j] = dropped input index,
 * dup_out[2j+1] = kept input index, ascending by dropped index, at most
 * dup_cap pairs; *n_dup_out = how many exist. m < 2^32. */
gqc_status gqc_build_csr(int32_t n, int64_t m, const gqc_edge* edges, int64_t* offsets, int32_t* nbr, double* w_out,
                         int64_t* nnz_out, int32_t* unit_out, int64_t* dup_out, int64_t dup_cap, int64_t* n_dup_out);

/* -------------------------------------------------------- multi-device API */
/* The row-sharded sweep of one process over several GPUs — the reference's
 * compute_potentials_parallel(g, sigma, workers) (potential.cpp:62-87) with
 * GPUs as the workers, and its callers cluster (ggd.cpp:59-62) and run_sweep
 * (sweep.cpp:50-57) for a whole sigma grid.
 *
 * devices[r] is the CUDA device of shard r (0 <= r < n_shards <= 32; a device
 * may be listed more than once and then hosts several shards). Shard r
 * computes the potentials of the row block gqc_row_shards() assigns it for
 * every sigma and owns sigma chunk r (ceil(n_sigma / n_shards) sigmas): its
 * potential kernel stores each chunk of its rows directly into the owning
 * shard's field over peer memory (NVLink/NVSwitch; staged + peer copy when
 * two devices cannot access each other), then every shard runs GGD for its
 * own chunk and writes its labels to the caller's sigma-major outputs. The
 * whole CSR is uploaded to every device. Outputs and errors are exactly those
 * of gqc_cluster_sweep_intra / gqc_potentials, bit for bit, for any shard
 * count. n_shards == 1 runs the single-device pipeline on devices[0]. */
gqc_status gqc_cluster_sweep_multi(const gqc_csr* g, const double* sigmas, int32_t n_sigma, const int32_t* devices,
                                   int32_t n_shards, double* v_out, int32_t* succ_out, int32_t* center_out,
                                   int32_t* cluster_index_out, int32_t* num_clusters_out, int64_t* intra_out);
gqc_status gqc_potentials_multi(const gqc_csr* g, const double* sigmas, int32_t n_sigma, const int32_t* devices,
                                int32_t n_shards, double* v_out);

/* Row blocks of a multi-device sweep: bounds[0] = 0 <= bounds[1] <= ... <=
 * bounds[n_shards] = n, shard r = rows [bounds[r], bounds[r+1]). Balanced by
 * the fast-forward kernel's cost per row (~ degree + 4), i.e. by an nnz
 * prefix over offsets; equal blocks w*floor(n/k) + min(w, n mod k)
 * (potential.cpp:70-74) under GQC_KERNEL_REPLAY, whose rows all cost n. */
gqc_status gqc_row_shards(const gqc_csr* g, int32_t n_shards, int32_t* bounds);

/* -------------------------------------------------------------- device API */
/* All pointers in gqc_csr and the buffers below are device pointers on the
 * current device; `stream` is a cudaStream_t (NULL = legacy default stream).
 * sigmas stays a host array (the per-sigma exp constants are a host concern).
 * Nothing is synchronized (except with GQC_OPT_HOP_CAP > 1, where a
 * potential launch reads the per-row event counts back once to size its
 * batches): errors from the kernels surface at the caller's next
 * synchronization. */

/* Potentials of rows [row_begin, row_end) for all sigmas, node-major:
 * v_rows[(i - row_begin) * n_sigma + k]. Row shards of a multi-GPU sweep. */
gqc_status gqc_dev_potentials(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                              int32_t row_end, double* v_rows, void* stream);

/* gqc_dev_potentials with the output packed in sigma chunks for a sigma-
 * sharded exchange: sigma k of row i goes to
 *     v_out[(k / chunk) * chunk_stride + (i - row_begin) * chunk + k % chunk],
 * so chunk q is a node-major [rows][chunk] block at q * chunk_stride (one
 * all-to-all then hands every rank the full rows of its own sigmas). Slots of
 * a last, partial chunk beyond n_sigma are not written. Same potentials as
 * gqc_dev_potentials (potential.cpp:18-37). */
gqc_status gqc_dev_potentials_packed(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                                     int32_t row_end, double* v_out, int32_t chunk, int64_t chunk_stride,
                                     void* stream);

/* gqc_dev_potentials with sigma chunk q (chunk sigmas each, n_chunks =
 * ceil(n_sigma / chunk) <= 32) of rows [row_begin, row_end) stored at
 *     chunk_ptrs[q][(i - row_begin) * chunk + k % chunk]
 * where each chunk_ptrs[q] is any device pointer the stream's device can
 * store to: local, a peer device's (NVLink), or another process's buffer
 * mapped with gqc_ipc_open. The potential kernel itself then delivers every
 * value to the rank that owns its sigma chunk — the multi-process form of the
 * fused exchange (no collective, no second copy of V). */
gqc_status gqc_dev_potentials_peer(const gqc_csr* g, const double* sigmas, int32_t n_sigma, int32_t row_begin,
                                   int32_t row_end, double* const* chunk_ptrs, int32_t n_chunks, int32_t chunk,
                                   void* stream);

/* Device memory shared between processes (CUDA IPC), on GQC_OPT_DEVICE:
 * gqc_ipc_alloc returns a dedicated allocation and its handle
 * (GQC_IPC_HANDLE_BYTES opaque bytes to pass to the other processes);
 * gqc_ipc_open maps a handle from another process, gqc_ipc_close unmaps it,
 * gqc_ipc_free releases an allocation of this process. */
#define GQC_IPC_HANDLE_BYTES 64
gqc_status gqc_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
gqc_status gqc_ipc_open(const void* handle, void** dev_ptr);
gqc_status gqc_ipc_close(void* dev_ptr);
gqc_status gqc_ipc_free(void* dev_ptr);

/* Scratch bytes gqc_dev_ggd needs for n nodes and n_sigma sigmas. */
size_t gqc_dev_ggd_workspace(int32_t n, int32_t n_sigma);

/* GGD for all sigmas from a node-major potential matrix v[n][n_sigma]:
 * sigma-major succ/center/cluster_index [n_sigma][n] and num_clusters[n_sigma]
 * (all device). succ may be NULL. */
gqc_status gqc_dev_ggd(const gqc_csr* g, const double* v, int32_t n_sigma, int32_t* succ, int32_t* center,
                       int32_t* cluster_index, int32_t* num_clusters, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Row-sharded GGD (multi-GPU): successors of rows [row_begin, row_end) from the
 * full node-major V, written node-major succ_rows[(i - row_begin) * n_sigma + k]
 * so equal row shards all-gather into one node-major succ[n][n_sigma]. */
gqc_status gqc_dev_successors(const gqc_csr* g, const double* v, int32_t n_sigma, int32_t row_begin, int32_t row_end,
                              int32_t* succ_rows, void* stream);

/* Centers and dense cluster indices (sigma-major [n_sigma][n]) and counts from
 * a node-major successor matrix succ_nm[n][n_sigma] built by gqc_dev_successors. */
size_t gqc_dev_resolve_workspace(int32_t n, int32_t n_sigma);
gqc_status gqc_dev_resolve(int32_t n, int32_t n_sigma, const int32_t* succ_nm, int32_t* center, int32_t* cluster_index,
                           int32_t* num_clusters, void* workspace, size_t workspace_bytes, void* stream);

/* Node-major [n][n_sigma] -> sigma-major [n_sigma][n] transpose (device). */
gqc_status gqc_dev_transpose(const double* v_nm, int32_t n, int32_t n_sigma, double* v_sm, void* stream);

/* Page-locked host memory for output staging (cudaHostAlloc on GQC_OPT_DEVICE):
 * label / field downloads into it run at PCIe speed and overlap the
 * remaining kernels (downloads into pageable memory are queued after them).
 * NULL on failure. */
void* gqc_host_alloc(size_t bytes);
void gqc_host_free(void* p);
/* Optional: size the context buffers of GQC_OPT_DEVICE for host-API sweeps
 * (gqc_cluster_sweep and friends) of graphs up to n nodes / nnz CSR entries
 * and n_sigma sigmas per call, and grow its stream-ordered scratch pool, so
 * the first call of a process does not allocate device memory on its
 * critical path (the CLI runs it on its device warm-up thread once the graph
 * is loaded). Later calls that need more still grow the buffers. */
gqc_status gqc_reserve(int32_t n, int64_t nnz, int32_t n_sigma);

/* Page-lock an existing host range (cudaHostRegister) / release it: a CSR
 * the caller keeps across calls then uploads at PCIe speed, under the
 * potential launch (the CLI registers its graph while it reads the labels). */
gqc_status gqc_host_register(void* p, size_t bytes);
gqc_status gqc_host_unregister(void* p);

/* Number of kernel launches the last gqc_* call issued (for launch accounting). */
int64_t gqc_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GQC_H */
