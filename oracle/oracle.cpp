// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT.
//
// A CPU restatement of the reference graphqc hot path (potential sweep + GGD)
// and of the host logic around it (ingestion, metrics, sigma grids, mutation
// detection, report formatting). Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library, and
// only as the checker or the timed CPU baseline — never as the product path.
//
// Every function cites the reference file:line it restates (paths relative to
// the reference's proj/ directory). The reference's build needs Eigen3, which
// this image lacks, so the restatement replaces Eigen::VectorXd by
// std::vector and restates the one third-party arithmetic the path depends
// on, Eigen 3.4's vectorised exp (pexp_double on SSE2 Packet2d), lane by lane.
//
// Pinning: tests/test_ref_pin.py checks this file bit for bit against the
// reference's OWN sources compiled in place (oracle/_ref, Makefile target
// `ref`, Eigen replaced by the restated subset in eigen_shim/): potentials,
// GGD, ingestion, metrics, sweep CSVs, grids. tests/test_oracle.py checks it
// against the reference's published goldens (README.md:58-59, :69;
// ggd_test.cpp:144-156; sweep_test.cpp:72-89, :144-153; metrics_test.cpp:65-97).
// Still unpinned: the exp BITS of an Eigen-built binary (no Eigen source here;
// both this file and eigen_shim restate Eigen 3.4's pexp_double).
//
// The k-hop distance extension (fill_khop) is NOT a reference feature; at hop
// cap 1 it is the reference's distance, and it is checked against a direct
// restatement of its definition in tests/test_oracle.py.
//
// Build: g++ -O2 -std=c++20 -ffp-contract=off (no -march: SSE2 scalar double,
// no FMA, exactly the reference's default Release arithmetic).
// ============================================================================
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace orc {

// ---------------------------------------------------------------------------
// Error model (graph.hpp:15-18; graphqc_main.cpp:373-390)
// ---------------------------------------------------------------------------
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum Status : int {
    OK = 0,
    E_INVAL = 1,   // std::invalid_argument
    E_RANGE = 2,   // std::out_of_range
    E_CYCLE = 3,   // std::logic_error
    E_IO = 4,      // IoError
    E_OTHER = 9,
};

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const IoError& e) {
        g_last_error = e.what();
        return E_IO;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return E_INVAL;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return E_RANGE;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return E_CYCLE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return E_OTHER;
    }
}

// ---------------------------------------------------------------------------
// format_double (format.cpp:7-11): shortest round-trip via std::to_chars
// ---------------------------------------------------------------------------
std::string format_double(double x) {
    char buf[32];
    auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), x);
    (void)ec;
    return std::string(buf, ptr);
}
std::string format_cell(const std::optional<double>& x) {
    return x ? format_double(*x) : std::string{};
}

// ---------------------------------------------------------------------------
// Third-party arithmetic: Eigen 3.4 pexp_double (GenericPacketMathFunctions.h)
// called from ArrayXd::exp at potential.cpp:26, one SSE2 lane at a time.
// SSE2 has no FMA, so every pmadd(a,b,c) is fl(fl(a*b)+c).
// ---------------------------------------------------------------------------
double eigen_pldexp(double a, double e) {
    // pldexp<Packet2d> (SSE/PacketMath.h): clamp e to [-2099, 2099], split 2^e
    // into 2^b * 2^b * 2^b * 2^(e-3b) with b = floor(e/4).
    e = std::min(std::max(e, -2099.0), 2099.0);
    const std::int32_t ei = static_cast<std::int32_t>(std::nearbyint(e));  // _mm_cvtpd_epi32 (e is integral)
    std::int32_t b = ei >> 2;                                            // arithmetic shift
    auto pow2 = [](std::int32_t k) {
        const std::uint64_t bits = static_cast<std::uint64_t>(static_cast<std::int64_t>(k) + 1023) << 52;
        double d;
        std::memcpy(&d, &bits, sizeof d);
        return d;
    };
    double c = pow2(b);
    double out = a * c;
    out = out * c;
    out = out * c;
    b = ei - b - b - b;
    c = pow2(b);
    return out * c;
}

double eigen_pexp(double x_in) {
    double x = x_in;
    // clamp x (pmin then pmax)
    x = std::min(x, 709.784);
    x = std::max(x, -709.784);
    // fx = floor(LOG2EF * x + 0.5)
    double fx = 1.4426950408889634073599 * x;
    fx = fx + 0.5;
    fx = std::floor(fx);
    // Cody-Waite reduction: x -= fx*C1; x -= fx*C2
    const double tmp = fx * 0.693145751953125;
    const double z = fx * 1.42860682030941723212e-6;
    x = x - tmp;
    x = x - z;
    const double x2 = x * x;
    // numerator
    double px = 1.26177193074810590878e-4;
    px = px * x2;
    px = px + 3.02994407707441961300e-2;
    px = px * x2;
    px = px + 9.99999999999999999910e-1;
    px = px * x;
    // denominator
    double qx = 3.00198505138664455042e-6;
    qx = qx * x2;
    qx = qx + 2.52448340349684104192e-3;
    qx = qx * x2;
    qx = qx + 2.27265548208155028766e-1;
    qx = qx * x2;
    qx = qx + 2.00000000000000000009e0;
    // x = 2 * px / (qx - px) + 1
    x = px / (qx - px);
    x = 2.0 * x;
    x = x + 1.0;
    // pmax(pldexp(x, fx), _x)  (_mm_max_pd: a > b ? a : b)
    const double r = eigen_pldexp(x, fx);
    return r > x_in ? r : x_in;
}

enum ExpMode : int { EXP_EIGEN = 0, EXP_GLIBC = 1 };

// ---------------------------------------------------------------------------
// Graph / CSR (graph.hpp:32-72, graph.cpp:25-71)
// ---------------------------------------------------------------------------
struct Edge {
    std::int32_t u, v;
    double w;
};

struct Graph {
    std::vector<std::int64_t> offsets{0};
    std::vector<std::int32_t> nbr;
    std::vector<double> wt;
    double W = 10.0;
    std::vector<std::string> names;
    std::unordered_map<std::string, std::int32_t> ids;

    std::int32_t n() const { return static_cast<std::int32_t>(offsets.size()) - 1; }
    std::int64_t nnz() const { return static_cast<std::int64_t>(nbr.size()); }
    void check_node(std::int32_t i) const {  // graph.cpp:73-76
        if (i < 0 || i >= n()) throw std::out_of_range("node id " + std::to_string(i) + " out of range");
    }
    double strength(std::int32_t i) const {  // graph.cpp:83-88
        check_node(i);
        double s = 0.0;
        for (std::int64_t k = offsets[i]; k < offsets[i + 1]; ++k) s += wt[k];
        return s;
    }
};

// graph.cpp:25-71: validate, intern default names, dedup with std::map keeping
// the first weight (warning on a conflicting one), drop self loops, fill rows
// in ascending key order so each row is ascending.
Graph make_graph(std::int32_t n, const std::vector<Edge>& edges, double W,
                 std::vector<std::string> names, bool warn = true) {
    if (n < 1) throw std::invalid_argument("graph needs at least one node");
    if (W <= 0.0) throw std::invalid_argument("default distance must be positive");
    if (!names.empty() && static_cast<std::int32_t>(names.size()) != n)
        throw std::invalid_argument("name list does not match node count");
    Graph g;
    g.W = W;
    if (names.empty()) {
        names.resize(n);
        for (std::int32_t i = 0; i < n; ++i) names[i] = std::to_string(i);
    }
    g.names = std::move(names);
    g.ids.reserve(g.names.size());
    for (std::int32_t i = 0; i < n; ++i)
        if (!g.ids.emplace(g.names[i], i).second)
            throw std::invalid_argument("duplicate node name: " + g.names[i]);

    std::map<std::pair<std::int32_t, std::int32_t>, double> unique;
    for (const Edge& e : edges) {
        if (e.u < 0 || e.u >= n || e.v < 0 || e.v >= n) throw std::out_of_range("edge endpoint out of range");
        if (e.w <= 0.0) throw std::invalid_argument("edge weight must be positive");
        if (e.u == e.v) continue;
        auto key = std::minmax(e.u, e.v);
        auto [it, inserted] = unique.emplace(key, e.w);
        if (!inserted && it->second != e.w && warn)
            std::cerr << "warning: duplicate edge " << g.names[key.first] << " " << g.names[key.second]
                      << " keeps weight " << format_double(it->second) << ", ignoring "
                      << format_double(e.w) << "\n";
    }
    std::vector<std::int32_t> deg(n, 0);
    for (const auto& [key, w] : unique) {
        ++deg[key.first];
        ++deg[key.second];
    }
    g.offsets.assign(n + 1, 0);
    for (std::int32_t i = 0; i < n; ++i) g.offsets[i + 1] = g.offsets[i] + deg[i];
    g.nbr.resize(g.offsets[n]);
    g.wt.resize(g.offsets[n]);
    std::vector<std::int64_t> cursor(g.offsets.begin(), g.offsets.end() - 1);
    for (const auto& [key, w] : unique) {
        g.nbr[cursor[key.first]] = key.second;
        g.wt[cursor[key.first]++] = w;
        g.nbr[cursor[key.second]] = key.first;
        g.wt[cursor[key.second]++] = w;
    }
    return g;
}

// graph.cpp:137-151
struct Line {
    std::size_t number;
    std::vector<std::string> tokens;
};
std::vector<Line> tokenized_lines(std::istream& in) {
    std::vector<Line> out;
    std::string line;
    std::size_t number = 0;
    while (std::getline(in, line)) {
        ++number;
        std::istringstream ls(line);
        std::vector<std::string> tokens;
        std::string tok;
        while (ls >> tok) tokens.push_back(tok);
        if (tokens.empty() || tokens[0][0] == '#') continue;
        out.push_back({number, std::move(tokens)});
    }
    return out;
}

// graph.cpp:153-159
double parse_weight(const std::string& tok, const std::string& where) {
    double w = 0.0;
    auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), w);
    if (ec != std::errc{} || ptr != tok.data() + tok.size())
        throw IoError(where + ": malformed weight '" + tok + "'");
    return w;
}

// graph.cpp:163-196
Graph parse_edge_list(std::istream& in, double W, const std::string& source) {
    if (W <= 0.0) throw std::invalid_argument("default distance must be positive");
    std::vector<std::string> names;
    std::unordered_map<std::string, std::int32_t> ids;
    auto intern = [&](const std::string& name) {
        auto [it, inserted] = ids.emplace(name, static_cast<std::int32_t>(names.size()));
        if (inserted) names.push_back(name);
        return it->second;
    };
    std::vector<Edge> edges;
    for (const Line& line : tokenized_lines(in)) {
        const std::string where = source + ": line " + std::to_string(line.number);
        if (line.tokens.size() != 2 && line.tokens.size() != 3)
            throw IoError(where + ": malformed line, expected 'u v' or 'u v w'");
        double w = 1.0;
        if (line.tokens.size() == 3) w = parse_weight(line.tokens[2], where);
        if (w <= 0.0) throw IoError(where + ": non-positive weight");
        const std::int32_t u = intern(line.tokens[0]);
        const std::int32_t v = intern(line.tokens[1]);
        if (u == v) continue;
        edges.push_back({u, v, w});
    }
    if (names.empty()) throw IoError(source + ": empty edge list");
    const std::int32_t n = static_cast<std::int32_t>(names.size());
    return make_graph(n, edges, W, std::move(names));
}
Graph load_edge_list(const std::string& path, double W) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path);
    return parse_edge_list(in, W, path);
}

// graph.cpp:204-233
struct LabelSet {
    std::vector<std::int32_t> labels;
    std::int32_t num_classes = 0;
};
LabelSet parse_labels(std::istream& in, const Graph& g, const std::string& source) {
    std::vector<std::int32_t> raw(g.n(), -1);
    std::vector<std::string> class_names;
    std::unordered_map<std::string, std::int32_t> class_ids;
    for (const Line& line : tokenized_lines(in)) {
        const std::string where = source + ": line " + std::to_string(line.number);
        if (line.tokens.size() != 2) throw IoError(where + ": malformed line, expected 'node label'");
        auto f = g.ids.find(line.tokens[0]);
        const std::int32_t node = f == g.ids.end() ? -1 : f->second;
        if (node < 0) throw IoError(where + ": unknown node '" + line.tokens[0] + "'");
        auto [it, inserted] = class_ids.emplace(line.tokens[1], static_cast<std::int32_t>(class_names.size()));
        if (inserted) class_names.push_back(line.tokens[1]);
        if (raw[node] != -1 && raw[node] != it->second)
            throw IoError(where + ": conflicting duplicate label for node '" + line.tokens[0] + "'");
        raw[node] = it->second;
    }
    for (std::int32_t i = 0; i < g.n(); ++i)
        if (raw[i] == -1) throw IoError(source + ": unlabeled node '" + g.names[i] + "'");
    return LabelSet{std::move(raw), static_cast<std::int32_t>(class_names.size())};
}
LabelSet load_labels(const std::string& path, const Graph& g) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path);
    return parse_labels(in, g, path);
}

// ---------------------------------------------------------------------------
// Potential engine (potential.cpp:12-87)
// ---------------------------------------------------------------------------
struct CsrView {
    std::int32_t n;
    const std::int64_t* offsets;
    const std::int32_t* nbr;
    const double* wt;  // nullptr => unit weights
    double W;
    int hop_cap = 1;   // 1 = the reference's distance (graph.cpp:258-267); > 1 = k-hop extension below
};

struct Workspace {  // potential.cpp:12-16 (+ BFS scratch of the k-hop extension)
    std::vector<double> dist2, gauss;
    std::vector<std::int32_t> hop, frontier, next;
    explicit Workspace(std::int32_t n) : dist2(n), gauss(n) {}
};

// k-hop distance extension (NOT in the reference, the
// north star's "multi-source BFS hop distances"): on a unit-weight graph,
// d(i,j) = 0 for j == i, h for a shortest path of h <= K hops, W otherwise.
// K = 1 is exactly the reference's pairwise_distance (graph.cpp:258-267,
// SPEC.md:69-77). The potential loop itself is unchanged (same Eigen
// packet/tail exp rule, same ascending sums). A plain level-synchronous BFS
// per row, written as the definition.
void fill_khop(const CsrView& g, std::int32_t i, Workspace& ws) {
    ws.hop.assign(g.n, -1);
    ws.frontier.assign(1, i);
    ws.hop[i] = 0;
    for (int h = 1; h <= g.hop_cap && !ws.frontier.empty(); ++h) {
        ws.next.clear();
        for (std::int32_t u : ws.frontier)
            for (std::int64_t k = g.offsets[u]; k < g.offsets[u + 1]; ++k) {
                const std::int32_t v = g.nbr[k];
                if (ws.hop[v] < 0) {
                    ws.hop[v] = h;
                    ws.next.push_back(v);
                }
            }
        if (h >= 2) {
            const double d = static_cast<double>(h);
            for (std::int32_t v : ws.next) ws.dist2[v] = d * d;
        }
        ws.frontier.swap(ws.next);
    }
}

// potential.cpp:18-37. ExpMode EIGEN: the linear-vectorised Eigen assignment
// evaluates whole Packet2d packets from index 0 with pexp and the N mod 2
// tail with scalar std::exp (glibc). ExpMode GLIBC: std::exp everywhere.
double potential_at(const CsrView& g, std::int32_t i, double inv, Workspace& ws, int mode) {
    const std::int32_t n = g.n;
    const double w2 = g.W * g.W;
    std::fill(ws.dist2.begin(), ws.dist2.end(), w2);
    for (std::int64_t k = g.offsets[i]; k < g.offsets[i + 1]; ++k) {
        const double w = g.wt ? g.wt[k] : 1.0;
        ws.dist2[g.nbr[k]] = w * w;
    }
    if (g.hop_cap > 1) fill_khop(g, i, ws);
    ws.dist2[i] = 0.0;

    const double neg = -inv;
    const std::int32_t packet_end = (mode == EXP_EIGEN) ? (n - n % 2) : 0;
    for (std::int32_t j = 0; j < packet_end; ++j) ws.gauss[j] = eigen_pexp(neg * ws.dist2[j]);
    for (std::int32_t j = packet_end; j < n; ++j) ws.gauss[j] = std::exp(neg * ws.dist2[j]);

    double num = 0.0;
    double den = 0.0;
    for (std::int32_t j = 0; j < n; ++j) {
        num += ws.dist2[j] * ws.gauss[j];
        den += ws.gauss[j];
    }
    return inv * (num / den);
}

// potential.cpp:39-42
double checked_inv_two_sigma_sq(double sigma) {
    if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
    return 1.0 / (2.0 * sigma * sigma);
}

// potential.cpp:62-87: contiguous blocks w*base + min(w, rem); caller does
// block 0. Bit-identical to the serial field (potential.cpp:53-60).
void compute_potentials_parallel(const CsrView& g, double sigma, int workers, int mode, double* out) {
    const double inv = checked_inv_two_sigma_sq(sigma);
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    const std::int32_t n = g.n;
    const std::int32_t base = n / workers;
    const std::int32_t rem = n % workers;
    auto block_begin = [&](int w) { return static_cast<std::int32_t>(w) * base + std::min<std::int32_t>(w, rem); };
    auto run_block = [&](std::int32_t b, std::int32_t e) {
        Workspace ws(n);
        for (std::int32_t i = b; i < e; ++i) out[i] = potential_at(g, i, inv, ws, mode);
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(run_block, block_begin(w), block_begin(w + 1));
    run_block(block_begin(0), block_begin(1));
    for (auto& t : pool) t.join();
}

// Row-sampled field (bench CPU baseline): the same per-row
// computation for an explicit list of rows, split over `workers` threads.
void potentials_rows(const CsrView& g, double sigma, int workers, int mode, const std::int32_t* rows,
                     std::int64_t nrows, double* out) {
    const double inv = checked_inv_two_sigma_sq(sigma);
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    std::vector<std::thread> pool;
    auto run = [&](std::int64_t b, std::int64_t e) {
        Workspace ws(g.n);
        for (std::int64_t k = b; k < e; ++k) {
            if (rows[k] < 0 || rows[k] >= g.n) throw std::out_of_range("row out of range");
            out[k] = potential_at(g, rows[k], inv, ws, mode);
        }
    };
    const std::int64_t base = nrows / workers, rem = nrows % workers;
    auto bb = [&](int w) { return w * base + std::min<std::int64_t>(w, rem); };
    for (int w = 1; w < workers; ++w) pool.emplace_back(run, bb(w), bb(w + 1));
    run(bb(0), bb(1));
    for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------------------
// GGD (ggd.cpp:7-62)
// ---------------------------------------------------------------------------
void build_successors(const CsrView& g, const double* v, std::int32_t* succ) {  // ggd.cpp:7-24
    for (std::int32_t i = 0; i < g.n; ++i) {
        std::int32_t best = i;
        for (std::int64_t k = g.offsets[i]; k < g.offsets[i + 1]; ++k) {
            const std::int32_t j = g.nbr[k];
            if (v[j] < v[best] || (v[j] == v[best] && j < best)) best = j;
        }
        succ[i] = best;
    }
}

struct Assignment {
    std::vector<std::int32_t> center, cluster_index, centers;
    std::int32_t num_clusters = 0;
};

Assignment resolve_centers(const std::int32_t* succ, std::int32_t n) {  // ggd.cpp:26-57
    Assignment out;
    out.center.assign(n, -1);
    std::vector<std::int32_t> path;
    for (std::int32_t i = 0; i < n; ++i) {
        if (out.center[i] != -1) continue;
        path.clear();
        std::int32_t x = i;
        std::int32_t steps = 0;
        while (out.center[x] == -1 && succ[x] != x) {
            if (succ[x] < 0 || succ[x] >= n) throw std::invalid_argument("successor id out of range");
            path.push_back(x);
            x = succ[x];
            if (++steps > n) throw std::logic_error("successor map contains a cycle");
        }
        const std::int32_t root = out.center[x] == -1 ? x : out.center[x];
        out.center[x] = root;
        for (std::int32_t p : path) out.center[p] = root;
    }
    for (std::int32_t i = 0; i < n; ++i)
        if (out.center[i] == i) out.centers.push_back(i);
    out.num_clusters = static_cast<std::int32_t>(out.centers.size());
    std::vector<std::int32_t> index_of(n, -1);
    for (std::int32_t k = 0; k < out.num_clusters; ++k) index_of[out.centers[k]] = k;
    out.cluster_index.resize(n);
    for (std::int32_t i = 0; i < n; ++i) out.cluster_index[i] = index_of[out.center[i]];
    return out;
}

CsrView view(const Graph& g) { return CsrView{g.n(), g.offsets.data(), g.nbr.data(), g.wt.data(), g.W}; }

Assignment cluster(const Graph& g, double sigma, int workers, int mode, std::vector<double>* v_out = nullptr) {
    std::vector<double> v(g.n());
    compute_potentials_parallel(view(g), sigma, workers, mode, v.data());  // ggd.cpp:59-62
    std::vector<std::int32_t> succ(g.n());
    build_successors(view(g), v.data(), succ.data());
    if (v_out) *v_out = v;
    return resolve_centers(succ.data(), g.n());
}

// ---------------------------------------------------------------------------
// Metrics (metrics.cpp:15-335)
// ---------------------------------------------------------------------------
double modularity(const Graph& g, const std::vector<std::int32_t>& clusters, double gamma) {  // :15-55
    const std::int32_t n = g.n();
    if (static_cast<std::int32_t>(clusters.size()) != n)
        throw std::invalid_argument("cluster assignment does not cover the graph");
    if (!(gamma > 0.0)) throw std::invalid_argument("gamma must be positive");
    std::int32_t k = 0;
    for (std::int32_t c : clusters) {
        if (c < 0) throw std::invalid_argument("negative cluster index");
        k = std::max(k, c + 1);
    }
    std::vector<double> strengths(n);
    for (std::int32_t i = 0; i < n; ++i) strengths[i] = g.strength(i);
    double w = 0.0;
    for (std::int32_t i = 0; i < n; ++i) w += strengths[i];
    if (w == 0.0) throw std::invalid_argument("modularity undefined for a graph with no edges");
    double intra = 0.0;
    for (std::int32_t i = 0; i < n; ++i) {
        double row = 0.0;
        for (std::int64_t t = g.offsets[i]; t < g.offsets[i + 1]; ++t)
            if (clusters[g.nbr[t]] == clusters[i]) row += g.wt[t];
        intra += row;
    }
    std::vector<double> cluster_strength(k, 0.0);
    for (std::int32_t i = 0; i < n; ++i) cluster_strength[clusters[i]] += strengths[i];
    double null_model = 0.0;
    for (std::int32_t c = 0; c < k; ++c) {
        const double frac = cluster_strength[c] / w;
        null_model += frac * frac;
    }
    return intra / w - gamma * null_model;
}

struct Contingency {  // metrics.hpp:15-20
    std::int32_t rows = 0, cols = 0;
    std::vector<std::int64_t> counts;  // row-major rows x cols
    std::vector<std::int64_t> row_sums, col_sums;
    std::int64_t total = 0;
    std::int64_t at(std::int32_t i, std::int32_t j) const { return counts[static_cast<std::size_t>(i) * cols + j]; }
};

Contingency contingency(const std::vector<std::int32_t>& truth, std::int32_t kt,
                        const std::vector<std::int32_t>& pred, std::int32_t kp) {  // :61-77
    if (truth.size() != pred.size()) throw std::invalid_argument("labelings cover different node sets");
    if (truth.empty()) throw std::invalid_argument("empty labelings");
    Contingency t;
    t.rows = kt;
    t.cols = kp;
    t.counts.assign(static_cast<std::size_t>(kt) * kp, 0);
    for (std::size_t i = 0; i < truth.size(); ++i) {
        if (truth[i] < 0 || truth[i] >= kt || pred[i] < 0 || pred[i] >= kp)
            throw std::invalid_argument("label index out of range");
        ++t.counts[static_cast<std::size_t>(truth[i]) * kp + pred[i]];
    }
    t.row_sums.assign(kt, 0);
    t.col_sums.assign(kp, 0);
    for (std::int32_t i = 0; i < kt; ++i)
        for (std::int32_t j = 0; j < kp; ++j) {
            t.row_sums[i] += t.at(i, j);
            t.col_sums[j] += t.at(i, j);
        }
    t.total = static_cast<std::int64_t>(truth.size());
    return t;
}

double comb2(std::int64_t x) { return 0.5 * static_cast<double>(x) * static_cast<double>(x - 1); }  // :88

bool partitions_identical(const Contingency& t) {  // :91-105
    for (std::int32_t i = 0; i < t.rows; ++i) {
        std::int64_t nz = 0;
        for (std::int32_t j = 0; j < t.cols; ++j)
            if (t.at(i, j) != 0) ++nz;
        if (nz != 1) return false;
    }
    for (std::int32_t j = 0; j < t.cols; ++j) {
        std::int64_t nz = 0;
        for (std::int32_t i = 0; i < t.rows; ++i)
            if (t.at(i, j) != 0) ++nz;
        if (nz != 1) return false;
    }
    return true;
}

double ari(const Contingency& t) {  // :109-123
    if (t.total < 2) throw std::invalid_argument("ari needs at least two samples");
    double sum_ij = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i)
        for (std::int32_t j = 0; j < t.cols; ++j) sum_ij += comb2(t.at(i, j));
    double sum_a = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i) sum_a += comb2(t.row_sums[i]);
    double sum_b = 0.0;
    for (std::int32_t j = 0; j < t.cols; ++j) sum_b += comb2(t.col_sums[j]);
    const double expected = sum_a * sum_b / comb2(t.total);
    const double denom = 0.5 * (sum_a + sum_b) - expected;
    if (denom == 0.0) return partitions_identical(t) ? 1.0 : 0.0;
    return (sum_ij - expected) / denom;
}

double fmi(const Contingency& t, bool warn = true) {  // :125-138
    double tp = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i)
        for (std::int32_t j = 0; j < t.cols; ++j) tp += comb2(t.at(i, j));
    double tp_fp = 0.0;
    for (std::int32_t j = 0; j < t.cols; ++j) tp_fp += comb2(t.col_sums[j]);
    double tp_fn = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i) tp_fn += comb2(t.row_sums[i]);
    if (tp_fp == 0.0 || tp_fn == 0.0) {
        if (warn) std::cerr << "warning: fmi undefined for an all-singleton partition, reporting 0\n";
        return 0.0;
    }
    return tp / std::sqrt(tp_fp * tp_fn);
}

double nmi(const Contingency& t) {  // :140-166
    const double n = static_cast<double>(t.total);
    double h_true = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i)
        if (t.row_sums[i] > 0) {
            const double p = t.row_sums[i] / n;
            h_true -= p * std::log(p);
        }
    double h_pred = 0.0;
    for (std::int32_t j = 0; j < t.cols; ++j)
        if (t.col_sums[j] > 0) {
            const double p = t.col_sums[j] / n;
            h_pred -= p * std::log(p);
        }
    if (h_true == 0.0 || h_pred == 0.0) return 0.0;
    double mi = 0.0;
    for (std::int32_t i = 0; i < t.rows; ++i)
        for (std::int32_t j = 0; j < t.cols; ++j) {
            if (t.at(i, j) == 0) continue;
            const double p = t.at(i, j) / n;
            const double pi = t.row_sums[i] / n;
            const double pj = t.col_sums[j] / n;
            mi += p * std::log(p / (pi * pj));
        }
    return mi / std::sqrt(h_true * h_pred);
}

std::vector<std::int32_t> best_mapping(const Contingency& t) {  // :171-209
    const std::int32_t k = t.rows;
    std::vector<std::int32_t> mapping(k);
    if (k <= 8) {
        std::vector<std::int32_t> perm(k);
        std::iota(perm.begin(), perm.end(), 0);
        std::int64_t best = -1;
        do {
            std::int64_t score = 0;
            for (std::int32_t j = 0; j < k; ++j) score += t.at(perm[j], j);
            if (score > best) {
                best = score;
                mapping = perm;
            }
        } while (std::next_permutation(perm.begin(), perm.end()));
        return mapping;
    }
    std::vector<bool> class_used(k, false), cluster_used(k, false);
    for (std::int32_t step = 0; step < k; ++step) {
        std::int64_t best = -1;
        std::int32_t bi = 0, bj = 0;
        for (std::int32_t i = 0; i < k; ++i) {
            if (class_used[i]) continue;
            for (std::int32_t j = 0; j < k; ++j) {
                if (cluster_used[j]) continue;
                if (t.at(i, j) > best) {
                    best = t.at(i, j);
                    bi = i;
                    bj = j;
                }
            }
        }
        class_used[bi] = true;
        cluster_used[bj] = true;
        mapping[bj] = bi;
    }
    return mapping;
}

struct Matched {
    double f1 = 0, accuracy = 0, recall = 0;
    std::vector<double> class_precision, class_recall, class_f1;
    std::vector<std::int32_t> cluster_to_class;
};

Matched matched_scores(const std::vector<std::int32_t>& truth, std::int32_t kt,
                       const std::vector<std::int32_t>& pred, std::int32_t kp) {  // :213-256
    if (kt != kp) throw std::invalid_argument("matched scores need equal cluster and class counts");
    const Contingency t = contingency(truth, kt, pred, kp);
    const std::int32_t k = kt;
    Matched m;
    m.cluster_to_class = best_mapping(t);
    std::int64_t matched = 0;
    for (std::int32_t j = 0; j < k; ++j) matched += t.at(m.cluster_to_class[j], j);
    m.accuracy = static_cast<double>(matched) / static_cast<double>(t.total);
    std::vector<std::int32_t> class_to_cluster(k);
    for (std::int32_t j = 0; j < k; ++j) class_to_cluster[m.cluster_to_class[j]] = j;
    m.class_precision.resize(k);
    m.class_recall.resize(k);
    m.class_f1.resize(k);
    for (std::int32_t c = 0; c < k; ++c) {
        const std::int32_t j = class_to_cluster[c];
        const double tp = static_cast<double>(t.at(c, j));
        const double fp = static_cast<double>(t.col_sums[j]) - tp;
        const double fn = static_cast<double>(t.row_sums[c]) - tp;
        const double precision = tp + fp > 0.0 ? tp / (tp + fp) : 0.0;
        const double recall = tp + fn > 0.0 ? tp / (tp + fn) : 0.0;
        m.class_precision[c] = precision;
        m.class_recall[c] = recall;
        m.class_f1[c] = precision + recall > 0.0 ? 2.0 * precision * recall / (precision + recall) : 0.0;
    }
    if (k == 2) {
        const std::int32_t positive = m.cluster_to_class[0];
        m.f1 = m.class_f1[positive];
        m.recall = m.class_recall[positive];
    } else {
        m.f1 = std::accumulate(m.class_f1.begin(), m.class_f1.end(), 0.0) / k;
        m.recall = std::accumulate(m.class_recall.begin(), m.class_recall.end(), 0.0) / k;
    }
    return m;
}

struct Report {  // metrics.hpp:45-53
    std::optional<double> modularity, nmi, ari, fmi;
    std::optional<Matched> matched;
    std::optional<std::int32_t> num_clusters;
    std::optional<double> sigma;
};

Report evaluate(const Graph& g, const Assignment& c, const LabelSet* labels, double gamma,
                std::optional<double> sigma) {  // :265-279
    Report r;
    r.modularity = modularity(g, c.cluster_index, gamma);
    r.num_clusters = c.num_clusters;
    r.sigma = sigma;
    if (labels) {
        const Contingency t = contingency(labels->labels, labels->num_classes, c.cluster_index, c.num_clusters);
        r.nmi = nmi(t);
        r.ari = ari(t);
        r.fmi = fmi(t);
        if (labels->num_classes == c.num_clusters)
            r.matched = matched_scores(labels->labels, labels->num_classes, c.cluster_index, c.num_clusters);
    }
    return r;
}

std::string metric_csv_header() { return "modularity,nmi,ari,fmi,f1,accuracy,recall,num_clusters,sigma"; }

std::string metric_csv_row(const Report& r) {  // :299-312
    std::ostringstream out;
    out << format_cell(r.modularity) << ',' << format_cell(r.nmi) << ',' << format_cell(r.ari) << ','
        << format_cell(r.fmi) << ',';
    if (r.matched)
        out << format_double(r.matched->f1) << ',' << format_double(r.matched->accuracy) << ','
            << format_double(r.matched->recall);
    else
        out << ",,";
    out << ',';
    if (r.num_clusters) out << *r.num_clusters;
    out << ',' << format_cell(r.sigma);
    return out.str();
}

// ---------------------------------------------------------------------------
// Sweep (sweep.cpp:11-80)
// ---------------------------------------------------------------------------
std::vector<double> log_sigma_grid(double W, int steps, double lo_f, double hi_f) {  // :11-26
    if (W <= 0.0 || lo_f <= 0.0 || hi_f <= lo_f) throw std::invalid_argument("invalid sigma grid bounds");
    if (steps < 1) throw std::invalid_argument("sigma grid needs at least one point");
    const double lo = std::log(lo_f * W);
    const double hi = std::log(hi_f * W);
    std::vector<double> grid(steps);
    if (steps == 1) {
        grid[0] = std::exp(lo);
        return grid;
    }
    for (int k = 0; k < steps; ++k) grid[k] = std::exp(lo + (hi - lo) * k / (steps - 1));
    return grid;
}

std::vector<double> linear_sigma_grid(double lo, double hi, int steps) {  // :28-38
    if (lo <= 0.0 || hi < lo) throw std::invalid_argument("invalid sigma grid bounds");
    if (steps < 1) throw std::invalid_argument("sigma grid needs at least one point");
    std::vector<double> grid(steps);
    if (steps == 1) {
        grid[0] = lo;
        return grid;
    }
    for (int k = 0; k < steps; ++k) grid[k] = lo + (hi - lo) * k / (steps - 1);
    return grid;
}

struct SweepRecord {
    double sigma;
    std::int32_t num_clusters;
    Report metrics;
};

std::vector<SweepRecord> run_sweep(const Graph& g, const std::vector<double>& sigmas, const LabelSet* labels,
                                   int workers, double gamma, int mode) {  // :40-59
    if (sigmas.empty()) throw std::invalid_argument("sigma grid is empty");
    for (std::size_t k = 0; k < sigmas.size(); ++k) {
        if (!(sigmas[k] > 0.0)) throw std::invalid_argument("sigma must be positive");
        if (k > 0 && sigmas[k] <= sigmas[k - 1]) throw std::invalid_argument("sigma grid must be strictly ascending");
    }
    std::vector<SweepRecord> records;
    for (double sigma : sigmas) {
        Assignment c = cluster(g, sigma, workers, mode);
        records.push_back({sigma, c.num_clusters, evaluate(g, c, labels, gamma, sigma)});
    }
    return records;
}

struct Mutation {
    double lo, hi;
    std::int32_t drop;
};
std::optional<Mutation> detect_mutation(const std::vector<SweepRecord>& r) {  // :61-71
    if (r.size() < 2) throw std::invalid_argument("mutation detection needs at least two records");
    std::optional<Mutation> best;
    for (std::size_t k = 0; k + 1 < r.size(); ++k) {
        const std::int32_t drop = r[k].num_clusters - r[k + 1].num_clusters;
        if (drop >= 1 && (!best || drop > best->drop)) best = Mutation{r[k].sigma, r[k + 1].sigma, drop};
    }
    return best;
}

std::string sweep_csv(const std::vector<SweepRecord>& records) {  // :73-80
    std::ostringstream out;
    out << "sigma,num_clusters,modularity,nmi,ari,fmi\n";
    for (const SweepRecord& r : records)
        out << format_double(r.sigma) << ',' << r.num_clusters << ',' << format_cell(r.metrics.modularity) << ','
            << format_cell(r.metrics.nmi) << ',' << format_cell(r.metrics.ari) << ','
            << format_cell(r.metrics.fmi) << '\n';
    return out.str();
}

// graphqc_main.cpp:68-73
std::string assignment_csv(const Graph& g, const Assignment& c) {
    std::ostringstream out;
    out << "node,center,cluster\n";
    for (std::int32_t i = 0; i < g.n(); ++i)
        out << g.names[i] << ',' << g.names[c.center[i]] << ',' << c.cluster_index[i] << '\n';
    return out.str();
}

// Copies s (NUL-terminated) when it fits; always reports the length so the
// caller can retry with a larger buffer.
void copy_out(const std::string& s, char* buf, std::int64_t cap, std::int64_t* len) {
    if (len) *len = static_cast<std::int64_t>(s.size());
    if (buf && cap > static_cast<std::int64_t>(s.size())) {
        std::memcpy(buf, s.data(), s.size());
        buf[s.size()] = 0;
    }
}

}  // namespace orc

// ===========================================================================
// C ABI for the Python test harness (ctypes). Status codes mirror the
// reference exception classes; orc_last_error() returns the message.
// ===========================================================================
using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

double orc_eigen_pexp(double x) { return eigen_pexp(x); }
double orc_glibc_exp(double x) { return std::exp(x); }

// Edge list (dense ids) -> CSR, graph.cpp:25-71. Buffers sized 2*m; *nnz out.
int orc_csr_from_edges(std::int32_t n, std::int64_t m, const std::int32_t* u, const std::int32_t* v,
                       const double* w, double W, std::int64_t* offsets, std::int32_t* nbr, double* wt,
                       std::int64_t* nnz) {
    return guarded([&] {
        std::vector<Edge> edges(m);
        for (std::int64_t k = 0; k < m; ++k) edges[k] = {u[k], v[k], w ? w[k] : 1.0};
        Graph g = make_graph(n, edges, W, {}, false);
        std::copy(g.offsets.begin(), g.offsets.end(), offsets);
        std::copy(g.nbr.begin(), g.nbr.end(), nbr);
        std::copy(g.wt.begin(), g.wt.end(), wt);
        *nnz = g.nnz();
    });
}

int orc_potentials(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* wt,
                   double W, double sigma, int workers, int mode, double* out) {
    return guarded([&] { compute_potentials_parallel(CsrView{n, offsets, nbr, wt, W}, sigma, workers, mode, out); });
}

int orc_potentials_rows(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* wt,
                        double W, double sigma, int workers, int mode, const std::int32_t* rows,
                        std::int64_t nrows, double* out) {
    return guarded([&] { potentials_rows(CsrView{n, offsets, nbr, wt, W}, sigma, workers, mode, rows, nrows, out); });
}

// k-hop extension entry points (hop_cap >= 1; > 1 needs unit weights).
int orc_potentials_khop(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* wt,
                        double W, double sigma, int hop_cap, int workers, int mode, const std::int32_t* rows,
                        std::int64_t nrows, double* out) {
    return guarded([&] {
        if (hop_cap < 1 || hop_cap > 7) throw std::invalid_argument("hop cap must be in 1..7");
        if (hop_cap > 1 && wt)
            for (std::int64_t k = 0; k < offsets[n]; ++k)
                if (wt[k] != 1.0) throw std::invalid_argument("k-hop distances need unit weights");
        CsrView g{n, offsets, nbr, wt, W, hop_cap};
        if (rows) potentials_rows(g, sigma, workers, mode, rows, nrows, out);
        else compute_potentials_parallel(g, sigma, workers, mode, out);
    });
}

int orc_build_successors(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* v,
                         std::int32_t* succ) {
    return guarded([&] { build_successors(CsrView{n, offsets, nbr, nullptr, 10.0}, v, succ); });
}

int orc_resolve_centers(std::int32_t n, const std::int32_t* succ, std::int32_t* center, std::int32_t* cluster_index,
                        std::int32_t* num_clusters) {
    return guarded([&] {
        Assignment a = resolve_centers(succ, n);
        std::copy(a.center.begin(), a.center.end(), center);
        std::copy(a.cluster_index.begin(), a.cluster_index.end(), cluster_index);
        *num_clusters = a.num_clusters;
    });
}

int orc_log_sigma_grid(double W, int steps, double lo_f, double hi_f, double* out) {
    return guarded([&] {
        auto g = log_sigma_grid(W, steps, lo_f, hi_f);
        std::copy(g.begin(), g.end(), out);
    });
}
int orc_linear_sigma_grid(double lo, double hi, int steps, double* out) {
    return guarded([&] {
        auto g = linear_sigma_grid(lo, hi, steps);
        std::copy(g.begin(), g.end(), out);
    });
}

// Metric row for an assignment of a CSR graph with optional labels
// (metrics.cpp:265-312). Writes the CSV row into buf.
int orc_metric_row(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* wt, double W,
                   const std::int32_t* cluster_index, std::int32_t num_clusters, const std::int32_t* labels,
                   std::int32_t num_classes, double gamma, double sigma, char* buf, std::int64_t cap,
                   std::int64_t* len) {
    return guarded([&] {
        Graph g;
        g.offsets.assign(offsets, offsets + n + 1);
        g.nbr.assign(nbr, nbr + offsets[n]);
        g.wt.resize(offsets[n]);
        for (std::int64_t k = 0; k < offsets[n]; ++k) g.wt[k] = wt ? wt[k] : 1.0;
        g.W = W;
        Assignment a;
        a.cluster_index.assign(cluster_index, cluster_index + n);
        a.num_clusters = num_clusters;
        LabelSet ls;
        if (labels) {
            ls.labels.assign(labels, labels + n);
            ls.num_classes = num_classes;
        }
        Report r = evaluate(g, a, labels ? &ls : nullptr, gamma, sigma);
        copy_out(metric_csv_row(r), buf, cap, len);
    });
}

// Mirrors `graphqc cluster <graph> [--labels L] --sigma S` (graphqc_main.cpp:86-105):
// assignment CSV into abuf, report (header + row) into rbuf.
int orc_run_cluster(const char* graph_path, const char* labels_path, double sigma, double W, int workers,
                    double gamma, int mode, char* abuf, std::int64_t acap, std::int64_t* alen, char* rbuf,
                    std::int64_t rcap, std::int64_t* rlen) {
    return guarded([&] {
        if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
        if (!(W > 0.0)) throw std::invalid_argument("default-distance must be positive");
        if (workers < 1) throw std::invalid_argument("workers must be at least 1");
        if (!(gamma > 0.0)) throw std::invalid_argument("gamma must be positive");
        Graph g = load_edge_list(graph_path, W);
        std::optional<LabelSet> labels;
        if (labels_path && *labels_path) labels = load_labels(labels_path, g);
        Assignment c = cluster(g, sigma, workers, mode);
        Report r = evaluate(g, c, labels ? &*labels : nullptr, gamma, sigma);
        copy_out(assignment_csv(g, c), abuf, acap, alen);
        copy_out(metric_csv_header() + "\n" + metric_csv_row(r) + "\n", rbuf, rcap, rlen);
    });
}

// Mirrors `graphqc sweep` (graphqc_main.cpp:115-157): sweep CSV into sbuf and
// the mutation line into mbuf.
int orc_run_sweep(const char* graph_path, const char* labels_path, double W, int workers, double gamma,
                  double sigma_min, double sigma_max, int steps, int log_grid, int mode, char* sbuf,
                  std::int64_t scap, std::int64_t* slen, char* mbuf, std::int64_t mcap, std::int64_t* mlen) {
    return guarded([&] {
        if (!(W > 0.0)) throw std::invalid_argument("default-distance must be positive");
        if (workers < 1) throw std::invalid_argument("workers must be at least 1");
        if (!(gamma > 0.0)) throw std::invalid_argument("gamma must be positive");
        if (steps < 1) throw std::invalid_argument("sigma-steps must be at least 1");
        const double lo = sigma_min > 0.0 ? sigma_min : 0.1 * W;
        const double hi = sigma_max > 0.0 ? sigma_max : 3.0 * W;
        if (!(lo > 0.0)) throw std::invalid_argument("sigma-min must be positive");
        if (!(hi >= lo)) throw std::invalid_argument("sigma-max must not be below sigma-min");
        std::vector<double> grid;
        if (steps == 1)
            grid = {lo};
        else if (log_grid)
            grid = log_sigma_grid(W, steps, lo / W, hi / W);
        else
            grid = linear_sigma_grid(lo, hi, steps);
        Graph g = load_edge_list(graph_path, W);
        std::optional<LabelSet> labels;
        if (labels_path && *labels_path) labels = load_labels(labels_path, g);
        auto records = run_sweep(g, grid, labels ? &*labels : nullptr, workers, gamma, mode);
        copy_out(sweep_csv(records), sbuf, scap, slen);
        std::string line = "mutation interval: none\n";
        if (records.size() >= 2) {
            if (auto m = detect_mutation(records))
                line = "mutation interval: [" + format_double(m->lo) + ", " + format_double(m->hi) +
                       "] drop=" + std::to_string(m->drop) + "\n";
        }
        copy_out(line, mbuf, mcap, mlen);
    });
}

int orc_detect_mutation(std::int32_t count, const double* sigmas, const std::int32_t* num_clusters, double* lo,
                        double* hi, std::int32_t* drop, std::int32_t* found) {
    return guarded([&] {
        std::vector<SweepRecord> r(count);
        for (std::int32_t k = 0; k < count; ++k) r[k] = {sigmas[k], num_clusters[k], {}};
        auto m = detect_mutation(r);
        *found = m ? 1 : 0;
        if (m) {
            *lo = m->lo;
            *hi = m->hi;
            *drop = m->drop;
        }
    });
}

// Contingency-based scores for two dense labelings (metrics.cpp:281-293,
// without modularity): out = {nmi, ari, fmi, f1, accuracy, recall}; matched
// fields are NaN when k_true != k_pred.
int orc_scores(std::int64_t n, const std::int32_t* truth, std::int32_t kt, const std::int32_t* pred,
               std::int32_t kp, double* out) {
    return guarded([&] {
        std::vector<std::int32_t> t(truth, truth + n), p(pred, pred + n);
        const Contingency c = contingency(t, kt, p, kp);
        out[0] = nmi(c);
        out[1] = ari(c);
        out[2] = fmi(c, false);
        out[3] = out[4] = out[5] = std::nan("");
        if (kt == kp) {
            Matched m = matched_scores(t, kt, p, kp);
            out[3] = m.f1;
            out[4] = m.accuracy;
            out[5] = m.recall;
        }
    });
}

int orc_modularity(std::int32_t n, const std::int64_t* offsets, const std::int32_t* nbr, const double* wt,
                   const std::int32_t* clusters, double gamma, double* out) {
    return guarded([&] {
        Graph g;
        g.offsets.assign(offsets, offsets + n + 1);
        g.nbr.assign(nbr, nbr + offsets[n]);
        g.wt.resize(offsets[n]);
        for (std::int64_t k = 0; k < offsets[n]; ++k) g.wt[k] = wt ? wt[k] : 1.0;
        *out = modularity(g, std::vector<std::int32_t>(clusters, clusters + n), gamma);
    });
}

}  // extern "C"
