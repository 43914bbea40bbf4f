// planner.cpp — host-side CDSP prefill scheduler: Eq. (1) latency model
// fit and Algorithms 1-3 of PAPER.md §5.1, producing the plan A that
// cdsp_plan_partition / cdsp_prefill_chunk consume.  The paper writes its scheduler in C++
// "to eliminate scheduling latency"; Table 2 reports <= 86.8 us per call.
//
// Readings: R21 (the recursion works inside the Step-0 group, queues advanced by
// Eq. 2), R22 (GetGroup node rules and tie-breaks), R23 (impossible extensions skipped), R24
// (Eq. 1 is quadratic in L: closed-form root instead of Newton), R25 (granule-aligned chunks),
// R26 (Illegal: length <= 0 or no split), R27 (line 11's garbled "if Illegal": recurse on legal
// plans).  Floating-point expressions keep the association order written in the comments so
// that plans are reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "common.cuh"

namespace cdsp {
namespace {

struct Inst {
    int id;
    double q;  // queuing latency T_i
};
using Pool = std::vector<Inst>;  // the instances a call may use
using Group = std::vector<int>;  // ring order

struct Alloc {
    std::vector<std::pair<int64_t, Group>> chunks;
};

struct Ctx {
    int node_size;
    const int32_t* sizes;
    int n_sizes;
    const cdsp_latency_model* models;
    double rate;
    int64_t granule;
    const cdsp_latency_model& model(int s) const {
        for (int i = 0; i < n_sizes; ++i)
            if (sizes[i] == s) return models[i];
        return models[0];  // unreachable: s always comes from sizes
    }
};

// Eq. (1): T_s(R) = a_s + b_s L + c_s (C L) + d_s L^2
double perf(const cdsp_latency_model& m, double C, double L) { return m.a + m.b * L + m.c * (C * L) + m.d * L * L; }

double qof(const Pool& p, int id) {
    for (const auto& x : p)
        if (x.id == id) return x.q;
    return 0.0;
}
bool has(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

// n shortest-queued of `ids` (ties: lower id)
std::vector<int> shortest(std::vector<int> ids, const Pool& p, size_t n) {
    std::sort(ids.begin(), ids.end(), [&](int a, int b) {
        const double qa = qof(p, a), qb = qof(p, b);
        return qa < qb || (qa == qb && a < b);
    });
    if (ids.size() > n) ids.resize(n);
    return ids;
}

// GetGroup: extend `initial` to s instances of the pool; false when impossible (R23)
bool get_group(const Pool& pool, int node_size, const Group& initial, int s, Group& out) {
    if (s < static_cast<int>(initial.size()) || s > static_cast<int>(pool.size())) return false;
    out = initial;
    int need = s - static_cast<int>(out.size());
    if (need == 0) return true;
    auto node = [&](int id) { return id / node_size; };
    if (!out.empty()) {  // (2) nodes already holding group instances first
        std::vector<int> cand;
        for (const auto& x : pool) {
            bool home = false;
            for (int g : out) home |= node(g) == node(x.id);
            if (home && !has(out, x.id)) cand.push_back(x.id);
        }
        for (int id : shortest(cand, pool, need)) out.push_back(id);
        need = s - static_cast<int>(out.size());
        if (need == 0) return true;
    }
    // (1) the remaining free nodes
    std::vector<int> nodes;
    for (const auto& x : pool)
        if (!has(nodes, node(x.id))) nodes.push_back(node(x.id));
    std::sort(nodes.begin(), nodes.end());
    auto members = [&](int nd) {
        std::vector<int> m;
        for (const auto& x : pool)
            if (node(x.id) == nd) m.push_back(x.id);
        return m;
    };
    std::vector<int> free_nodes;
    for (int nd : nodes) {
        bool used = false;
        for (int id : members(nd)) used |= has(out, id);
        if (!used) free_nodes.push_back(nd);
    }
    const int k_full = need / node_size;
    if (k_full > 0) {  // top-k full nodes by their longest queue (R22)
        std::vector<std::pair<double, int>> order;
        for (int nd : free_nodes) {
            const auto m = members(nd);
            if (static_cast<int>(m.size()) != node_size) continue;
            double mx = -std::numeric_limits<double>::infinity();
            for (int id : m) mx = std::max(mx, qof(pool, id));
            order.push_back({mx, nd});
        }
        std::sort(order.begin(), order.end());
        if (static_cast<int>(order.size()) < k_full) return false;
        for (int i = 0; i < k_full; ++i) {
            for (int id : shortest(members(order[i].second), pool, node_size)) out.push_back(id);
            free_nodes.erase(std::find(free_nodes.begin(), free_nodes.end(), order[i].second));
        }
        need = s - static_cast<int>(out.size());
    }
    if (need > 0) {  // the node whose need-th shortest queue is minimal
        bool found = false;
        std::pair<double, int> best{0.0, 0};
        for (int nd : free_nodes) {
            const auto m = members(nd);
            if (static_cast<int>(m.size()) < need) continue;
            std::vector<double> qs;
            for (int id : m) qs.push_back(qof(pool, id));
            std::sort(qs.begin(), qs.end());
            const std::pair<double, int> key{qs[need - 1], nd};
            if (!found || key < best) {
                best = key;
                found = true;
            }
        }
        if (!found) return false;
        for (int id : shortest(members(best.second), pool, need)) out.push_back(id);
    }
    return true;
}

double max_queue(const Pool& p, const Group& g) {
    double m = -std::numeric_limits<double>::infinity();
    for (int id : g) m = std::max(m, qof(p, id));
    return m;
}

int64_t total_len(const Alloc& A) {
    int64_t C = 0;
    for (const auto& c : A.chunks) C += c.first;
    return C;
}

// Algorithm 2
bool single_chunk(int64_t L, const Alloc& A, const std::vector<int>& S, const Pool& pool, const Ctx& cx, Group& opt_group,
                  double& opt_ttft) {
    const double C = static_cast<double>(total_len(A));
    const Group initial = A.chunks.empty() ? Group{} : A.chunks.back().second;
    opt_ttft = std::numeric_limits<double>::infinity();
    bool any = false;
    std::vector<int> ss = S;
    std::sort(ss.begin(), ss.end());
    for (int s : ss) {
        Group g;
        if (!get_group(pool, cx.node_size, initial, s, g)) continue;
        const double ttft = max_queue(pool, g) + perf(cx.model(s), C, static_cast<double>(L));
        if (ttft < opt_ttft * (1.0 - cx.rate)) {
            opt_ttft = ttft;
            opt_group = g;
            any = true;
        }
    }
    return any;
}

// Eq. (1) <= budget, largest L (R24)
double solve_len(const cdsp_latency_model& m, double C, double budget) {
    const double B = m.b + m.c * C;
    if (budget <= m.a) return 0.0;
    if (m.d <= 0.0) return B > 0 ? (budget - m.a) / B : std::numeric_limits<double>::infinity();
    return (-B + std::sqrt(B * B + 4.0 * m.d * (budget - m.a))) / (2.0 * m.d);
}

// R25: the largest multiple of g not above x, by an exact floor of x / g: the rounded quotient
// x / g can land on the next integer when x sits just below a multiple of g, so the integer
// candidate is corrected against exact products (k g < 2^53 is exact in a double).
int64_t whole_granules(double x, int64_t g) {
    if (!(x > 0.0)) return 0;
    const double gd = static_cast<double>(g);
    int64_t k = static_cast<int64_t>(x / gd);
    while (k > 0 && static_cast<double>(k) * gd > x) --k;
    while (static_cast<double>(k + 1) * gd <= x) ++k;
    return k * g;
}

// Algorithm 3
bool chunk_plan(int64_t L, const Alloc& A, int s_cur, int s_next, const Pool& pool, const Ctx& cx, int64_t& l_chunk,
                Group& cur) {
    const double C = static_cast<double>(total_len(A));
    const Group initial = A.chunks.empty() ? Group{} : A.chunks.back().second;
    Group nxt;
    if (!get_group(pool, cx.node_size, initial, s_cur, cur)) return false;
    if (!get_group(pool, cx.node_size, cur, s_next, nxt)) return false;
    const double budget = max_queue(pool, nxt) - max_queue(pool, cur);
    const double x = std::min(static_cast<double>(L), solve_len(cx.model(s_cur), C, budget));
    l_chunk = whole_granules(x, cx.granule);
    return true;
}

// Algorithm 1 (recursive); returns false when no allocation exists
bool cdsp_sched(int64_t L, const Alloc& A, const std::vector<int>& S, const Pool& pool, const Ctx& cx, Alloc& opt,
                double& opt_ttft) {
    Group group;
    double ttft;
    if (!single_chunk(L, A, S, pool, cx, group, ttft)) return false;  // line 3
    opt = A;
    opt.chunks.push_back({L, group});  // line 4
    opt_ttft = ttft;
    std::vector<int> s_cdsp;
    for (int s : S)
        if (s <= static_cast<int>(group.size())) s_cdsp.push_back(s);  // line 6
    std::sort(s_cdsp.begin(), s_cdsp.end());
    Pool in_group;  // line 10 works within instance_group (R21)
    for (int id : group) in_group.push_back({id, qof(pool, id)});
    const double C = static_cast<double>(total_len(A));
    for (size_t i = 0; i < s_cdsp.size(); ++i)
        for (size_t j = 0; j < s_cdsp.size(); ++j) {
            const int s_cur = s_cdsp[i], s_next = s_cdsp[j];
            if (!(s_cur < s_next)) continue;  // line 7
            int64_t l_chunk;
            Group cur;
            if (!chunk_plan(L, A, s_cur, s_next, in_group, cx, l_chunk, cur)) continue;  // line 10
            if (l_chunk <= 0 || l_chunk >= L) continue;                                 // line 11 (R26, R27)
            const double elapsed =
                max_queue(in_group, cur) + perf(cx.model(s_cur), C, static_cast<double>(l_chunk));
            Pool p2;  // Eq. (2)
            for (const auto& x : in_group) p2.push_back({x.id, std::max(0.0, x.q - elapsed)});
            std::vector<int> s2;
            for (int s : s_cdsp)
                if (s >= s_next) s2.push_back(s);  // line 15
            Alloc a2 = A;
            a2.chunks.push_back({l_chunk, cur});
            Alloc rest_alloc;
            double rest;
            if (!cdsp_sched(L - l_chunk, a2, s2, p2, cx, rest_alloc, rest)) continue;  // line 17
            if (elapsed + rest < opt_ttft) {                                          // line 19
                opt = rest_alloc;
                opt_ttft = elapsed + rest;
            }
        }
    return true;
}

}  // namespace
}  // namespace cdsp

using namespace cdsp;

extern "C" {

cdsp_status cdsp_fit_latency_model(int32_t n, const double* C, const double* L, const double* T,
                                   cdsp_latency_model* out) {
    CDSP_REQUIRE(n >= 4 && C && L && T && out, CDSP_ERR_INVALID, "need n >= 4 samples and non-NULL arrays");
    // least squares on the features [1, L, C L, L^2], columns scaled to unit max,
    // Householder QR (the features span ~20 orders of magnitude: no normal equations)
    const int m = n, k = 4;
    std::vector<double> X(static_cast<size_t>(m) * k), y(T, T + m);
    double scale[4] = {0, 0, 0, 0};
    for (int i = 0; i < m; ++i) {
        const double f[4] = {1.0, L[i], C[i] * L[i], L[i] * L[i]};
        for (int j = 0; j < k; ++j) {
            X[static_cast<size_t>(i) * k + j] = f[j];
            scale[j] = std::max(scale[j], std::fabs(f[j]));
        }
    }
    for (int j = 0; j < k; ++j) {
        if (scale[j] == 0.0) scale[j] = 1.0;
        for (int i = 0; i < m; ++i) X[static_cast<size_t>(i) * k + j] /= scale[j];
    }
    for (int j = 0; j < k; ++j) {  // Householder on column j
        double nrm = 0.0;
        for (int i = j; i < m; ++i) nrm += X[static_cast<size_t>(i) * k + j] * X[static_cast<size_t>(i) * k + j];
        nrm = std::sqrt(nrm);
        CDSP_REQUIRE(nrm > 0.0, CDSP_ERR_INVALID, "samples do not determine coefficient %d", j);
        const double x0 = X[static_cast<size_t>(j) * k + j];
        const double alpha = x0 > 0 ? -nrm : nrm;
        std::vector<double> v(m, 0.0);
        for (int i = j; i < m; ++i) v[i] = X[static_cast<size_t>(i) * k + j];
        v[j] -= alpha;
        double vv = 0.0;
        for (int i = j; i < m; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        for (int c = j; c < k; ++c) {
            double dot = 0.0;
            for (int i = j; i < m; ++i) dot += v[i] * X[static_cast<size_t>(i) * k + c];
            const double f = 2.0 * dot / vv;
            for (int i = j; i < m; ++i) X[static_cast<size_t>(i) * k + c] -= f * v[i];
        }
        double dot = 0.0;
        for (int i = j; i < m; ++i) dot += v[i] * y[i];
        const double f = 2.0 * dot / vv;
        for (int i = j; i < m; ++i) y[i] -= f * v[i];
    }
    double beta[4];
    for (int j = k - 1; j >= 0; --j) {  // back substitution R beta = Q^T y
        double s = y[j];
        for (int c = j + 1; c < k; ++c) s -= X[static_cast<size_t>(j) * k + c] * beta[c];
        const double rjj = X[static_cast<size_t>(j) * k + j];
        CDSP_REQUIRE(rjj != 0.0, CDSP_ERR_INVALID, "rank-deficient samples");
        beta[j] = s / rjj;
    }
    out->a = beta[0] / scale[0];
    out->b = beta[1] / scale[1];
    out->c = beta[2] / scale[2];
    out->d = beta[3] / scale[3];
    return CDSP_OK;
}

cdsp_status cdsp_schedule_prefill(int64_t L, int32_t n_instances, const double* queue, int32_t node_size,
                                  int32_t n_sizes, const int32_t* sizes, const cdsp_latency_model* models,
                                  double improvement_rate, int64_t granule, cdsp_schedule* out) {
    CDSP_REQUIRE(queue && sizes && models && out, CDSP_ERR_INVALID, "NULL argument");
    CDSP_REQUIRE(n_instances >= 1 && n_instances <= 1024, CDSP_ERR_INVALID, "n_instances %d", n_instances);
    CDSP_REQUIRE(node_size >= 1, CDSP_ERR_INVALID, "node_size %d", node_size);
    CDSP_REQUIRE(n_sizes >= 1 && n_sizes <= 4, CDSP_ERR_INVALID, "n_sizes %d not in [1,4]", n_sizes);
    int max_s = 1;
    for (int i = 0; i < n_sizes; ++i) {
        CDSP_REQUIRE(sizes[i] == 1 || sizes[i] == 2 || sizes[i] == 4 || sizes[i] == 8, CDSP_ERR_PLAN,
                     "SP size %d not in {1,2,4,8}", sizes[i]);
        for (int j = 0; j < i; ++j) CDSP_REQUIRE(sizes[i] != sizes[j], CDSP_ERR_INVALID, "duplicate SP size");
        max_s = std::max(max_s, static_cast<int>(sizes[i]));
    }
    CDSP_REQUIRE(granule >= 1 && granule % (2 * max_s) == 0, CDSP_ERR_SHAPE,
                 "granule %lld must be a multiple of 2 * max SP size", static_cast<long long>(granule));
    CDSP_REQUIRE(L >= granule && L % granule == 0, CDSP_ERR_SHAPE, "prompt length %lld not a granule multiple",
                 static_cast<long long>(L));
    CDSP_REQUIRE(improvement_rate >= 0.0 && improvement_rate < 1.0, CDSP_ERR_INVALID, "improvement rate %f",
                 improvement_rate);
    Pool pool;
    for (int i = 0; i < n_instances; ++i) {
        CDSP_REQUIRE(queue[i] >= 0.0 && std::isfinite(queue[i]), CDSP_ERR_INVALID, "queue[%d] = %f", i, queue[i]);
        pool.push_back({i, queue[i]});
    }
    const Ctx cx{node_size, sizes, n_sizes, models, improvement_rate, granule};
    std::vector<int> S(sizes, sizes + n_sizes);
    Alloc opt;
    double ttft;
    CDSP_REQUIRE(cdsp_sched(L, Alloc{}, S, pool, cx, opt, ttft), CDSP_ERR_PLAN,
                 "no SP size fits the instance pool");
    CDSP_REQUIRE(static_cast<int>(opt.chunks.size()) <= CDSP_MAX_CHUNKS, CDSP_ERR_CAPACITY, "too many chunks");
    std::memset(out, 0, sizeof(*out));
    out->n_chunks = static_cast<int32_t>(opt.chunks.size());
    for (size_t c = 0; c < opt.chunks.size(); ++c) {
        out->len[c] = opt.chunks[c].first;
        out->sp[c] = static_cast<int32_t>(opt.chunks[c].second.size());
        for (size_t r = 0; r < opt.chunks[c].second.size(); ++r) out->ranks[c][r] = opt.chunks[c].second[r];
    }
    out->ttft = ttft;
    return CDSP_OK;
}

}  // extern "C"
