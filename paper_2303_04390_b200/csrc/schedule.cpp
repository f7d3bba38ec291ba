// schedule.cpp -- see schedule.hpp.
#include "schedule.hpp"

#include <algorithm>
#include <cstdio>

#include "../../include/phylograd.h"

namespace pg {

namespace {

int fail(std::string *err, int code, const char *fmt, long a = 0, long b = 0) {
    char buf[256];
    std::snprintf(buf, sizeof buf, fmt, a, b);
    if (err) *err = buf;
    return code;
}

}  // namespace

int build_plan(int32_t N, const int32_t *ops, int32_t n_ops, Plan *out, std::string *err) {
    if (N < 2) return fail(err, PG_ERR_ARG, "tips must be >= 2 (got %ld)", N);
    if (!ops) return fail(err, PG_ERR_ARG, "ops is NULL");
    if (n_ops != N - 1)
        return fail(err, PG_ERR_TOPOLOGY, "need N-1 = %ld operations, got %ld", N - 1, n_ops);
    const int32_t nn = 2 * N - 1, root = 2 * N - 2;
    std::vector<int32_t> ca(nn, -1), cb(nn, -1), defined(nn, 0), used(nn, 0);
    for (int32_t n = 0; n < N; ++n) defined[n] = 1;
    for (int32_t o = 0; o < n_ops; ++o) {
        int32_t d = ops[3 * o], a = ops[3 * o + 1], b = ops[3 * o + 2];
        if (d < N || d > root)
            return fail(err, PG_ERR_TOPOLOGY, "op %ld: dest %ld is not an internal node id", o, d);
        if (a < 0 || a > root || b < 0 || b > root || a == b || a == d || b == d)
            return fail(err, PG_ERR_TOPOLOGY, "op %ld: bad children (dest %ld)", o, d);
        if (defined[d]) return fail(err, PG_ERR_TOPOLOGY, "op %ld: node %ld defined twice", o, d);
        for (int32_t c : {a, b}) {
            if (!defined[c])
                return fail(err, PG_ERR_TOPOLOGY, "op %ld: child %ld used before it is defined", o, c);
            if (used[c]) return fail(err, PG_ERR_TOPOLOGY, "node %ld has two parents (op %ld)", c, o);
            used[c] = 1;
        }
        defined[d] = 1;
        ca[d] = a;
        cb[d] = b;
    }
    if (ops[3 * (n_ops - 1)] != root)
        return fail(err, PG_ERR_TOPOLOGY, "last op must define the root %ld", root);
    // every non-root node has exactly one parent; the root none
    for (int32_t v = 0; v < nn; ++v)
        if ((v != root) != (used[v] != 0))
            return fail(err, PG_ERR_TOPOLOGY, "node %ld is not connected to the root", v);

    // ---- post program: Sethi-Ullman stack need, iterative ----------------
    std::vector<int32_t> need(nn, 0), size(nn, 1);
    for (int32_t o = 0; o < n_ops; ++o) {
        int32_t d = ops[3 * o], a = ca[d], b = cb[d];
        size[d] = size[a] + size[b];
        int32_t ia = a >= N, ib = b >= N;
        int32_t a_first = std::max({need[a], ia + need[b], 1});
        int32_t b_first = std::max({need[b], ib + need[a], 1});
        need[d] = std::min(a_first, b_first);
    }
    Plan plan;
    plan.N = N;
    plan.child_a = ca;
    plan.child_b = cb;
    plan.post.reserve(N - 1);
    plan.pre.reserve(N - 1);
    {
        // frame: node, base slot, stage (0 = start, 1 = after first, 2 = after second)
        struct F { int32_t k, base, stage, first, second, code1; };
        std::vector<F> st;
        st.push_back({root, 0, 0, -1, -1, 0});
        int32_t maxslot = 0;
        while (!st.empty()) {
            F &f = st.back();
            int32_t a = ca[f.k], b = cb[f.k];
            if (f.stage == 0) {
                int32_t ia = a >= N, ib = b >= N;
                int32_t a_first = std::max({need[a], ia + need[b], 1});
                int32_t b_first = std::max({need[b], ib + need[a], 1});
                f.first = (a_first <= b_first) ? a : b;
                f.second = (f.first == a) ? b : a;
                f.stage = 1;
                if (f.first >= N) { st.push_back({f.first, f.base, 0, -1, -1, 0}); continue; }
            }
            if (f.stage == 1) {
                int32_t next = f.base;
                if (f.first >= N) { f.code1 = -(f.base + 1); next = f.base + 1; }
                else f.code1 = f.first;
                f.stage = 2;
                if (f.second >= N) { int32_t k2 = f.second; st.push_back({k2, next, 0, -1, -1, 0}); continue; }
            }
            // stage 2: both children ready
            int32_t code2;
            if (f.second >= N) code2 = -((f.first >= N ? f.base + 1 : f.base) + 1);
            else code2 = f.second;
            plan.post.push_back({f.k, f.code1, code2, f.base});
            maxslot = std::max({maxslot, f.base + 1, code2 < 0 ? -code2 : 0});
            st.pop_back();
        }
        plan.post_depth = maxslot;
    }

    // ---- pre program: descend into the smaller subtree first -------------
    {
        struct E { int32_t k, slot; };
        std::vector<E> st;
        st.push_back({root, -1});
        int32_t sp = 0, maxsp = 0;
        while (!st.empty()) {
            E e = st.back();
            st.pop_back();
            if (e.slot >= 0) sp = e.slot;   // popping the top slot
            int32_t a = ca[e.k], b = cb[e.k];
            int32_t sooner = (size[a] <= size[b]) ? a : b;
            int32_t later = (sooner == a) ? b : a;
            int32_t sl = -1, ss = -1;
            if (later >= N) sl = sp++;
            if (sooner >= N) ss = sp++;
            maxsp = std::max(maxsp, sp);
            int32_t slot_a = (a == later) ? sl : ss, slot_b = (b == later) ? sl : ss;
            plan.pre.push_back({e.slot, a, b, (slot_a + 1) | ((slot_b + 1) << 16)});
            if (later >= N) st.push_back({later, sl});
            if (sooner >= N) st.push_back({sooner, ss});
        }
        plan.pre_depth = std::max(maxsp, 1);
    }
    // ---- level-batched schedule (codon path) -------------------------------
    {
        std::vector<int32_t> height(nn, 0), depth(nn, 0);
        int32_t H = 0;
        for (int32_t o = 0; o < n_ops; ++o) {
            const int32_t d = ops[3 * o];
            height[d] = 1 + std::max(height[ca[d]], height[cb[d]]);
            H = std::max(H, height[d]);
        }
        int32_t Dmax = 0;
        for (int32_t o = n_ops - 1; o >= 0; --o) {
            const int32_t d = ops[3 * o];
            depth[ca[d]] = depth[cb[d]] = depth[d] + 1;
            Dmax = std::max(Dmax, depth[d]);
        }
        // bucket by level (stable in op order): O(N)
        std::vector<std::vector<int32_t>> byh(H + 1), byd(Dmax + 1);
        for (int32_t o = 0; o < n_ops; ++o) byh[height[ops[3 * o]]].push_back(ops[3 * o]);
        for (int32_t o = n_ops - 1; o >= 0; --o) byd[depth[ops[3 * o]]].push_back(ops[3 * o]);
        plan.post_off.assign(1, 0);
        for (int32_t h = 1; h <= H; ++h) {
            plan.level_nodes.insert(plan.level_nodes.end(), byh[h].begin(), byh[h].end());
            plan.post_off.push_back((int32_t)plan.level_nodes.size());
        }
        plan.pre_off.assign(1, (int32_t)plan.level_nodes.size());
        for (int32_t dd = 0; dd <= Dmax; ++dd) {
            plan.level_nodes.insert(plan.level_nodes.end(), byd[dd].begin(), byd[dd].end());
            plan.pre_off.push_back((int32_t)plan.level_nodes.size());
        }
    }
    if ((int32_t)plan.post.size() != N - 1 || (int32_t)plan.pre.size() != N - 1)
        return fail(err, PG_ERR_TOPOLOGY, "internal planning error (%ld/%ld ops)",
                    (long)plan.post.size(), (long)plan.pre.size());
    *out = std::move(plan);
    return PG_OK;
}

void encode_tip_modes(Plan *plan, const std::vector<uint8_t> &tip_is_partial) {
    auto enc = [&](int32_t c) {
        if (c >= 0) {
            int32_t node = c & ~kTipPartialBit;
            if (node < plan->N && tip_is_partial[node]) return node | kTipPartialBit;
            return node;
        }
        return c;
    };
    for (auto &o : plan->post) { o.y = enc(o.y); o.z = enc(o.z); }
    for (auto &o : plan->pre) {
        auto enc_pre = [&](int32_t c) {
            int32_t node = c & ~kTipPartialBit;
            return (node < plan->N && tip_is_partial[node]) ? (node | kTipPartialBit) : node;
        };
        o.y = enc_pre(o.y);
        o.z = enc_pre(o.z);
    }
}

}  // namespace pg
