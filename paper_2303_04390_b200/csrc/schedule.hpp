// schedule.hpp -- host-side traversal planning (no CUDA).
//
// Turns the caller's post-order operation list (N-1 triples (dest, c1, c2),
// PAPER.md P:197-201 numbering, 0-based) into the two static per-pattern
// programs the traversal kernel executes:
//
//  * post program (Eq. 2): internal nodes in a depth-first
//    post-order in which, at every node, the child subtree that needs more
//    stack is evaluated first (Sethi-Ullman order).  Intermediate branch-top
//    vectors u = P p live in explicit per-thread stack slots; the plan names
//    the slot of every operand and result.
//  * pre program (Eq. 4): internal nodes in a depth-first
//    pre-order that descends into the smaller subtree first, so pending q
//    vectors never exceed ~log2(N) slots.
//
// Slot numbers are small (<= log2 N + 2 for bifurcating trees), so the whole
// per-pattern working set of both passes stays on chip; only u is written to
// HBM (post) and read back once (pre).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pg {

struct Op4 { int32_t x, y, z, w; };

// post op: x = node k (root when k == 2N-2), y/z = child codes, w = out slot
// pre  op: x = slot of q_k (-1 = root, q = pi), y/z = child nodes (codes),
//          w = (slot_y + 1) | ((slot_z + 1) << 16), 0 => tip child (no push)
// child code: >= 0 tip node id (bit 30 set when the tip uses partials),
//             <  0 internal: post = -(slot+1); pre = -(node+1)
constexpr int32_t kTipPartialBit = 1 << 30;

struct Plan {
    int32_t N = 0;
    std::vector<Op4> post, pre;
    int32_t post_depth = 0, pre_depth = 0;
    std::vector<int32_t> child_a, child_b;   // by node (internal only)
    // level-batched schedule (codon path): internal nodes grouped by height
    // (post, tips = 0) and by depth (pre, root = 0); level i of each is
    // level_nodes[off[i] .. off[i+1])
    std::vector<int32_t> level_nodes, post_off, pre_off;
};

// Returns 0 on success, else a PG_ERR_* code with *err filled.
int build_plan(int32_t N, const int32_t *ops, int32_t n_ops, Plan *out, std::string *err);

// Re-encode tip child codes with the partial-tip bit (mode per tip).
void encode_tip_modes(Plan *plan, const std::vector<uint8_t> &tip_is_partial);

}  // namespace pg
