// hedl_compile: hypothesis node arrays -> canonical DAG program.
//
// Paper: a hypothesis is a flat array of DL operations (§IV);
// an evaluation plan fixes the order of operations and their inputs
// (PAPER.md:532).  Here the plan is a hash-consed DAG shared by all roots
// (common-subexpression reuse), with topological levels for level-synchronous
// batched launches and the per-node algorithmic byte model of SURVEY 8(d).
//
// Canonicalisation (default): complement folded into operand
// references (the paper's per-operand isNegated XOR flag, Alg. 1-2),
// so NOT NOT C == C; n-ary AND/OR flattened, operands sorted and deduplicated
// (an n-ary operation is one step).  No algebraic rewrites.
#include <algorithm>
#include <cmath>

#include "internal.h"

using namespace hedl;

namespace {

inline uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}

struct Builder {
    hedl_program *p;
    const hedl_kb *kb;
    bool cse;
    std::vector<uint32_t> table;   // open addressing: node id + 1, 0 = empty
    uint64_t mask = 0;
    uint32_t count = 0;

    uint64_t hash_node(const CNode &n, const uint32_t *ops) const {
        uint64_t h = mix(n.kind, n.pred);
        h = mix(h, n.dir);
        h = mix(h, n.n);
        uint32_t lo, hi;
        std::memcpy(&lo, &n.lo, 4);
        std::memcpy(&hi, &n.hi, 4);
        h = mix(h, ((uint64_t)lo << 32) | hi);
        for (uint32_t i = 0; i < n.op_count; ++i) h = mix(h, ops[i]);
        return h;
    }
    bool same(const CNode &a, const CNode &b, const uint32_t *bops) const {
        if (a.kind != b.kind || a.pred != b.pred || a.dir != b.dir || a.n != b.n || a.op_count != b.op_count) return false;
        if (std::memcmp(&a.lo, &b.lo, 4) || std::memcmp(&a.hi, &b.hi, 4)) return false;
        return std::equal(bops, bops + b.op_count, p->ops.begin() + a.op_begin);
    }
    void grow() {
        uint64_t cap = table.empty() ? 1024 : table.size() * 2;
        std::vector<uint32_t> t(cap, 0);
        uint64_t m = cap - 1;
        for (uint32_t id = 0; id < p->nodes.size(); ++id) {
            const CNode &n = p->nodes[id];
            uint64_t h = hash_node(n, p->ops.data() + n.op_begin) & m;
            while (t[h]) h = (h + 1) & m;
            t[h] = id + 1;
        }
        table.swap(t);
        mask = m;
    }
    // intern node `n` with operands `ops`; returns node id
    uint32_t intern(CNode n, const uint32_t *ops) {
        uint64_t h = 0;
        if (cse) {
            if ((uint64_t)(p->nodes.size() + 1) * 2 > table.size()) grow();
            h = hash_node(n, ops) & mask;
            while (table[h]) {
                const uint32_t id = table[h] - 1;
                if (same(p->nodes[id], n, ops)) return id;
                h = (h + 1) & mask;
            }
        }
        n.op_begin = (uint32_t)p->ops.size();
        p->ops.insert(p->ops.end(), ops, ops + n.op_count);
        uint32_t lvl = 0;
        bool has_node = false;
        for (uint32_t i = 0; i < n.op_count; ++i)
            if (ref_type(ops[i]) == RT_NODE) {
                has_node = true;
                lvl = std::max(lvl, p->nodes[ref_id(ops[i])].level);
            }
        n.level = has_node ? lvl + 1 : 0;
        const double W4b = 4.0 * kb->W;
        if (n.kind == NK_AND || n.kind == NK_OR) n.bytes = (n.op_count + 1) * W4b;
        else if (n.kind == NK_RESTRICT) n.bytes = kb->dir_bytes[n.dir] + 2 * W4b;
        else n.bytes = kb->data_bytes[n.dir] + W4b;
        const uint32_t id = (uint32_t)p->nodes.size();
        p->nodes.push_back(n);
        if (cse) table[h] = id + 1;
        return id;
    }
};

}  // namespace

extern "C" hedl_status hedl_compile(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                                    const uint32_t *child_idx, uint64_t n_child_idx,
                                    const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                                    hedl_program **out) {
    if (!kb || !out) return fail(HEDL_ERR_INVALID_ARG, "null kb/out");
    *out = nullptr;
    if ((n_nodes && !nodes) || (n_child_idx && !child_idx) || (n_roots && !roots))
        return fail(HEDL_ERR_INVALID_ARG, "null node/child/root array");
    if (n_nodes >= (1u << 28)) return fail(HEDL_ERR_INVALID_ARG, "too many nodes in one program (max 2^28)");
    const bool rewrite = !(flags & HEDL_COMPILE_NO_REWRITE);
    const bool compat = flags & HEDL_COMPILE_COMPAT_PAPER_MAX;

    hedl_program *p = new hedl_program();
    p->kb = kb;
    p->flags = flags;
    p->nodes.reserve(n_nodes);
    p->ops.reserve(n_child_idx + n_roots);
    Builder B{p, kb, !(flags & HEDL_COMPILE_NO_CSE)};

    const uint32_t UNSET = 0xffffffffu;
    std::vector<uint32_t> ref(n_nodes, UNSET);
    std::vector<uint8_t> state(n_nodes, 0);     // 0 new, 1 on stack, 2 done
    std::vector<std::pair<uint32_t, uint32_t>> stack;
    std::vector<uint32_t> tmp;
    auto bad = [&](hedl_status st, uint32_t i, const std::string &m) {
        delete p;
        return fail(st, "node " + std::to_string(i) + ": " + m);
    };

    for (uint32_t ri = 0; ri < n_roots; ++ri) {
        if (roots[ri] >= n_nodes) { delete p; return fail(HEDL_ERR_OUT_OF_RANGE, "root " + std::to_string(ri) + " out of range"); }
        if (state[roots[ri]] == 2) continue;
        stack.clear();
        stack.push_back({roots[ri], 0});
        state[roots[ri]] = 1;
        while (!stack.empty()) {
            const uint32_t i = stack.back().first;
            const hedl_node &nd = nodes[i];
            if ((uint64_t)nd.child_begin + nd.child_count > n_child_idx)
                return bad(HEDL_ERR_OUT_OF_RANGE, i, "child range out of bounds");
            uint32_t &k = stack.back().second;
            if (k < nd.child_count) {
                const uint32_t c = child_idx[nd.child_begin + k++];
                if (c >= n_nodes) return bad(HEDL_ERR_OUT_OF_RANGE, i, "child id out of range");
                if (state[c] == 1) return bad(HEDL_ERR_BAD_EXPR, i, "cycle");
                if (state[c] == 0) { state[c] = 1; stack.push_back({c, 0}); }
                continue;
            }
            // all children are done: build the canonical reference of node i
            const uint32_t *ch = child_idx + nd.child_begin;
            const uint32_t cc = nd.child_count;
            const bool is_role = nd.op >= HEDL_OP_EXISTS && nd.op <= HEDL_OP_EXACT;
            if (nd.flags & ~HEDL_FLAG_INV) return bad(HEDL_ERR_BAD_EXPR, i, "unknown flag bits");
            if ((nd.flags & HEDL_FLAG_INV) && !is_role) return bad(HEDL_ERR_BAD_EXPR, i, "inverse flag on a non-role node");
            uint32_t r = 0;
            switch (nd.op) {
            case HEDL_OP_TOP:
            case HEDL_OP_BOTTOM:
                if (cc) return bad(HEDL_ERR_BAD_EXPR, i, "TOP/BOTTOM take no children");
                r = mkref(RT_TOP, 0, nd.op == HEDL_OP_BOTTOM);
                break;
            case HEDL_OP_ATOM:
                if (cc) return bad(HEDL_ERR_BAD_EXPR, i, "ATOM takes no children");
                if (nd.arg >= kb->C) return bad(HEDL_ERR_OUT_OF_RANGE, i, "concept id out of range");
                r = mkref(RT_ATOM, nd.arg, 0);
                break;
            case HEDL_OP_NOT:
                if (cc != 1) return bad(HEDL_ERR_BAD_EXPR, i, "NOT takes one child");
                r = ref[ch[0]] ^ 1u;   // complement over Delta (Q1); NOT NOT C == C
                break;
            case HEDL_OP_AND:
            case HEDL_OP_OR: {
                const uint8_t kind = nd.op == HEDL_OP_AND ? NK_AND : NK_OR;
                tmp.clear();
                for (uint32_t j = 0; j < cc; ++j) {
                    const uint32_t cr = ref[ch[j]];
                    if (rewrite && ref_type(cr) == RT_NODE && !ref_comp(cr) && p->nodes[ref_id(cr)].kind == kind) {
                        const CNode &sub = p->nodes[ref_id(cr)];
                        for (uint32_t q = 0; q < sub.op_count; ++q) tmp.push_back(p->ops[sub.op_begin + q]);
                    } else {
                        tmp.push_back(cr);
                    }
                }
                if (rewrite) {
                    std::sort(tmp.begin(), tmp.end());
                    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
                }
                if (tmp.empty()) {                         // empty AND = TOP, empty OR = BOTTOM
                    r = mkref(RT_TOP, 0, kind == NK_OR);
                } else if (tmp.size() == 1 && rewrite) {
                    r = tmp[0];
                } else {
                    CNode n{};
                    n.kind = kind;
                    n.op_count = (uint32_t)tmp.size();
                    r = mkref(RT_NODE, B.intern(n, tmp.data()), 0);
                }
                break;
            }
            case HEDL_OP_EXISTS: case HEDL_OP_FORALL: case HEDL_OP_MIN: case HEDL_OP_MAX: case HEDL_OP_EXACT: {
                if (cc != 1) return bad(HEDL_ERR_BAD_EXPR, i, "role restriction takes one child");
                if (nd.arg >= kb->R) return bad(HEDL_ERR_OUT_OF_RANGE, i, "role id out of range");
                if (nd.n > 0xfffffffeu) return bad(HEDL_ERR_BAD_EXPR, i, "n > 2^32-2");
                CNode n{};
                n.kind = NK_RESTRICT;
                n.dir = (uint16_t)(2 * nd.arg + (nd.flags & HEDL_FLAG_INV ? 1 : 0));
                n.op_count = 1;
                uint32_t child = ref[ch[0]];
                switch (nd.op) {
                case HEDL_OP_EXISTS: n.pred = P_GE; n.n = 1; n.sat = 1; break;           // Alg. 4
                case HEDL_OP_FORALL: n.pred = P_LE; n.n = 0; n.sat = 1; child ^= 1u; break; // Alg. 6
                case HEDL_OP_MIN: n.pred = P_GE; n.n = nd.n; n.sat = nd.n; break;        // Alg. 7 MIN
                case HEDL_OP_MAX: n.pred = compat ? P_LEP : P_LE; n.n = nd.n; n.sat = nd.n + 1; break;
                default: n.pred = P_EQ; n.n = nd.n; n.sat = nd.n + 1; break;             // EXACTLY
                }
                r = mkref(RT_NODE, B.intern(n, &child), 0);
                break;
            }
            case HEDL_OP_DRANGE: {
                if (cc) return bad(HEDL_ERR_BAD_EXPR, i, "DRANGE takes no children");
                if (std::isnan(nd.lo) || std::isnan(nd.hi)) return bad(HEDL_ERR_BAD_EXPR, i, "NaN bound");
                if (nd.arg >= kb->D) return bad(HEDL_ERR_OUT_OF_RANGE, i, "data property id out of range");
                CNode n{};
                n.kind = NK_DRANGE;
                n.dir = (uint16_t)nd.arg;
                n.lo = nd.lo;
                n.hi = nd.hi;
                r = mkref(RT_NODE, B.intern(n, nullptr), 0);
                break;
            }
            default:
                return bad(HEDL_ERR_BAD_EXPR, i, "unknown opcode");
            }
            ref[i] = r;
            state[i] = 2;
            stack.pop_back();
        }
    }
    // every root becomes a computed, uncomplemented node (a 1-operand AND
    // materialises atoms, constants and complemented references)
    p->root_node.resize(n_roots);
    for (uint32_t ri = 0; ri < n_roots; ++ri) {
        const uint32_t r = ref[roots[ri]];
        if (ref_type(r) == RT_NODE && !ref_comp(r)) {
            p->root_node[ri] = ref_id(r);
        } else {
            CNode n{};
            n.kind = NK_AND;
            n.op_count = 1;
            p->root_node[ri] = B.intern(n, &r);
        }
    }
    uint32_t maxl = 0;
    for (const CNode &n : p->nodes) maxl = std::max(maxl, n.level);
    p->n_levels = p->nodes.empty() ? 0 : maxl + 1;
    // B(h): bytes of the root's sub-DAG (each node once) + fused coverage (8W + 32)
    p->root_bytes.resize(n_roots);
    p->stamp.assign(p->nodes.size(), 0);
    std::vector<uint32_t> st;
    for (uint32_t ri = 0; ri < n_roots; ++ri) {
        const uint32_t gen = ++p->stamp_gen;
        double b = 8.0 * kb->W + 32;
        st.assign(1, p->root_node[ri]);
        p->stamp[p->root_node[ri]] = gen;
        while (!st.empty()) {
            const uint32_t id = st.back();
            st.pop_back();
            const CNode &n = p->nodes[id];
            b += n.bytes;
            for (uint32_t q = 0; q < n.op_count; ++q) {
                const uint32_t o = p->ops[n.op_begin + q];
                if (ref_type(o) == RT_NODE && p->stamp[ref_id(o)] != gen) {
                    p->stamp[ref_id(o)] = gen;
                    st.push_back(ref_id(o));
                }
            }
        }
        p->root_bytes[ri] = b;
    }
    *out = p;
    return HEDL_OK;
}

extern "C" hedl_status hedl_program_get_info(const hedl_program *p, hedl_program_info *out) {
    if (!p || !out) return fail(HEDL_ERR_INVALID_ARG, "null program/out");
    std::memset(out, 0, sizeof(*out));
    out->n_roots = (uint32_t)p->root_node.size();
    out->n_nodes = (uint32_t)p->nodes.size();
    out->n_levels = p->n_levels;
    for (const CNode &n : p->nodes) {
        if (n.kind == NK_AND || n.kind == NK_OR) out->n_bool++;
        else if (n.kind == NK_RESTRICT) out->n_restrict++;
        else out->n_drange++;
        out->alg_bytes_shared += n.bytes;
    }
    for (double b : p->root_bytes) out->alg_bytes_total += b;
    return HEDL_OK;
}

extern "C" hedl_status hedl_program_root_bytes(const hedl_program *p, uint32_t first, uint32_t n, double *out) {
    if (!p || (n && !out)) return fail(HEDL_ERR_INVALID_ARG, "null program/out");
    if ((uint64_t)first + n > p->root_bytes.size()) return fail(HEDL_ERR_OUT_OF_RANGE, "root range");
    std::copy(p->root_bytes.begin() + first, p->root_bytes.begin() + first + n, out);
    return HEDL_OK;
}
