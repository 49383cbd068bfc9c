// hedl_compile: hypothesis node arrays -> canonical DAG program.
//
// Paper: a hypothesis is a flat array of DL operations (§IV);
// an evaluation plan fixes the order of operations and their inputs
// (PAPER.md:532).  Here the plan is a hash-consed DAG shared by all roots
// (common-subexpression reuse), with topological levels for level-synchronous
// batched launches and the per-node algorithmic byte model of SURVEY 8(d).
//
// Plans are generated in parallel on host threads, as in the paper (PAPER.md:578
// "Using CPU multithreading, HT-HEDL first generates evaluation plans ... in
// parallel"): the roots are cut into contiguous shards canonicalised
// independently, then merged level by level into one DAG through a lock-free
// hash-consing table, so CSE stays global across the whole batch.
//
// Canonicalisation (default): complement folded into operand
// references (the paper's per-operand isNegated XOR flag, Alg. 1-2),
// so NOT NOT C == C; n-ary AND/OR flattened, operands sorted and deduplicated
// (an n-ary operation is one step).  No algebraic rewrites.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <thread>

#include "internal.h"

using namespace hedl;

namespace {

constexpr uint8_t NK_DEAD = 0xff;     // a node id reserved by a thread that lost an insert race

inline uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}

uint64_t hash_node(const CNode &n, const uint32_t *ops) {
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

bool same_node(const CNode &a, const uint32_t *aops, const CNode &b, const uint32_t *bops) {
    if (a.kind != b.kind || a.pred != b.pred || a.dir != b.dir || a.n != b.n || a.op_count != b.op_count) return false;
    if (std::memcmp(&a.lo, &b.lo, 4) || std::memcmp(&a.hi, &b.hi, 4)) return false;
    return std::equal(aops, aops + a.op_count, bops);
}

double node_bytes(const hedl_kb *kb, const CNode &n) {
    const double W4b = 4.0 * kb->W;
    if (n.kind == NK_AND || n.kind == NK_OR) return (n.op_count + 1) * W4b;
    if (n.kind == NK_RESTRICT) return kb->dir_bytes[n.dir] + 2 * W4b;
    if (n.kind == NK_STRING) {     // pairs CSR (+ the role's interned values for CONTAIN) + output
        const hedl_sdir &sd = kb->sdirs[n.dir];
        return kb->str_bytes[n.dir] + (n.pred == SM_CONTAIN ? sd.dict_bytes + 8.0 * (sd.V + 1) : 0.0) + W4b;
    }
    return kb->data_bytes[n.dir] + W4b;
}

// ---- single-threaded DAG of one shard ---------------------------------------------
struct LocalDag {
    std::vector<CNode, NoInitAlloc<CNode>> nodes;
    std::vector<uint32_t, NoInitAlloc<uint32_t>> ops;
    std::vector<uint8_t> rootonly;  // created for a root and kept out of the CSE table
    std::vector<uint32_t> table;   // open addressing: node id + 1, 0 = empty
    uint64_t mask = 0, inserted = 0;
    bool cse = true;

    void grow() {
        const uint64_t cap = table.empty() ? 1024 : table.size() * 2;
        std::vector<uint32_t> t(cap, 0);
        const uint64_t m = cap - 1;
        for (uint32_t id = 0; id < nodes.size(); ++id) {
            if (rootonly[id]) continue;
            uint64_t h = hash_node(nodes[id], ops.data() + nodes[id].op_begin) & m;
            while (t[h]) h = (h + 1) & m;
            t[h] = id + 1;
        }
        table.swap(t);
        mask = m;
    }
    // nocse: a root's own conjunction/disjunction -- almost never shared and cheap on the
    // GPU (example-projected), so it skips the table here and in the global merge
    uint32_t intern(CNode n, const uint32_t *o, bool nocse = false) {
        uint64_t h = 0;
        const bool use = cse && !nocse;
        if (use) {
            if ((inserted + 1) * 2 > table.size()) grow();
            h = hash_node(n, o) & mask;
            while (table[h]) {
                const uint32_t id = table[h] - 1;
                if (same_node(nodes[id], ops.data() + nodes[id].op_begin, n, o)) return id;
                h = (h + 1) & mask;
            }
        }
        n.op_begin = (uint32_t)ops.size();
        ops.insert(ops.end(), o, o + n.op_count);
        uint32_t lvl = 0;
        bool has_node = false;
        for (uint32_t i = 0; i < n.op_count; ++i)
            if (ref_type(o[i]) == RT_NODE) {
                has_node = true;
                lvl = std::max(lvl, nodes[ref_id(o[i])].level);
            }
        n.level = has_node ? lvl + 1 : 0;
        const uint32_t id = (uint32_t)nodes.size();
        nodes.push_back(n);
        rootonly.push_back(!use);
        if (use) { table[h] = id + 1; ++inserted; }
        return id;
    }
};

// memo over hypothesis-node ids: id -> (canonical ref, DFS state)
struct Memo {
    std::vector<uint32_t> keys, vals;
    std::vector<uint8_t> st;
    uint64_t mask = 0, used = 0;
    explicit Memo(uint64_t expect) {
        uint64_t cap = 1024;
        while (cap < expect * 2) cap <<= 1;
        keys.assign(cap, 0xffffffffu);
        vals.assign(cap, 0);
        st.assign(cap, 0);
        mask = cap - 1;
    }
    static uint64_t h(uint32_t k) { return (uint64_t)k * 0x9E3779B97F4A7C15ull >> 20; }
    uint64_t slot(uint32_t k) {
        uint64_t i = h(k) & mask;
        while (keys[i] != 0xffffffffu && keys[i] != k) i = (i + 1) & mask;
        return i;
    }
    uint8_t state(uint32_t k) {
        const uint64_t i = slot(k);
        return keys[i] == k ? st[i] : 0;
    }
    void set(uint32_t k, uint8_t s, uint32_t v) {
        if ((used + 1) * 2 > keys.size()) rehash();
        const uint64_t i = slot(k);
        if (keys[i] != k) { keys[i] = k; ++used; }
        st[i] = s;
        vals[i] = v;
    }
    uint32_t val(uint32_t k) { return vals[slot(k)]; }
    void rehash() {
        std::vector<uint32_t> ok, ov;
        std::vector<uint8_t> os;
        ok.swap(keys); ov.swap(vals); os.swap(st);
        keys.assign(ok.size() * 2, 0xffffffffu);
        vals.assign(ok.size() * 2, 0);
        st.assign(ok.size() * 2, 0);
        mask = keys.size() - 1;
        for (size_t i = 0; i < ok.size(); ++i)
            if (ok[i] != 0xffffffffu) {
                uint64_t j = h(ok[i]) & mask;
                while (keys[j] != 0xffffffffu) j = (j + 1) & mask;
                keys[j] = ok[i]; vals[j] = ov[i]; st[j] = os[i];
            }
    }
};

// dense window over the ids a shard mostly touches (post-order flattened trees keep a
// root's nodes just below it), with the hash memo for everything else
struct WinMemo {
    uint32_t lo = 0, hi = 0;
    std::vector<uint32_t> vals;
    std::vector<uint8_t> st;
    Memo far;
    WinMemo(uint32_t lo_, uint32_t hi_, uint64_t expect) : lo(lo_), hi(hi_), far(expect / 16 + 64) {
        vals.assign((size_t)(hi - lo) + 1, 0);
        st.assign((size_t)(hi - lo) + 1, 0);
    }
    bool in(uint32_t k) const { return k >= lo && k <= hi; }
    uint8_t state(uint32_t k) { return in(k) ? st[k - lo] : far.state(k); }
    void set(uint32_t k, uint8_t s, uint32_t v) {
        if (in(k)) { st[k - lo] = s; vals[k - lo] = v; }
        else far.set(k, s, v);
    }
    uint32_t val(uint32_t k) { return in(k) ? vals[k - lo] : far.val(k); }
};

struct Shard {
    LocalDag dag;
    std::vector<uint32_t> root_ref;   // canonical (local) reference of each root of the shard
    hedl_status err = HEDL_OK;
    std::string msg;
};

struct Input {
    const hedl_kb *kb;
    const hedl_node *nodes;
    uint32_t n_nodes;
    const uint32_t *child_idx;
    uint64_t n_child_idx;
    const uint32_t *roots;
    uint32_t n_roots;
    uint32_t flags;
    uint32_t n_pat;                       // string-pattern table (hedl_compile_ex)
    const uint64_t *pat_off;
    const uint8_t *pat_bytes;
    const std::vector<uint32_t> *pat_canon;   // pattern id -> program pattern id (CONTAIN), or ~0
};

// canonicalise roots [r0, r1) into sh.dag (iterative post-order DFS, cycle check)
void canon_shard(const Input &in, uint32_t r0, uint32_t r1, Shard &sh) {
    const hedl_kb *kb = in.kb;
    const bool rewrite = !(in.flags & HEDL_COMPILE_NO_REWRITE);
    const bool compat = in.flags & HEDL_COMPILE_COMPAT_PAPER_MAX;
    LocalDag &D = sh.dag;
    D.cse = !(in.flags & HEDL_COMPILE_NO_CSE);
    const uint64_t expect = (uint64_t)in.n_nodes * (r1 - r0) / std::max<uint32_t>(1, in.n_roots) + 64;
    D.nodes.reserve(expect / 3 + 16);
    D.ops.reserve(expect / 2 + 16);
    uint32_t rmin = 0xffffffffu, rmax = 0;
    for (uint32_t ri = r0; ri < r1; ++ri) {
        rmin = std::min(rmin, in.roots[ri]);
        rmax = std::max(rmax, in.roots[ri]);
    }
    const uint64_t per_root = (uint64_t)in.n_nodes / std::max<uint32_t>(1, in.n_roots) + 16;
    const uint32_t wlo = rmin == 0xffffffffu ? 0 : (uint32_t)(rmin > 4 * per_root ? rmin - 4 * per_root : 0);
    const uint32_t whi = rmin == 0xffffffffu ? 0 : std::min<uint32_t>(rmax, in.n_nodes ? in.n_nodes - 1 : 0);
    const bool dense_ok = (uint64_t)whi - wlo <= 8 * expect + (1u << 16);   // else the window is not worth it
    WinMemo memo(wlo, dense_ok ? whi : wlo, expect);
    std::vector<std::pair<uint32_t, uint32_t>> stack;
    std::vector<uint32_t> tmp;
    sh.root_ref.resize(r1 - r0);
    auto bad = [&](hedl_status st, uint32_t i, const std::string &m) {
        sh.err = st;
        sh.msg = "node " + std::to_string(i) + ": " + m;
    };
    for (uint32_t ri = r0; ri < r1; ++ri) {
        const uint32_t root = in.roots[ri];
        if (root >= in.n_nodes) { sh.err = HEDL_ERR_OUT_OF_RANGE; sh.msg = "root " + std::to_string(ri) + " out of range"; return; }
        if (memo.state(root) != 2) {
            stack.clear();
            stack.push_back({root, 0});
            memo.set(root, 1, 0);
            while (!stack.empty()) {
                const uint32_t i = stack.back().first;
                const hedl_node &nd = in.nodes[i];
                if ((uint64_t)nd.child_begin + nd.child_count > in.n_child_idx)
                    return bad(HEDL_ERR_OUT_OF_RANGE, i, "child range out of bounds");
                uint32_t &k = stack.back().second;
                if (k < nd.child_count) {
                    const uint32_t c = in.child_idx[nd.child_begin + k++];
                    if (c >= in.n_nodes) return bad(HEDL_ERR_OUT_OF_RANGE, i, "child id out of range");
                    const uint8_t cs = memo.state(c);
                    if (cs == 1) return bad(HEDL_ERR_BAD_EXPR, i, "cycle");
                    if (cs == 0) { memo.set(c, 1, 0); stack.push_back({c, 0}); }
                    continue;
                }
                // all children are done: build the canonical reference of node i
                const bool at_root = stack.size() == 1;      // the hypothesis' own node
                const uint32_t *ch = in.child_idx + nd.child_begin;
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
                    r = memo.val(ch[0]) ^ 1u;   // complement over Delta (Q1); NOT NOT C == C
                    break;
                case HEDL_OP_AND:
                case HEDL_OP_OR: {
                    const uint8_t kind = nd.op == HEDL_OP_AND ? NK_AND : NK_OR;
                    tmp.clear();
                    for (uint32_t j = 0; j < cc; ++j) {
                        const uint32_t cr = memo.val(ch[j]);
                        if (rewrite && ref_type(cr) == RT_NODE && !ref_comp(cr) && D.nodes[ref_id(cr)].kind == kind) {
                            const CNode &sub = D.nodes[ref_id(cr)];
                            for (uint32_t q = 0; q < sub.op_count; ++q) tmp.push_back(D.ops[sub.op_begin + q]);
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
                        r = mkref(RT_NODE, D.intern(n, tmp.data(), at_root), 0);
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
                    uint32_t child = memo.val(ch[0]);
                    switch (nd.op) {
                    case HEDL_OP_EXISTS: n.pred = P_GE; n.n = 1; n.sat = 1; break;           // Alg. 4
                    case HEDL_OP_FORALL: n.pred = P_LE; n.n = 0; n.sat = 1; child ^= 1u; break; // Alg. 6
                    case HEDL_OP_MIN: n.pred = P_GE; n.n = nd.n; n.sat = nd.n; break;        // Alg. 7 MIN
                    case HEDL_OP_MAX: n.pred = compat ? P_LEP : P_LE; n.n = nd.n; n.sat = nd.n + 1; break;
                    default: n.pred = P_EQ; n.n = nd.n; n.sat = nd.n + 1; break;             // EXACTLY
                    }
                    r = mkref(RT_NODE, D.intern(n, &child), 0);        // restrictions are always shared
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
                    r = mkref(RT_NODE, D.intern(n, nullptr), 0);
                    break;
                }
                case HEDL_OP_SEQUAL:
                case HEDL_OP_SCONTAIN: {
                    if (cc) return bad(HEDL_ERR_BAD_EXPR, i, "string restriction takes no children");
                    if (nd.arg >= kb->S) return bad(HEDL_ERR_OUT_OF_RANGE, i, "string role id out of range");
                    if (nd.n >= in.n_pat) return bad(HEDL_ERR_OUT_OF_RANGE, i, "pattern id out of range");
                    const uint64_t a = in.pat_off[nd.n], b = in.pat_off[nd.n + 1];
                    CNode n{};
                    n.kind = NK_STRING;
                    n.dir = (uint16_t)nd.arg;
                    if (nd.op == HEDL_OP_SEQUAL) {
                        // interned-id compare; an absent value short-circuits to BOTTOM
                        const auto &ids = kb->sdirs[nd.arg].ids;
                        auto it = ids.find(std::string((const char *)in.pat_bytes + a, (const char *)in.pat_bytes + b));
                        if (it == ids.end()) { r = mkref(RT_TOP, 0, 1); break; }
                        n.pred = SM_EQUAL;
                        n.n = it->second;
                    } else {
                        if (a == b) return bad(HEDL_ERR_BAD_EXPR, i, "empty CONTAIN pattern");
                        n.pred = SM_CONTAIN;
                        n.n = (*in.pat_canon)[nd.n];
                    }
                    r = mkref(RT_NODE, D.intern(n, nullptr), 0);
                    break;
                }
                default:
                    return bad(HEDL_ERR_BAD_EXPR, i, "unknown opcode");
                }
                memo.set(i, 2, r);
                stack.pop_back();
            }
        }
        sh.root_ref[ri - r0] = memo.val(root);
    }
}

// ---- lock-free global DAG (level-synchronous merge of the shards) -------------------
struct Global {
    hedl_program *p;
    const hedl_kb *kb;
    bool cse;
    struct FreeDel { void operator()(std::atomic<uint32_t> *q) const { std::free(q); } };
    std::unique_ptr<std::atomic<uint32_t>, FreeDel> table;
    uint64_t mask = 0;
    std::atomic<uint32_t> n_count{0};
    std::atomic<uint64_t> ops_count{0};
    static constexpr uint32_t kNodeBlock = 4096, kOpsBlock = 16384;

    // per-thread allocation cursor: ids and operand slots come in private blocks, so
    // threads neither contend on the counters nor false-share node cache lines
    struct Cursor {
        uint32_t next = 0, end = 0;
        uint64_t onext = 0, oend = 0;
    };

    uint32_t intern(CNode n, const uint32_t *o, Cursor &cur, bool nocse = false) {
        uint32_t mine = 0xffffffffu;
        auto materialise = [&]() {
            if (cur.next == cur.end) {
                cur.next = n_count.fetch_add(kNodeBlock, std::memory_order_relaxed);
                cur.end = cur.next + kNodeBlock;
            }
            mine = cur.next++;
            uint64_t ob;
            if (n.op_count > kOpsBlock) {
                ob = ops_count.fetch_add(n.op_count, std::memory_order_relaxed);
            } else {
                if (cur.onext + n.op_count > cur.oend) {
                    cur.onext = ops_count.fetch_add(kOpsBlock, std::memory_order_relaxed);
                    cur.oend = cur.onext + kOpsBlock;
                }
                ob = cur.onext;
                cur.onext += n.op_count;
            }
            std::copy(o, o + n.op_count, p->ops.begin() + ob);
            n.op_begin = (uint32_t)ob;
            uint32_t lvl = 0;
            bool has_node = false;
            for (uint32_t i = 0; i < n.op_count; ++i)
                if (ref_type(o[i]) == RT_NODE) {
                    has_node = true;
                    lvl = std::max(lvl, p->nodes[ref_id(o[i])].level);
                }
            n.level = has_node ? lvl + 1 : 0;
            n.bytes = node_bytes(kb, n);
            p->nodes[mine] = n;
        };
        if (!cse || nocse) {
            materialise();
            return mine;
        }
        uint64_t h = hash_node(n, o) & mask;
        for (;;) {
            uint32_t v = table.get()[h].load(std::memory_order_acquire);
            if (v == 0) {
                if (mine == 0xffffffffu) materialise();
                uint32_t expected = 0;
                if (table.get()[h].compare_exchange_strong(expected, mine + 1, std::memory_order_acq_rel,
                                                     std::memory_order_acquire))
                    return mine;
                v = expected;
            }
            const uint32_t id = v - 1;
            const CNode &c = p->nodes[id];
            if (same_node(c, p->ops.data() + c.op_begin, n, o)) {
                if (mine != 0xffffffffu) p->nodes[mine].kind = NK_DEAD;   // lost the race: a hole
                return id;
            }
            h = (h + 1) & mask;
        }
    }
};

template <class F>
void run_threads(unsigned n, F f) {
    if (n <= 1) { f(0u); return; }
    std::vector<std::thread> th;
    th.reserve(n);
    for (unsigned t = 0; t < n; ++t) th.emplace_back(f, t);
    for (auto &x : th) x.join();
}

}  // namespace

extern "C" hedl_status hedl_compile(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                                    const uint32_t *child_idx, uint64_t n_child_idx,
                                    const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                                    hedl_program **out) {
    return hedl_compile_ex(kb, nodes, n_nodes, child_idx, n_child_idx, roots, n_roots, flags, 0, nullptr, nullptr, out);
}

extern "C" hedl_status hedl_compile_ex(const hedl_kb *kb, const hedl_node *nodes, uint32_t n_nodes,
                                       const uint32_t *child_idx, uint64_t n_child_idx,
                                       const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                                       uint32_t n_patterns, const uint64_t *pat_off, const uint8_t *pat_bytes,
                                       hedl_program **out) {
    if (!kb || !out) return fail(HEDL_ERR_INVALID_ARG, "null kb/out");
    *out = nullptr;
    if ((n_nodes && !nodes) || (n_child_idx && !child_idx) || (n_roots && !roots))
        return fail(HEDL_ERR_INVALID_ARG, "null node/child/root array");
    if (n_nodes >= (1u << 28)) return fail(HEDL_ERR_INVALID_ARG, "too many nodes in one program (max 2^28)");
    if (n_patterns && !pat_off) return fail(HEDL_ERR_INVALID_ARG, "null pattern offsets");
    for (uint32_t q = 0; q < n_patterns; ++q)
        if (pat_off[q + 1] < pat_off[q]) return fail(HEDL_ERR_INVALID_ARG, "pattern offsets not ascending");
    if (n_patterns && pat_off[n_patterns] > pat_off[0] && !pat_bytes) return fail(HEDL_ERR_INVALID_ARG, "null pattern bytes");
    const double t0 = now_ms();
    // CONTAIN patterns: deduplicated into the program's own table (equal patterns -> one node)
    std::vector<uint32_t> pat_canon;
    std::vector<std::string> prog_pats;
    if (n_patterns) {
        pat_canon.assign(n_patterns, ~0u);
        std::unordered_map<std::string, uint32_t> seen;
        for (uint32_t i = 0; i < n_nodes; ++i) {
            if (nodes[i].op != HEDL_OP_SCONTAIN || nodes[i].n >= n_patterns || pat_canon[nodes[i].n] != ~0u) continue;
            const uint32_t q = nodes[i].n;
            std::string key((const char *)pat_bytes + pat_off[q], (const char *)pat_bytes + pat_off[q + 1]);
            auto it = seen.find(key);
            if (it == seen.end()) {
                it = seen.emplace(key, (uint32_t)prog_pats.size()).first;
                prog_pats.push_back(std::move(key));
            }
            pat_canon[q] = it->second;
        }
    }
    const Input in{kb, nodes, n_nodes, child_idx, n_child_idx, roots, n_roots, flags,
                   n_patterns, pat_off, pat_bytes, &pat_canon};
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (const char *e = std::getenv("HEDL_COMPILE_THREADS")) hw = std::max(1, std::atoi(e));   // tests / tuning
    const unsigned T = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)hw, 32ull, (uint64_t)n_roots / 4096}));
    std::vector<Shard> sh(T);
    run_threads(T, [&](unsigned t) {
        const uint32_t a = (uint32_t)((uint64_t)n_roots * t / T), b = (uint32_t)((uint64_t)n_roots * (t + 1) / T);
        canon_shard(in, a, b, sh[t]);
    });
    for (unsigned t = 0; t < T; ++t)
        if (sh[t].err) return fail(sh[t].err, sh[t].msg);
    const double t1 = now_ms();

    hedl_program *p = new hedl_program();
    p->kb = kb;
    p->flags = flags;
    p->patterns.swap(prog_pats);
    p->root_node.resize(n_roots);
    if (T == 1) {
        // one shard: its DAG is the program
        Shard &s0 = sh[0];
        p->nodes.swap(s0.dag.nodes);
        p->ops.swap(s0.dag.ops);
        for (CNode &n : p->nodes) n.bytes = node_bytes(kb, n);
        LocalDag &D = s0.dag;
        D.nodes.swap(p->nodes);      // intern below needs the DAG: swap back temporarily
        D.ops.swap(p->ops);
        for (uint32_t ri = 0; ri < n_roots; ++ri) {
            const uint32_t r = s0.root_ref[ri];
            if (ref_type(r) == RT_NODE && !ref_comp(r)) {
                p->root_node[ri] = ref_id(r);
            } else {                 // a 1-operand AND materialises atoms, constants, complements
                CNode n{};
                n.kind = NK_AND;
                n.op_count = 1;
                const uint32_t id = D.intern(n, &r, true);
                D.nodes[id].bytes = node_bytes(kb, D.nodes[id]);
                p->root_node[ri] = id;
            }
        }
        p->nodes.swap(D.nodes);
        p->ops.swap(D.ops);
    } else {
        // level-synchronous merge into one lock-free hash-consed DAG
        uint64_t tot_nodes = n_roots, tot_ops = n_roots;
        uint32_t maxl = 0;
        for (auto &s : sh) {
            tot_nodes += s.dag.nodes.size();
            tot_ops += s.dag.ops.size();
            for (const CNode &n : s.dag.nodes) maxl = std::max(maxl, n.level);
        }
        const double tm0 = now_ms();
        // capacity: every local node + materialised roots + one partly used block per thread and phase
        const uint64_t cap_nodes = tot_nodes + (uint64_t)T * (maxl + 2) * Global::kNodeBlock;
        uint64_t max_ops = 0;
        for (auto &s : sh)
            for (const CNode &n : s.dag.nodes) max_ops = std::max<uint64_t>(max_ops, n.op_count);
        const uint64_t cap_ops = 2 * tot_ops + (uint64_t)T * (maxl + 2) * Global::kOpsBlock + max_ops;
        if (cap_nodes >= (1ull << 29)) { delete p; return fail(HEDL_ERR_INVALID_ARG, "program too large"); }
        p->nodes.resize(cap_nodes);
        p->ops.resize(cap_ops);
        std::vector<Global::Cursor> cursors(T);
        Global G{p, kb, !(flags & HEDL_COMPILE_NO_CSE)};
        if (G.cse) {
            uint64_t cap = 1024;
            while (cap < tot_nodes * 2) cap <<= 1;
            // calloc: zero pages come lazily from the OS (first touch by the merging threads)
            G.table.reset(reinterpret_cast<std::atomic<uint32_t> *>(std::calloc(cap, sizeof(uint32_t))));
            G.mask = cap - 1;
        }
        std::vector<std::vector<uint32_t>> gmap(T);
        std::vector<std::vector<uint32_t>> by_level(T);   // local ids ordered by level
        std::vector<std::vector<uint32_t>> lvl_off(T);
        run_threads(T, [&](unsigned t) {
            const auto &L = sh[t].dag.nodes;
            gmap[t].assign(L.size(), 0);
            std::vector<uint32_t> cnt(maxl + 2, 0);
            for (const CNode &n : L) cnt[n.level + 1]++;
            for (uint32_t l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
            lvl_off[t] = cnt;
            by_level[t].resize(L.size());
            std::vector<uint32_t> pos(cnt.begin(), cnt.end() - 1);
            for (uint32_t i = 0; i < L.size(); ++i) by_level[t][pos[L[i].level]++] = i;
        });
        const bool rewrite = !(flags & HEDL_COMPILE_NO_REWRITE);
        auto remap = [&](unsigned t, uint32_t r) {
            return ref_type(r) == RT_NODE ? mkref(RT_NODE, gmap[t][ref_id(r)], ref_comp(r)) : r;
        };
        const double tm1 = now_ms();
        timing_note("compile: merge setup", tm1 - tm0);
        for (uint32_t l = 0; l <= maxl; ++l) {
            run_threads(T, [&](unsigned t) {
                const LocalDag &D = sh[t].dag;
                std::vector<uint32_t> tmp;
                for (uint32_t k = lvl_off[t][l]; k < lvl_off[t][l + 1]; ++k) {
                    const uint32_t li = by_level[t][k];
                    CNode n = D.nodes[li];
                    tmp.resize(n.op_count);
                    for (uint32_t q = 0; q < n.op_count; ++q) tmp[q] = remap(t, D.ops[n.op_begin + q]);
                    if (rewrite && (n.kind == NK_AND || n.kind == NK_OR)) std::sort(tmp.begin(), tmp.end());
                    gmap[t][li] = G.intern(n, tmp.data(), cursors[t], D.rootonly[li] != 0);
                }
            });
        }
        run_threads(T, [&](unsigned t) {
            const uint32_t a = (uint32_t)((uint64_t)n_roots * t / T);
            for (uint32_t k = 0; k < sh[t].root_ref.size(); ++k) {
                const uint32_t r = remap(t, sh[t].root_ref[k]);
                if (ref_type(r) == RT_NODE && !ref_comp(r)) {
                    p->root_node[a + k] = ref_id(r);
                } else {
                    CNode n{};
                    n.kind = NK_AND;
                    n.op_count = 1;
                    p->root_node[a + k] = G.intern(n, &r, cursors[t], true);
                }
            }
        });
        // ids reserved in a cursor block but never used are holes
        for (const Global::Cursor &c : cursors)
            for (uint32_t i = c.next; i < c.end; ++i) p->nodes[i].kind = NK_DEAD;
        p->nodes.resize(std::min<uint64_t>(G.n_count.load(), cap_nodes));
        p->ops.resize(std::min<uint64_t>(G.ops_count.load(), cap_ops));
        timing_note("compile: merge levels+roots", now_ms() - tm1);
    }
    uint32_t maxl = 0;
    bool any = false;
    for (const CNode &n : p->nodes)
        if (n.kind != NK_DEAD) { maxl = std::max(maxl, n.level); any = true; }
    p->n_levels = any ? maxl + 1 : 0;
    p->stamp.assign(p->nodes.size(), 0);
    const_cast<hedl_kb *>(kb)->refs.fetch_add(1);        // released by hedl_program_free
    timing_note("compile: shards", t1 - t0);
    timing_note("compile: total", now_ms() - t0);
    *out = p;
    return HEDL_OK;
}

// B(h): bytes of the root's sub-DAG (each node once) + fused coverage (8W + 32).
// Computed lazily (only the info/bytes queries need it), so compile stays lean.
static void ensure_root_bytes(hedl_program *p) {
    std::lock_guard<std::mutex> lk(p->mu);
    if (p->dev && dc_download(p)) return;
    if (p->root_bytes.size() == p->root_node.size()) return;
    const hedl_kb *kb = p->kb;
    const uint32_t n_roots = (uint32_t)p->root_node.size();
    p->root_bytes.resize(n_roots);
    if (p->stamp.size() < p->nodes.size()) p->stamp.assign(p->nodes.size(), 0);
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
}

extern "C" hedl_status hedl_program_get_info(const hedl_program *p, hedl_program_info *out) {
    if (!p || !out) return fail(HEDL_ERR_INVALID_ARG, "null program/out");
    ensure_root_bytes(const_cast<hedl_program *>(p));
    std::memset(out, 0, sizeof(*out));
    out->n_roots = (uint32_t)p->root_node.size();
    out->n_nodes = 0;
    out->n_levels = p->n_levels;
    for (const CNode &n : p->nodes) {
        if (n.kind == NK_DEAD) continue;
        out->n_nodes++;
        if (n.kind == NK_AND || n.kind == NK_OR) out->n_bool++;
        else if (n.kind == NK_RESTRICT) out->n_restrict++;
        else if (n.kind == NK_STRING) out->n_string++;
        else out->n_drange++;
        out->alg_bytes_shared += n.bytes;
    }
    for (double b : p->root_bytes) out->alg_bytes_total += b;
    return HEDL_OK;
}

extern "C" hedl_status hedl_program_root_bytes(const hedl_program *p, uint32_t first, uint32_t n, double *out) {
    if (!p || (n && !out)) return fail(HEDL_ERR_INVALID_ARG, "null program/out");
    ensure_root_bytes(const_cast<hedl_program *>(p));
    if ((uint64_t)first + n > p->root_bytes.size()) return fail(HEDL_ERR_OUT_OF_RANGE, "root range");
    std::copy(p->root_bytes.begin() + first, p->root_bytes.begin() + first + n, out);
    return HEDL_OK;
}
