// hedl_compile_text: the s-expression front end of SPEC.md:347-355 ("Hypothesis grammar"),
// extended as SURVEY 8(b) states -- (NOT e) for any e (reading Q1), TOP / BOTTOM, empty
// AND / OR (= TOP / BOTTOM), (DRANGE d lo hi) closed float32 intervals
// (reading Q9) and nested (INV r).  The text becomes the hedl_node arrays of
// include/hedl.h (post-order: children before parents) and goes through hedl_compile_ex;
// only the parsing lives here.
//
//   expr    := NAME | TOP | BOTTOM
//            | "(" ("AND"|"OR") expr* ")" | "(" "NOT" expr ")"
//            | "(" ("SOME"|"ONLY") role expr ")"
//            | "(" ("MIN"|"EXACTLY"|"MAX") INT role expr ")"
//            | "(" "DSOME" NUMROLE (">="|"=="|"<=") DECIMAL ")"     (Q9)
//            | "(" "DRANGE" NUMROLE DECIMAL DECIMAL ")"
//            | "(" "SSOME" STRROLE ("EQUAL"|"CONTAIN") STRING ")"
//   role    := NAME | "(" "INV" role ")"
//
// DECIMAL is converted with strtof (round to nearest even, reading Q8); "inf" / "-inf" are
// accepted.  STRING is a double-quoted literal, backslash escapes the next byte.
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

using namespace hedl;

namespace {

struct ParseError {
    size_t pos;
    std::string msg;
};

struct Tok {
    enum Kind { LP, RP, ATOM, STR, END } kind;
    size_t pos;
    std::string text;
};

class Lexer {
  public:
    explicit Lexer(const char *s) : s_(s), n_(std::strlen(s)) {}
    Tok next() {
        while (i_ < n_ && std::isspace((unsigned char)s_[i_])) ++i_;
        if (i_ >= n_) return {Tok::END, i_, ""};
        const size_t p = i_;
        if (s_[i_] == '(') { ++i_; return {Tok::LP, p, "("}; }
        if (s_[i_] == ')') { ++i_; return {Tok::RP, p, ")"}; }
        if (s_[i_] == '"') {
            std::string v;
            for (++i_;; ++i_) {
                if (i_ >= n_) throw ParseError{p, "unterminated string literal"};
                if (s_[i_] == '\\') {
                    if (++i_ >= n_) throw ParseError{p, "unterminated string literal"};
                    v.push_back(s_[i_]);
                } else if (s_[i_] == '"') {
                    ++i_;
                    break;
                } else {
                    v.push_back(s_[i_]);
                }
            }
            return {Tok::STR, p, v};
        }
        while (i_ < n_ && !std::isspace((unsigned char)s_[i_]) && s_[i_] != '(' && s_[i_] != ')' && s_[i_] != '"') ++i_;
        return {Tok::ATOM, p, std::string(s_ + p, i_ - p)};
    }

  private:
    const char *s_;
    size_t n_, i_ = 0;
};

// name -> id for one kind of entity; without a name list the ids are spelled <prefix><id>
class Names {
  public:
    Names(uint32_t n, const char *const *list, char prefix, uint32_t count, const char *what)
        : prefix_(prefix), count_(count), what_(what) {
        if (list)
            for (uint32_t i = 0; i < n; ++i)
                if (list[i]) map_.emplace(list[i], i);
        named_ = list != nullptr;
    }
    uint32_t get(const Tok &t) const {
        if (named_) {
            auto it = map_.find(t.text);
            if (it == map_.end()) throw ParseError{t.pos, std::string("unknown ") + what_ + " '" + t.text + "'"};
            return it->second;
        }
        if (t.text.size() >= 2 && t.text[0] == prefix_) {
            char *end = nullptr;
            errno = 0;
            const unsigned long long v = std::strtoull(t.text.c_str() + 1, &end, 10);
            if (!errno && end && !*end && std::isdigit((unsigned char)t.text[1]) && v < count_) return (uint32_t)v;
        }
        throw ParseError{t.pos, std::string("unknown ") + what_ + " '" + t.text + "' (expected " + prefix_ + "<id>, id < " +
                                    std::to_string(count_) + ")"};
    }

  private:
    std::unordered_map<std::string, uint32_t> map_;
    char prefix_;
    uint32_t count_;
    const char *what_;
    bool named_ = false;
};

struct Builder {
    std::vector<hedl_node> nodes;
    std::vector<uint32_t> kids;
    std::vector<std::string> patterns;
    std::unordered_map<std::string, uint32_t> pat_id;

    uint32_t add(uint8_t op, uint8_t flags, uint32_t arg, uint32_t n, float lo, float hi, const std::vector<uint32_t> &ch) {
        hedl_node d{};
        d.op = op;
        d.flags = flags;
        d.arg = arg;
        d.n = n;
        d.lo = lo;
        d.hi = hi;
        d.child_begin = (uint32_t)kids.size();
        d.child_count = (uint32_t)ch.size();
        kids.insert(kids.end(), ch.begin(), ch.end());
        nodes.push_back(d);
        return (uint32_t)nodes.size() - 1;
    }
    uint32_t pattern(const std::string &v) {
        auto it = pat_id.find(v);
        if (it != pat_id.end()) return it->second;
        patterns.push_back(v);
        pat_id.emplace(v, (uint32_t)patterns.size() - 1);
        return (uint32_t)patterns.size() - 1;
    }
};

class Parser {
  public:
    Parser(const char *text, const Names &c, const Names &r, const Names &d, const Names &s, Builder &b)
        : lex_(text), c_(c), r_(r), d_(d), s_(s), b_(b) {
        tok_ = lex_.next();
    }
    uint32_t hypothesis() {
        const uint32_t id = expr();
        if (tok_.kind != Tok::END) throw ParseError{tok_.pos, "trailing input after the hypothesis"};
        return id;
    }

  private:
    Tok take() {
        Tok t = tok_;
        tok_ = lex_.next();
        return t;
    }
    void expect(Tok::Kind k, const char *what) {
        if (tok_.kind != k) throw ParseError{tok_.pos, std::string("expected ") + what};
        take();
    }
    Tok keyword() {
        if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a constructor keyword"};
        return take();
    }
    // role := NAME | "(" "INV" role ")"; (r^-)^- = r (reading Q12)
    std::pair<uint32_t, bool> role() {
        if (tok_.kind == Tok::LP) {
            take();
            Tok k = keyword();
            if (k.text != "INV") throw ParseError{k.pos, "expected INV"};
            auto r = role();
            expect(Tok::RP, "')'");
            return {r.first, !r.second};
        }
        if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a role name"};
        return {r_.get(take()), false};
    }
    float decimal() {
        if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a number"};
        Tok t = take();
        char *end = nullptr;
        errno = 0;
        const float v = std::strtof(t.text.c_str(), &end);
        if (!end || *end || end == t.text.c_str()) throw ParseError{t.pos, "malformed number '" + t.text + "'"};
        return v;                           // a NaN bound is rejected by the compiler (BAD_EXPR)
    }
    uint32_t cardinality() {
        if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a cardinality"};
        Tok t = take();
        if (!t.text.empty() && t.text[0] == '-') throw ParseError{t.pos, "negative cardinality"};
        char *end = nullptr;
        errno = 0;
        const unsigned long long v = std::strtoull(t.text.c_str(), &end, 10);
        if (t.text.empty() || !std::isdigit((unsigned char)t.text[0]) || !end || *end)
            throw ParseError{t.pos, "malformed cardinality '" + t.text + "'"};
        if (errno || v > 0xffffffffull) throw ParseError{t.pos, "cardinality out of range"};
        return (uint32_t)v;
    }
    uint32_t expr() {
        if (tok_.kind == Tok::ATOM) {
            Tok t = take();
            if (t.text == "TOP") return b_.add(HEDL_OP_TOP, 0, 0, 0, 0, 0, {});
            if (t.text == "BOTTOM") return b_.add(HEDL_OP_BOTTOM, 0, 0, 0, 0, 0, {});
            return b_.add(HEDL_OP_ATOM, 0, c_.get(t), 0, 0, 0, {});
        }
        if (tok_.kind != Tok::LP) throw ParseError{tok_.pos, tok_.kind == Tok::END ? "unexpected end of hypothesis"
                                                                                 : "expected a concept or '('"};
        take();
        const Tok k = keyword();
        uint32_t id;
        if (k.text == "AND" || k.text == "OR") {
            std::vector<uint32_t> ch;
            while (tok_.kind != Tok::RP) {
                if (tok_.kind == Tok::END) throw ParseError{tok_.pos, "unexpected end of hypothesis"};
                ch.push_back(expr());
            }
            id = b_.add(k.text == "AND" ? HEDL_OP_AND : HEDL_OP_OR, 0, 0, 0, 0, 0, ch);
        } else if (k.text == "NOT") {
            const uint32_t c = expr();
            id = b_.add(HEDL_OP_NOT, 0, 0, 0, 0, 0, {c});
        } else if (k.text == "SOME" || k.text == "ONLY") {
            const auto r = role();
            const uint32_t c = expr();
            id = b_.add(k.text == "SOME" ? HEDL_OP_EXISTS : HEDL_OP_FORALL, r.second ? HEDL_FLAG_INV : 0, r.first, 0, 0, 0,
                        {c});
        } else if (k.text == "MIN" || k.text == "EXACTLY" || k.text == "MAX") {
            const uint32_t n = cardinality();
            const auto r = role();
            const uint32_t c = expr();
            const uint8_t op = k.text == "MIN" ? HEDL_OP_MIN : k.text == "MAX" ? HEDL_OP_MAX : HEDL_OP_EXACT;
            id = b_.add(op, r.second ? HEDL_FLAG_INV : 0, r.first, n, 0, 0, {c});
        } else if (k.text == "DSOME") {
            if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a numeric role"};
            const uint32_t d = d_.get(take());
            if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected >=, == or <="};
            const Tok cmp = take();
            const float v = decimal();
            float lo, hi;                   // reading Q9: >=v = [v,+inf], ==v = [v,v], <=v = [-inf,v]
            if (cmp.text == ">=") { lo = v; hi = INFINITY; }
            else if (cmp.text == "==") { lo = v; hi = v; }
            else if (cmp.text == "<=") { lo = -INFINITY; hi = v; }
            else throw ParseError{cmp.pos, "expected >=, == or <="};
            id = b_.add(HEDL_OP_DRANGE, 0, d, 0, lo, hi, {});
        } else if (k.text == "DRANGE") {
            if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a numeric role"};
            const uint32_t d = d_.get(take());
            const float lo = decimal();
            const float hi = decimal();
            id = b_.add(HEDL_OP_DRANGE, 0, d, 0, lo, hi, {});
        } else if (k.text == "SSOME") {
            if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected a string role"};
            const uint32_t s = s_.get(take());
            if (tok_.kind != Tok::ATOM) throw ParseError{tok_.pos, "expected EQUAL or CONTAIN"};
            const Tok mode = take();
            if (mode.text != "EQUAL" && mode.text != "CONTAIN") throw ParseError{mode.pos, "expected EQUAL or CONTAIN"};
            if (tok_.kind != Tok::STR) throw ParseError{tok_.pos, "expected a string literal"};
            const uint32_t pid = b_.pattern(take().text);
            id = b_.add(mode.text == "EQUAL" ? HEDL_OP_SEQUAL : HEDL_OP_SCONTAIN, 0, s, pid, 0, 0, {});
        } else {
            throw ParseError{k.pos, "unknown constructor '" + k.text + "'"};
        }
        expect(Tok::RP, "')'");
        return id;
    }

    Lexer lex_;
    Tok tok_;
    const Names &c_, &r_, &d_, &s_;
    Builder &b_;
};

}  // namespace

extern "C" hedl_status hedl_compile_text(const hedl_kb *kb, const hedl_names *names, const char *const *exprs,
                                         uint32_t n_exprs, uint32_t flags, hedl_program **out, uint32_t *err_index,
                                         uint32_t *err_pos) {
    if (!kb || !out) return fail(HEDL_ERR_INVALID_ARG, "null kb/out");
    *out = nullptr;
    if (n_exprs && !exprs) return fail(HEDL_ERR_INVALID_ARG, "null expression array");
    if (flags & HEDL_COMPILE_HOST_INPUT) return fail(HEDL_ERR_INVALID_ARG, "HOST_INPUT is a hedl_compile_device flag");
    const hedl_names none{};
    const hedl_names &nm = names ? *names : none;
    const Names cn(nm.n_concepts, nm.concepts, 'c', kb->C, "concept");
    const Names rn(nm.n_roles, nm.roles, 'r', kb->R, "role");
    const Names dn(nm.n_data, nm.data, 'd', kb->D, "data property");
    const Names sn(nm.n_strings, nm.strings, 's', kb->S, "string role");
    Builder b;
    std::vector<uint32_t> roots(n_exprs);
    for (uint32_t i = 0; i < n_exprs; ++i) {
        if (!exprs[i]) {
            if (err_index) *err_index = i;
            if (err_pos) *err_pos = 0;
            return fail(HEDL_ERR_INVALID_ARG, "hypothesis " + std::to_string(i) + " is null");
        }
        try {
            Parser ps(exprs[i], cn, rn, dn, sn, b);
            roots[i] = ps.hypothesis();
        } catch (const ParseError &e) {
            if (err_index) *err_index = i;
            if (err_pos) *err_pos = (uint32_t)e.pos;
            return fail(HEDL_ERR_PARSE, "hypothesis " + std::to_string(i) + ", byte " + std::to_string(e.pos) + ": " + e.msg);
        } catch (const std::bad_alloc &) {
            return fail(HEDL_ERR_OOM, "out of host memory while parsing");
        }
    }
    if (b.nodes.size() >= (1ull << 32)) return fail(HEDL_ERR_INVALID_ARG, "too many nodes");
    std::vector<uint64_t> pat_off(b.patterns.size() + 1, 0);
    std::string blob;
    for (size_t q = 0; q < b.patterns.size(); ++q) {
        blob += b.patterns[q];
        pat_off[q + 1] = blob.size();
    }
    return hedl_compile_ex(kb, b.nodes.data(), (uint32_t)b.nodes.size(), b.kids.data(), b.kids.size(), roots.data(),
                           n_exprs, flags, (uint32_t)b.patterns.size(), pat_off.data(), (const uint8_t *)blob.data(), out);
}
