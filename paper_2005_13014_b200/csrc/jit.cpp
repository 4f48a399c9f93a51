// Stencil programs from text: the paper's compiler contribution done
// B200-native on the host, in C++.
//
//   parse     the stencil language of include/oec.h (one `apply` per stencil.apply, accesses at
//             constant offsets = stencil.access P:355, select = loop.if/select P:402, `store` =
//             stencil.store P:366) into an SSA expression DAG per operator;
//   verify    SSA order (an operator reads inputs and EARLIER operators only, so the def-use
//             graph is acyclic), alias-free parameters (an array is loaded or stored,
//             never both), every output stored exactly once, types (conditions only in
//             select / && / || / !);
//   shape     shape inference (§5.2): walk the operators in reverse order; the
//   infer.    iteration domain of an operator is the bounding box of what its consumers read
//             (stores: the domain), an input's access extent is the union of its consumers'
//             domains grown by their access offsets -- "verify the input array is large enough";
//   inline    stencil inlining (§5.1): the generated kernel evaluates every operator at
//             every offset its consumers read it, recursively, so no temporary touches memory;
//             each (operator, offset) instance and each (input, offset) load is emitted once --
//             the common subexpression elimination the paper runs after inlining;
//   unroll    stencil unrolling (§5.1) along j by 2 or 4: one thread evaluates U
//             points; instances shared between them are emitted once (CSE);
//   original  the paper's "original" level: one kernel per operator over its inferred
//             domain, temporaries materialised in a device workspace;
//   codegen   CUDA C++ with the domain size and every stride as compile-time constants ("size
//             specialization for just-in-time compilation", P:338 -- every access becomes a
//             load at an immediate offset from one base register), compiled by NVRTC for
//             sm_100a with -fmad=false (the oracle's operation order, no contraction), loaded
//             through the driver API and cached per specialisation.
//
// Execution model of the generated kernels: the paper's (one thread per point, everything
// inlined, registers only, no synchronisation).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <ctype.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "oec_internal.h"

namespace oec {
namespace jit {

// ---------------------------------------------------------------------------------------------
// IR
// ---------------------------------------------------------------------------------------------
enum Op { LIT, SCALAR, ACC_IN, ACC_TMP, NEG, ADD, SUB, MUL, DIV, LT, GT, LE, GE, EQ, NE, AND, OR, NOT, SELECT,
          MIN, MAX, ABS, SQRT };

struct Node {
    int op = LIT;
    double lit = 0;
    int a = -1, b = -1, c = -1;  // operand node indices (earlier in the same operator)
    int ref = -1;                // SCALAR: scalar index; ACC_IN: input index; ACC_TMP: temp index
    int off[3] = {0, 0, 0};      // access offset
    bool boolean = false;
};

struct Operator {  // one stencil.apply
    std::vector<int> results;  // temp indices it defines
    std::vector<Node> nodes;   // operands precede their users
    std::vector<int> roots;    // one per result
    int line = 0;
    bool live = false;         // some output depends on it
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // iteration domain relative to the domain (shape inference)
};

struct Program {
    std::string name;
    long long uid = 0;  // distinguishes re-registrations in the kernel cache
    std::vector<std::string> in_names;
    std::vector<int> in_kinv;
    std::vector<std::string> sc_names;
    std::vector<double> sc_dflt;
    std::vector<std::string> out_names;
    std::vector<int> out_temp;
    std::vector<std::string> temp_names;
    std::vector<int> temp_op, temp_slot;
    std::vector<Operator> ops;
    std::vector<std::array<int, 3>> in_lo, in_hi;
    std::vector<int> in_used;
    std::vector<int> temp_buffered;  // read by a later live operator (needs a buffer at the original level)
};

struct Error {
    std::string msg;
};

// ---------------------------------------------------------------------------------------------
// lexer
// ---------------------------------------------------------------------------------------------
enum TokKind { T_END, T_NAME, T_NUM, T_PUNCT };
struct Tok {
    int kind = T_END;
    std::string s;
    double num = 0;
    bool integral = false;
    int line = 0, col = 0;
};

static std::vector<Tok> lex(const char *src) {
    std::vector<Tok> out;
    int line = 1, col = 1;
    const char *p = src;
    auto adv = [&](int n) {
        for (int q = 0; q < n; ++q) {
            if (*p == '\n') { ++line; col = 1; } else ++col;
            ++p;
        }
    };
    static const char *two[] = {"->", "<=", ">=", "==", "!=", "&&", "||"};
    while (*p) {
        if (*p == '#') {
            while (*p && *p != '\n') adv(1);
            continue;
        }
        if (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n' || *p == ';') {
            adv(1);
            continue;
        }
        Tok t;
        t.line = line;
        t.col = col;
        if (isalpha((unsigned char)*p) || *p == '_') {
            const char *q = p;
            while (isalnum((unsigned char)*q) || *q == '_') ++q;
            t.kind = T_NAME;
            t.s.assign(p, q - p);
            adv((int)(q - p));
        } else if (isdigit((unsigned char)*p) || (*p == '.' && isdigit((unsigned char)p[1]))) {
            const char *q = p;
            bool integral = true;
            while (isdigit((unsigned char)*q)) ++q;
            if (*q == '.') {
                integral = false;
                ++q;
                while (isdigit((unsigned char)*q)) ++q;
            }
            if (*q == 'e' || *q == 'E') {
                const char *r = q + 1;
                if (*r == '+' || *r == '-') ++r;
                if (isdigit((unsigned char)*r)) {
                    integral = false;
                    q = r;
                    while (isdigit((unsigned char)*q)) ++q;
                }
            }
            t.kind = T_NUM;
            t.s.assign(p, q - p);
            t.num = strtod(t.s.c_str(), nullptr);  // correctly rounded decimal -> binary64
            t.integral = integral;
            adv((int)(q - p));
        } else {
            t.kind = T_PUNCT;
            bool found = false;
            for (const char *tw : two)
                if (p[0] == tw[0] && p[1] == tw[1]) {
                    t.s = tw;
                    adv(2);
                    found = true;
                    break;
                }
            if (!found) {
                if (!strchr("()[]{},=+-*/<>!:", *p)) {
                    char m[96];
                    snprintf(m, sizeof m, "line %d:%d: unexpected character '%c'", line, col, *p);
                    throw Error{m};
                }
                t.s.assign(p, 1);
                adv(1);
            }
        }
        out.push_back(t);
    }
    Tok e;
    e.line = line;
    e.col = col;
    out.push_back(e);
    return out;
}

// ---------------------------------------------------------------------------------------------
// parser + verifier
// ---------------------------------------------------------------------------------------------
static bool reserved(const std::string &s) {
    static const char *kw[] = {"program", "input", "scalar", "output", "apply", "return", "store", "end",
                               "select", "min", "max", "abs", "sqrt", "ij", "ijk"};
    for (const char *k : kw)
        if (s == k) return true;
    return false;
}

struct Parser {
    std::vector<Tok> t;
    size_t pos = 0;
    Program P;
    // symbol kinds
    enum { S_INPUT, S_SCALAR, S_OUTPUT, S_TEMP };
    std::map<std::string, std::pair<int, int>> sym;  // name -> (kind, index)
    // current operator
    Operator *cur = nullptr;
    std::map<std::string, int> locals;

    [[noreturn]] void fail(const Tok &at, const std::string &m) {
        char b[64];
        snprintf(b, sizeof b, "line %d:%d: ", at.line, at.col);
        throw Error{b + m};
    }
    const Tok &peek(int k = 0) { return t[std::min(pos + k, t.size() - 1)]; }
    bool is(const char *s, int k = 0) { return peek(k).kind == T_PUNCT && peek(k).s == s; }
    bool is_kw(const char *s) { return peek().kind == T_NAME && peek().s == s; }
    const Tok &take() { return t[pos < t.size() - 1 ? pos++ : pos]; }
    void expect(const char *s) {
        if (!is(s)) fail(peek(), std::string("expected '") + s + "'" + (peek().kind == T_END ? " before the end" : ", got '" + peek().s + "'"));
        take();
    }
    std::string name(const char *what) {
        if (peek().kind != T_NAME) fail(peek(), std::string("expected ") + what);
        return take().s;
    }
    void declare(const Tok &at, const std::string &n, int kind, int idx) {
        if (reserved(n)) fail(at, "'" + n + "' is a reserved word");
        if (sym.count(n)) fail(at, "'" + n + "' is already defined");
        sym[n] = {kind, idx};
    }
    int signed_int() {
        bool neg = false;
        if (is("-")) {
            take();
            neg = true;
        } else if (is("+")) take();
        const Tok &n = peek();
        if (n.kind != T_NUM || !n.integral || n.num > 64) fail(n, "expected an integer offset in [-64, 64]");
        take();
        return neg ? -(int)n.num : (int)n.num;
    }

    int add(Node n) {
        cur->nodes.push_back(n);
        return (int)cur->nodes.size() - 1;
    }
    void need_num(const Tok &at, int idx, const char *ctx) {
        if (cur->nodes[idx].boolean) fail(at, std::string("a condition cannot be used as a number (") + ctx + ")");
    }
    void need_bool(const Tok &at, int idx, const char *ctx) {
        if (!cur->nodes[idx].boolean) fail(at, std::string("expected a condition (") + ctx + ")");
    }
    int bin(int op, int a, int b, bool boolean) {
        Node n;
        n.op = op;
        n.a = a;
        n.b = b;
        n.boolean = boolean;
        return add(n);
    }

    // expr := or
    int expr() { return p_or(); }
    int p_or() {
        int l = p_and();
        while (is("||")) {
            const Tok &at = take();
            int r = p_and();
            need_bool(at, l, "||");
            need_bool(at, r, "||");
            l = bin(OR, l, r, true);
        }
        return l;
    }
    int p_and() {
        int l = p_cmp();
        while (is("&&")) {
            const Tok &at = take();
            int r = p_cmp();
            need_bool(at, l, "&&");
            need_bool(at, r, "&&");
            l = bin(AND, l, r, true);
        }
        return l;
    }
    int p_cmp() {
        int l = p_add();
        static const std::pair<const char *, int> ops[] = {{"<", LT}, {">", GT}, {"<=", LE}, {">=", GE}, {"==", EQ}, {"!=", NE}};
        for (auto &o : ops)
            if (is(o.first)) {
                const Tok &at = take();
                int r = p_add();
                need_num(at, l, o.first);
                need_num(at, r, o.first);
                return bin(o.second, l, r, true);
            }
        return l;
    }
    int p_add() {
        int l = p_mul();
        while (is("+") || is("-")) {
            const Tok &at = take();
            int r = p_mul();
            need_num(at, l, at.s.c_str());
            need_num(at, r, at.s.c_str());
            l = bin(at.s == "+" ? ADD : SUB, l, r, false);
        }
        return l;
    }
    int p_mul() {
        int l = p_unary();
        while (is("*") || is("/")) {
            const Tok &at = take();
            int r = p_unary();
            need_num(at, l, at.s.c_str());
            need_num(at, r, at.s.c_str());
            l = bin(at.s == "*" ? MUL : DIV, l, r, false);
        }
        return l;
    }
    int p_unary() {
        if (is("-")) {
            const Tok &at = take();
            int a = p_unary();
            need_num(at, a, "unary -");
            Node n;
            n.op = NEG;
            n.a = a;
            return add(n);
        }
        if (is("!")) {
            const Tok &at = take();
            int a = p_unary();
            need_bool(at, a, "!");
            Node n;
            n.op = NOT;
            n.a = a;
            n.boolean = true;
            return add(n);
        }
        return atom();
    }
    int atom() {
        const Tok &at = peek();
        if (at.kind == T_NUM) {
            take();
            Node n;
            n.op = LIT;
            n.lit = at.num;
            return add(n);
        }
        if (is("(")) {
            take();
            int e = expr();
            expect(")");
            return e;
        }
        if (at.kind != T_NAME) fail(at, at.kind == T_END ? "unexpected end of program" : "unexpected '" + at.s + "'");
        std::string nm = take().s;
        if (is("(")) {  // function
            static const std::pair<const char *, int> fns[] = {{"select", 3}, {"min", 2}, {"max", 2}, {"abs", 1}, {"sqrt", 1}};
            int arity = -1;
            for (auto &f : fns)
                if (nm == f.first) arity = f.second;
            if (arity < 0) fail(at, "unknown function '" + nm + "'");
            take();
            std::vector<int> args;
            while (true) {
                args.push_back(expr());
                if (is(",")) {
                    take();
                    continue;
                }
                expect(")");
                break;
            }
            if ((int)args.size() != arity) fail(at, nm + "() takes " + std::to_string(arity) + " arguments");
            Node n;
            if (nm == "select") {
                need_bool(at, args[0], "select condition");
                need_num(at, args[1], "select value");
                need_num(at, args[2], "select value");
                n.op = SELECT;
                n.c = args[0];
                n.a = args[1];
                n.b = args[2];
            } else {
                for (int x : args) need_num(at, x, nm.c_str());
                n.op = nm == "min" ? MIN : nm == "max" ? MAX : nm == "abs" ? ABS : SQRT;
                n.a = args[0];
                if (arity > 1) n.b = args[1];
            }
            return add(n);
        }
        int off[3] = {0, 0, 0};
        bool has_off = false;
        if (is("[")) {
            take();
            for (int d = 0; d < 3; ++d) {
                off[d] = signed_int();
                if (d < 2) expect(",");
            }
            expect("]");
            has_off = true;
        }
        if (!has_off) {
            auto l = locals.find(nm);
            if (l != locals.end()) return l->second;
        }
        auto s = sym.find(nm);
        if (s == sym.end()) fail(at, "'" + nm + "' is not defined (inputs and operators must be declared before use)");
        Node n;
        switch (s->second.first) {
        case S_SCALAR:
            if (has_off) fail(at, "scalar '" + nm + "' cannot be accessed at an offset");
            n.op = SCALAR;
            n.ref = s->second.second;
            return add(n);
        case S_OUTPUT: fail(at, "output '" + nm + "' cannot be read (parameters are loaded or stored, never both, P:381)");
        case S_INPUT: n.op = ACC_IN; break;
        default: n.op = ACC_TMP; break;
        }
        n.ref = s->second.second;
        for (int d = 0; d < 3; ++d) n.off[d] = off[d];
        return add(n);
    }

    void parse_apply(const Tok &kw) {
        Operator op;
        op.line = kw.line;
        std::vector<std::pair<Tok, std::string>> names;
        while (true) {
            const Tok &at = peek();
            names.push_back({at, name("an operator result name")});
            if (is(",")) {
                take();
                continue;
            }
            break;
        }
        P.ops.push_back(op);
        cur = &P.ops.back();
        locals.clear();
        std::vector<int> rets;
        std::vector<Tok> ret_at;
        if (is("=")) {  // short form: apply r = expr
            take();
            ret_at.push_back(peek());
            rets.push_back(expr());
        } else {
            expect("{");
            while (!is_kw("return")) {
                const Tok &at = peek();
                std::string ln = name("a local assignment or 'return'");
                if (locals.count(ln) || sym.count(ln) || reserved(ln)) fail(at, "'" + ln + "' is already defined");
                expect("=");
                int e = expr();
                locals[ln] = e;
            }
            take();
            while (true) {
                ret_at.push_back(peek());
                rets.push_back(expr());
                if (is(",")) {
                    take();
                    continue;
                }
                break;
            }
            expect("}");
        }
        if (rets.size() != names.size())
            fail(kw, "operator defines " + std::to_string(names.size()) + " results but returns " + std::to_string(rets.size()));
        for (size_t r = 0; r < rets.size(); ++r) need_num(ret_at[r], rets[r], "return value");
        int opi = (int)P.ops.size() - 1;
        for (size_t r = 0; r < names.size(); ++r) {
            int ti = (int)P.temp_names.size();
            declare(names[r].first, names[r].second, S_TEMP, ti);
            P.temp_names.push_back(names[r].second);
            P.temp_op.push_back(opi);
            P.temp_slot.push_back((int)r);
            cur->results.push_back(ti);
        }
        cur->roots = rets;
        cur = nullptr;
    }

    void parse() {
        if (!is_kw("program")) fail(peek(), "a stencil program starts with 'program NAME'");
        take();
        const Tok &pn = peek();
        P.name = name("the program name");
        if (reserved(P.name)) fail(pn, "'" + P.name + "' is a reserved word");
        while (peek().kind != T_END && !is_kw("end")) {
            const Tok &kw = peek();
            if (kw.kind != T_NAME) fail(kw, "expected a declaration (input, scalar, output, apply, store)");
            take();
            if (kw.s == "input") {
                const Tok &at = peek();
                std::string n = name("an input name");
                int kinv = 0;
                if (is(":")) {
                    take();
                    const Tok &k = peek();
                    std::string dims = name("'ij' or 'ijk'");
                    if (dims == "ij") kinv = 1;
                    else if (dims != "ijk") fail(k, "input dimensions are 'ij' (k-invariant) or 'ijk'");
                }
                declare(at, n, S_INPUT, (int)P.in_names.size());
                P.in_names.push_back(n);
                P.in_kinv.push_back(kinv);
            } else if (kw.s == "scalar") {
                const Tok &at = peek();
                std::string n = name("a scalar name");
                double v = 0;
                if (is("=")) {
                    take();
                    bool neg = false;
                    if (is("-")) {
                        take();
                        neg = true;
                    }
                    if (peek().kind != T_NUM) fail(peek(), "expected the scalar's default value");
                    v = take().num;
                    if (neg) v = -v;
                }
                declare(at, n, S_SCALAR, (int)P.sc_names.size());
                P.sc_names.push_back(n);
                P.sc_dflt.push_back(v);
            } else if (kw.s == "output") {
                const Tok &at = peek();
                std::string n = name("an output name");
                declare(at, n, S_OUTPUT, (int)P.out_names.size());
                P.out_names.push_back(n);
                P.out_temp.push_back(-1);
            } else if (kw.s == "apply") {
                parse_apply(kw);
            } else if (kw.s == "store") {
                const Tok &at = peek();
                std::string tn = name("the stored operator result");
                expect("->");
                const Tok &ot = peek();
                std::string on = name("an output name");
                auto ts = sym.find(tn);
                if (ts == sym.end() || ts->second.first != S_TEMP) fail(at, "'" + tn + "' is not an operator result");
                auto os = sym.find(on);
                if (os == sym.end() || os->second.first != S_OUTPUT) fail(ot, "'" + on + "' is not a declared output");
                if (P.out_temp[os->second.second] >= 0) fail(ot, "output '" + on + "' is stored twice");
                P.out_temp[os->second.second] = ts->second.second;
            } else {
                fail(kw, "unknown declaration '" + kw.s + "'");
            }
        }
        if (is_kw("end")) take();
        if (peek().kind != T_END) fail(peek(), "text after 'end'");
        if (P.out_names.empty()) fail(peek(), "the program has no output");
        for (size_t o = 0; o < P.out_names.size(); ++o)
            if (P.out_temp[o] < 0) fail(peek(), "output '" + P.out_names[o] + "' is never stored");
    }
};

// shape inference (§5.2)
static void infer_shapes(Program &P) {
    const int nin = (int)P.in_names.size();
    std::vector<bool> in_set(nin, false);
    P.in_lo.assign(nin, {0, 0, 0});
    P.in_hi.assign(nin, {0, 0, 0});
    P.in_used.assign(nin, 0);
    P.temp_buffered.assign(P.temp_names.size(), 0);
    auto grow = [](int lo[3], int hi[3], bool &set, const int clo[3], const int chi[3], const int off[3]) {
        for (int d = 0; d < 3; ++d) {
            int a = clo[d] + off[d], b = chi[d] + off[d];
            if (!set || a < lo[d]) lo[d] = a;
            if (!set || b > hi[d]) hi[d] = b;
        }
        set = true;
    };
    static const int Z[3] = {0, 0, 0};
    for (size_t o = 0; o < P.out_names.size(); ++o) {
        Operator &op = P.ops[P.temp_op[P.out_temp[o]]];
        grow(op.lo, op.hi, op.live, Z, Z, Z);  // the store range is the domain
    }
    for (int a = (int)P.ops.size() - 1; a >= 0; --a) {
        Operator &op = P.ops[a];
        if (!op.live) continue;
        for (const Node &n : op.nodes) {
            if (n.op == ACC_IN) {
                int off[3] = {n.off[0], n.off[1], P.in_kinv[n.ref] ? 0 : n.off[2]};
                bool s = in_set[n.ref];
                grow(P.in_lo[n.ref].data(), P.in_hi[n.ref].data(), s, op.lo, op.hi, off);
                in_set[n.ref] = s;
                if (P.in_kinv[n.ref]) P.in_lo[n.ref][2] = P.in_hi[n.ref][2] = 0;
                P.in_used[n.ref] = 1;
            } else if (n.op == ACC_TMP) {
                Operator &pr = P.ops[P.temp_op[n.ref]];
                grow(pr.lo, pr.hi, pr.live, op.lo, op.hi, n.off);
                P.temp_buffered[n.ref] = 1;
            }
        }
    }
    // extents are reported relative to the domain: lo <= 0 <= hi (the store range is covered)
    for (int q = 0; q < nin; ++q)
        for (int d = 0; d < 3; ++d) {
            P.in_lo[q][d] = std::min(P.in_lo[q][d], 0);
            P.in_hi[q][d] = std::max(P.in_hi[q][d], 0);
        }
}

// ---------------------------------------------------------------------------------------------
// code generation
// ---------------------------------------------------------------------------------------------
struct Spec {
    int dtype = OEC_F64;
    int variant = OEC_VARIANT_NAIVE;
    int unroll = 1;
    int unroll_dim = 1;  // 1: j, 2: k
    int tile_cfg = 0;    // OEC_VARIANT_TILED: index into TILE_CFGS
    int n[3] = {0, 0, 0};  // domain size
    std::vector<int32_t> in_sj, in_sk, out_sj, out_sk;
};

// OEC_VARIANT_TILED: the B200 execution model for a stencil-language program.  Persistent CTAs of
// 256 threads walk items = (64 x 8 tile of (i, j), one k-level); every 3D input's box -- the tile
// grown by that input's access extent (shape inference) in i, j and k -- is staged into a
// shared-memory ring by TMA (one elected thread, mbarrier completion), the inlined expression
// reads shared memory at immediate offsets, k-invariant inputs are read through L1, outputs are
// stored straight from registers.  S stages keep the next items' boxes in flight while one is
// computed.
struct TileLayout {
    int ti = 64, tj = 8, rows = 2;   // tile, rows per thread (256 threads = ti x (tj / rows))
    int ntile[3] = {0, 0, 0};        // items per dim (k: one level per item)
    std::vector<int> staged;         // per input: 1 = TMA box in shared memory
    std::vector<int> w, h, dpt;      // box extents (i, j, k) per staged input
    std::vector<int> swap;           // tensor dims ordered (i, k, j) -- shared memory [j][k][i]
    std::vector<int> off;            // byte offset of the box within a stage
    std::vector<int32_t> ssj, ssk;   // shared-memory strides (elements)
    int stage_bytes = 0, stages = 2, smem = 0;
    int stage_bytes_tx(int esz) const {  // bytes the boxes of one stage deliver (complete_tx count)
        int b = 0;
        for (size_t q = 0; q < staged.size(); ++q)
            if (staged[q]) b += w[q] * h[q] * dpt[q] * esz;
        return b;
    }
};

// tiled configurations (rows per thread, shared-memory budget per CTA in KB): fewer rows and a
// smaller ring give more resident CTAs (latency hiding), more rows share loads between rows;
// AUTO tries them all, OEC_VARIANT_TILED uses the first (measured best on most of the suite).
// (measured: deeper rings -- {1, 110}, {1, 80} -- are slower at 128^2 and 1024^2; more resident
// CTAs matter more than bytes in flight per CTA, profiles/ncu_summary_r01.md)
static const int TILE_CFGS[][2] = {{1, 56}, {1, 36}, {2, 110}, {4, 110}};
static const int N_TILE_CFGS = 4;

static TileLayout tile_layout(const Program &P, const Spec &S, int esz) {
    TileLayout L;
    L.rows = TILE_CFGS[S.tile_cfg][0];
    const int cta_kb = TILE_CFGS[S.tile_cfg][1];
    L.ti = S.n[0] >= 64 ? 64 : 32;
    L.tj = (256 / L.ti) * L.rows;
    L.ntile[0] = (S.n[0] + L.ti - 1) / L.ti;
    L.ntile[1] = (S.n[1] + L.tj - 1) / L.tj;
    L.ntile[2] = S.n[2];
    const int nin = (int)P.in_names.size();
    L.staged.assign(nin, 0);
    L.w.assign(nin, 0);
    L.h.assign(nin, 0);
    L.dpt.assign(nin, 0);
    L.swap.assign(nin, 0);
    L.off.assign(nin, 0);
    L.ssj.assign(nin, 0);
    L.ssk.assign(nin, 0);
    int at = 0;
    for (int q = 0; q < nin; ++q) {
        if (!P.in_used[q]) continue;
        L.staged[q] = 1;  // k-invariant inputs: a 2D (i, j) box, read at every level
        int w = L.ti + P.in_hi[q][0] - P.in_lo[q][0];
        // the box starts on a 16-byte boundary (a misaligned start faults with an illegal
        // instruction, measured on B200): up to 16/esz - 1 extra leading columns, whose count (the
        // shift) is a launch argument; inner extent a multiple of 16 bytes
        const int per16 = 16 / esz;
        w = (w + per16 - 1 + per16 - 1) / per16 * per16;
        L.w[q] = w;
        L.h[q] = L.tj + P.in_hi[q][1] - P.in_lo[q][1];
        L.dpt[q] = P.in_kinv[q] ? 1 : 1 + P.in_hi[q][2] - P.in_lo[q][2];
        L.swap[q] = !P.in_kinv[q] && S.in_sk[q] < S.in_sj[q];
        if (P.in_kinv[q]) {  // shared memory [j][i]; k offsets of a k-invariant input read the same box
            L.ssj[q] = w;
            L.ssk[q] = 0;
        } else if (L.swap[q]) {  // shared memory [j][k][i]
            L.ssk[q] = w;
            L.ssj[q] = w * L.dpt[q];
        } else {  // [k][j][i]
            L.ssj[q] = w;
            L.ssk[q] = w * L.h[q];
        }
        L.off[q] = at;
        at += (w * L.h[q] * L.dpt[q] * esz + 127) / 128 * 128;
    }
    L.stage_bytes = at;
    // 2..4 stages, at most ~110 KB per CTA so two CTAs share an SM
    L.stages = at > 0 ? std::max(2, std::min(4, (cta_kb * 1024) / std::max(at, 1))) : 1;
    L.smem = L.stages * at + 2 * 8 * L.stages + 16;  // ring + full / empty barriers
    return L;
}

static int unroll_of(int variant) {
    return (variant == OEC_VARIANT_UNROLL2 || variant == OEC_VARIANT_UNROLL2_K)   ? 2
           : (variant == OEC_VARIANT_UNROLL4 || variant == OEC_VARIANT_UNROLL4_K) ? 4
                                                                                 : 1;
}
static int unroll_dim_of(int variant) {
    return (variant == OEC_VARIANT_UNROLL2_K || variant == OEC_VARIANT_UNROLL4_K) ? 2 : 1;
}

// launch geometry of the paper's execution model: one thread per point (U points along j)
static void block_of(const int n[3], int *bx, int *by) {
    *bx = n[0] <= 32 ? 32 : n[0] <= 64 ? 64 : 128;
    *by = 256 / *bx;
}

struct TempLayout {  // a materialised temporary (original level): dense box over the operator's domain
    int lo[3], e[3];
    int32_t sj, sk;
    size_t elems;
};

static std::vector<TempLayout> temp_layouts(const Program &P, const Spec &S, size_t *total) {
    std::vector<TempLayout> L(P.temp_names.size());
    *total = 0;
    for (size_t t = 0; t < P.temp_names.size(); ++t) {
        const Operator &op = P.ops[P.temp_op[t]];
        TempLayout &l = L[t];
        for (int d = 0; d < 3; ++d) {
            l.lo[d] = op.lo[d];
            l.e[d] = S.n[d] + op.hi[d] - op.lo[d];
        }
        l.sj = (l.e[0] + 31) / 32 * 32;  // 256-byte row pitch (f64)
        l.sk = l.sj * l.e[1];
        l.elems = (op.live && P.temp_buffered[t]) ? (size_t)l.sk * l.e[2] : 0;
        *total += (l.elems + 63) / 64 * 64;
    }
    return L;
}

static std::string lit(double v, bool f32) {
    char b[64];
    if (f32) {
        float f = (float)v;  // rounded once to binary32 (R21)
        snprintf(b, sizeof b, "%af", (double)f);
    } else {
        snprintf(b, sizeof b, "%a", v);
    }
    std::string s = b;
    if (s.find("inf") != std::string::npos || s.find("nan") != std::string::npos)
        throw Error{"non-finite literal"};
    return "(" + s + ")";
}

struct Emitter {
    const Program &P;
    const Spec &S;
    bool f32;
    bool original;                // temporaries are loads from buffers (original level)
    const std::vector<TempLayout> *tl = nullptr;
    std::ostringstream o;
    std::string ind = "        ";
    int nv = 0;
    std::map<std::tuple<int, int, int, int>, std::string> loads, tloads;
    std::map<std::tuple<int, int, int, int>, std::vector<std::string>> inst;

    Emitter(const Program &p, const Spec &s, bool orig) : P(p), S(s), f32(s.dtype == OEC_F32), original(orig) {}

    std::string fresh(const char *pfx) { return pfx + std::to_string(nv++); }

    std::string load_in(int q, const int off[3]) {
        int dk = P.in_kinv[q] ? 0 : off[2];
        auto key = std::make_tuple(q, off[0], off[1], dk);
        auto it = loads.find(key);
        if (it != loads.end()) return it->second;
        long long c = (long long)off[0] + (long long)off[1] * S.in_sj[q] + (long long)dk * S.in_sk[q];
        std::string v = fresh("x");
        o << ind << "const T " << v << " = b" << q << "[" << c << "];\n";
        loads[key] = v;
        return v;
    }
    std::string load_tmp(int t, const int off[3]) {
        auto key = std::make_tuple(t, off[0], off[1], off[2]);
        auto it = tloads.find(key);
        if (it != tloads.end()) return it->second;
        const TempLayout &l = (*tl)[t];
        long long c = (long long)off[0] + (long long)off[1] * l.sj + (long long)off[2] * l.sk;
        std::string v = fresh("y");
        o << ind << "const T " << v << " = bt" << t << "[" << c << "];\n";
        tloads[key] = v;
        return v;
    }
    std::string temp(int t, const int off[3]) {
        if (original) return load_tmp(t, off);
        return instance(P.temp_op[t], off)[P.temp_slot[t]];
    }
    // operator `a` evaluated at offset `off` from the thread's point (inlining)
    const std::vector<std::string> &instance(int a, const int off[3]) {
        auto key = std::make_tuple(a, off[0], off[1], off[2]);
        auto it = inst.find(key);
        if (it != inst.end()) return it->second;
        const Operator &op = P.ops[a];
        std::vector<char> reach(op.nodes.size(), 0);
        for (int r : op.roots) reach[r] = 1;
        for (int q = (int)op.nodes.size() - 1; q >= 0; --q)
            if (reach[q]) {
                const Node &n = op.nodes[q];
                if (n.a >= 0) reach[n.a] = 1;
                if (n.b >= 0) reach[n.b] = 1;
                if (n.c >= 0) reach[n.c] = 1;
            }
        std::vector<std::string> v(op.nodes.size());
        const char *fabs_ = f32 ? "fabsf" : "fabs", *sqrt_ = f32 ? "sqrtf" : "sqrt";
        for (size_t q = 0; q < op.nodes.size(); ++q) {
            if (!reach[q]) continue;
            const Node &n = op.nodes[q];
            int aoff[3] = {off[0] + n.off[0], off[1] + n.off[1], off[2] + n.off[2]};
            switch (n.op) {
            case LIT: v[q] = lit(n.lit, f32); continue;
            case SCALAR: v[q] = "s" + std::to_string(n.ref); continue;
            case ACC_IN: v[q] = load_in(n.ref, aoff); continue;
            case ACC_TMP: v[q] = temp(n.ref, aoff); continue;
            default: break;
            }
            std::string e;
            const std::string &A = n.a >= 0 ? v[n.a] : e, &B = n.b >= 0 ? v[n.b] : e;
            switch (n.op) {
            case NEG: e = "-" + A; break;
            case ADD: e = A + " + " + B; break;
            case SUB: e = A + " - " + B; break;
            case MUL: e = A + " * " + B; break;
            case DIV: e = A + " / " + B; break;
            case LT: e = A + " < " + B; break;
            case GT: e = A + " > " + B; break;
            case LE: e = A + " <= " + B; break;
            case GE: e = A + " >= " + B; break;
            case EQ: e = A + " == " + B; break;
            case NE: e = A + " != " + B; break;
            case AND: e = A + " && " + B; break;
            case OR: e = A + " || " + B; break;
            case NOT: e = "!" + A; break;
            case SELECT: e = v[n.c] + " ? " + A + " : " + B; break;
            case MIN: e = "(" + B + " < " + A + ") ? " + B + " : " + A; break;  // min(a,b) := b < a ? b : a
            case MAX: e = "(" + B + " > " + A + ") ? " + B + " : " + A; break;  // max(a,b) := b > a ? b : a
            case ABS: e = std::string(fabs_) + "(" + A + ")"; break;
            case SQRT: e = std::string(sqrt_) + "(" + A + ")"; break;
            }
            std::string nm = fresh(n.boolean ? "c" : "v");
            o << ind << (n.boolean ? "const bool " : "const T ") << nm << " = " << e << ";\n";
            v[q] = nm;
        }
        std::vector<std::string> res;
        for (int r : op.roots) res.push_back(v[r]);
        return inst.emplace(key, res).first->second;
    }
    void reset() {
        loads.clear();
        tloads.clear();
        inst.clear();
    }
};

static void emit_header(std::ostringstream &o, const Program &P, const Spec &S, const char *what) {
    o << "// generated by liboec (csrc/jit.cpp) from stencil program '" << P.name << "': " << what << "\n"
      << "// domain " << S.n[0] << " x " << S.n[1] << " x " << S.n[2] << ", " << (S.dtype == OEC_F32 ? "f32" : "f64")
      << "; every size and stride is a compile-time constant (size specialization, P:338)\n"
      << "typedef " << (S.dtype == OEC_F32 ? "float" : "double") << " T;\n";
}

static std::string kernel_params(const Program &P, bool outputs, const std::vector<int> *tmps_read,
                                 const std::vector<int> *tmps_written) {
    std::ostringstream o;
    const char *sep = "";
    for (size_t q = 0; q < P.in_names.size(); ++q) {
        o << sep << "const T *__restrict__ f" << q;
        sep = ", ";
    }
    if (tmps_read)
        for (int t : *tmps_read) {
            o << sep << "const T *__restrict__ ft" << t;
            sep = ", ";
        }
    if (tmps_written)
        for (int t : *tmps_written) {
            o << sep << "T *__restrict__ wt" << t;
            sep = ", ";
        }
    if (outputs)
        for (size_t q = 0; q < P.out_names.size(); ++q) {
            o << sep << "T *__restrict__ g" << q;
            sep = ", ";
        }
    for (size_t q = 0; q < P.sc_names.size(); ++q) {
        o << sep << "const T s" << q;
        sep = ", ";
    }
    return o.str();
}

// inline / inline+unroll(U): one kernel, every operator inlined into the outputs.  Unrolling
// along j (dim 1) or k (dim 2): one thread evaluates U points; operator instances and loads
// shared between them are emitted once (CSE), e.g. the k+1 plane of a k-unrolled thread.
static std::string gen_fused(const Program &P, const Spec &S) {
    std::ostringstream o;
    const int U = S.unroll, ud = S.unroll_dim;
    int bx, by;
    block_of(S.n, &bx, &by);
    const char *dn = ud == 2 ? "k" : "j";
    emit_header(o, P, S,
                U == 1 ? "inline (P:431)"
                       : ("inline+unroll(" + std::to_string(U) + ") along " + dn + " (P:447-451)").c_str());
    o << "extern \"C\" __global__ void __launch_bounds__(" << bx * by << ") oec_jit_fused("
      << kernel_params(P, true, nullptr, nullptr) << ") {\n"
      << "    const int i = blockIdx.x * " << bx << " + threadIdx.x;\n";
    if (ud == 2)
        o << "    const int j = blockIdx.y * " << by << " + threadIdx.y;\n"
          << "    const int k0 = blockIdx.z * " << U << ";\n"
          << "    if (i >= " << S.n[0] << " || j >= " << S.n[1] << ") return;\n";
    else
        o << "    const int j0 = (blockIdx.y * " << by << " + threadIdx.y) * " << U << ";\n"
          << "    const int k = blockIdx.z;\n"
          << "    if (i >= " << S.n[0] << " || j0 >= " << S.n[1] << ") return;\n";
    // rows: points per thread; jv / kv: the first point's j / k expressions
    auto body = [&](int rows, const char *jv, const char *kv) {
        Emitter E(P, S, false);
        for (size_t q = 0; q < P.in_names.size(); ++q)
            if (P.in_used[q])
                E.o << E.ind << "const T *__restrict__ b" << q << " = f" << q << " + (i + " << jv << " * " << S.in_sj[q]
                    << (P.in_kinv[q] ? std::string() : std::string(" + ") + kv + " * " + std::to_string(S.in_sk[q]))
                    << ");\n";
        std::vector<std::vector<std::string>> vals(rows);
        for (int u = 0; u < rows; ++u)
            for (size_t q = 0; q < P.out_names.size(); ++q) {
                int t = P.out_temp[q];
                int off[3] = {0, ud == 1 ? u : 0, ud == 2 ? u : 0};
                vals[u].push_back(E.temp(t, off));
            }
        // stores after all loads (outputs kept in registers)
        for (int u = 0; u < rows; ++u)
            for (size_t q = 0; q < P.out_names.size(); ++q)
                E.o << E.ind << "g" << q << "[i + (" << jv << (ud == 1 ? " + " + std::to_string(u) : std::string()) << ") * "
                    << S.out_sj[q] << " + (" << kv << (ud == 2 ? " + " + std::to_string(u) : std::string()) << ") * "
                    << S.out_sk[q] << "] = " << vals[u][q] << ";\n";
        return E.o.str();
    };
    const int N = S.n[ud];
    const std::string v0 = ud == 2 ? "k0" : "j0";
    const char *jv = ud == 2 ? "j" : "j0", *kv = ud == 2 ? "k0" : "k";
    if (N % U == 0) {
        o << "    {\n" << body(U, jv, kv) << "    }\n";
    } else {
        o << "    if (" << v0 << " + " << U << " <= " << N << ") {\n"
          << body(U, jv, kv) << "    } else {\n"
          << "      for (int r = " << v0 << "; r < " << N << "; ++r) {\n"
          << body(1, ud == 2 ? "j" : "r", ud == 2 ? "r" : "k") << "      }\n    }\n";
    }
    o << "}\n";
    return o.str();
}

// original: one kernel per live operator over its inferred domain, temporaries in HBM
static std::string gen_original(const Program &P, const Spec &S, const std::vector<TempLayout> &L,
                                std::vector<int> *kernel_ops) {
    std::ostringstream o;
    emit_header(o, P, S, "original level (P:616): one kernel per stencil.apply, temporaries materialised");
    for (size_t a = 0; a < P.ops.size(); ++a) {
        const Operator &op = P.ops[a];
        if (!op.live) continue;
        kernel_ops->push_back((int)a);
        int e[3];
        for (int d = 0; d < 3; ++d) e[d] = S.n[d] + op.hi[d] - op.lo[d];
        int bx, by;
        block_of(e, &bx, &by);
        std::vector<int> tr, tw;
        for (size_t t = 0; t < P.temp_names.size(); ++t) {
            if (L[t].elems && P.temp_op[t] == (int)a) tw.push_back((int)t);
            if (L[t].elems && P.temp_op[t] < (int)a) tr.push_back((int)t);
        }
        o << "extern \"C\" __global__ void __launch_bounds__(" << bx * by << ") oec_jit_op" << a << "("
          << kernel_params(P, true, &tr, &tw) << ") {\n"
          << "    const int i = " << op.lo[0] << " + (int)(blockIdx.x * " << bx << " + threadIdx.x);\n"
          << "    const int j = " << op.lo[1] << " + (int)(blockIdx.y * " << by << " + threadIdx.y);\n"
          << "    const int k = " << op.lo[2] << " + (int)blockIdx.z;\n"
          << "    if (i >= " << S.n[0] + op.hi[0] << " || j >= " << S.n[1] + op.hi[1] << ") return;\n";
        Emitter E(P, S, true);
        E.tl = &L;
        E.ind = "    ";
        for (size_t q = 0; q < P.in_names.size(); ++q)
            E.o << E.ind << "const T *__restrict__ b" << q << " = f" << q << " + (i + j * " << S.in_sj[q]
                << (P.in_kinv[q] ? "" : " + k * " + std::to_string(S.in_sk[q])) << ");\n";
        for (int t : tr)
            E.o << E.ind << "const T *__restrict__ bt" << t << " = ft" << t << " + (i + j * " << L[t].sj << " + k * "
                << L[t].sk << ");\n";
        static const int Z[3] = {0, 0, 0};
        const std::vector<std::string> res = E.instance((int)a, Z);
        for (int t : tw)
            E.o << E.ind << "wt" << t << "[i + j * " << L[t].sj << " + k * " << L[t].sk << "] = " << res[P.temp_slot[t]]
                << ";\n";
        bool any_out = false;
        for (size_t q = 0; q < P.out_names.size(); ++q)
            if (P.temp_op[P.out_temp[q]] == (int)a) any_out = true;
        if (any_out) {
            E.o << E.ind << "if (i >= 0 && i < " << S.n[0] << " && j >= 0 && j < " << S.n[1] << " && k >= 0 && k < "
                << S.n[2] << ") {\n";
            for (size_t q = 0; q < P.out_names.size(); ++q)
                if (P.temp_op[P.out_temp[q]] == (int)a)
                    E.o << E.ind << "    g" << q << "[i + j * " << S.out_sj[q] << " + k * " << S.out_sk[q]
                        << "] = " << res[P.temp_slot[P.out_temp[q]]] << ";\n";
            E.o << E.ind << "}\n";
        }
        o << E.o.str() << "}\n";
    }
    return o.str();
}

// ---------------------------------------------------------------------------------------------
// NVRTC (dlopen'ed: liboec loads without it; JIT calls fail with OEC_ERR_UNSUPPORTED) and the
// driver API (through the runtime's entry points: no link dependence on libcuda)
// ---------------------------------------------------------------------------------------------
struct Nvrtc {
    bool ok = false;
    std::string why;
    decltype(&nvrtcCreateProgram) create;
    decltype(&nvrtcCompileProgram) compile;
    decltype(&nvrtcGetProgramLogSize) log_size;
    decltype(&nvrtcGetProgramLog) log;
    decltype(&nvrtcGetCUBINSize) cubin_size;
    decltype(&nvrtcGetCUBIN) cubin;
    decltype(&nvrtcDestroyProgram) destroy;
    decltype(&nvrtcGetErrorString) errstr;
    decltype(&nvrtcVersion) version;
};
static Nvrtc g_nv;
static std::once_flag g_nv_once;

static void load_nvrtc() {
    const char *cands[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    void *h = nullptr;
    for (const char *c : cands)
        if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
        g_nv.why = "NVRTC (libnvrtc.so.12) not loadable";
        return;
    }
#define SYM(f, n)                                            \
    g_nv.f = (decltype(g_nv.f))dlsym(h, n);                  \
    if (!g_nv.f) {                                           \
        g_nv.why = std::string("NVRTC lacks ") + n;          \
        return;                                              \
    }
    SYM(create, "nvrtcCreateProgram")
    SYM(compile, "nvrtcCompileProgram")
    SYM(log_size, "nvrtcGetProgramLogSize")
    SYM(log, "nvrtcGetProgramLog")
    SYM(cubin_size, "nvrtcGetCUBINSize")
    SYM(cubin, "nvrtcGetCUBIN")
    SYM(destroy, "nvrtcDestroyProgram")
    SYM(errstr, "nvrtcGetErrorString")
    SYM(version, "nvrtcVersion")
#undef SYM
    g_nv.ok = true;
}

// compile CUDA source to an sm_100a cubin
static oec_status nvrtc_compile(const std::string &src, const char *pname, std::vector<char> *cubin) {
    std::call_once(g_nv_once, load_nvrtc);
    if (!g_nv.ok) return set_error(OEC_ERR_UNSUPPORTED, "%s: %s", pname, g_nv.why.c_str());
    nvrtcProgram prog;
    nvrtcResult r = g_nv.create(&prog, src.c_str(), "oec_jit.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return set_error(OEC_ERR_CUDA, "%s: nvrtcCreateProgram: %s", pname, g_nv.errstr(r));
    // -fmad=false: no contraction (R3); IEEE division / sqrt, no flush to zero
    const char *opts[] = {"-arch=sm_100a", "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                          "-std=c++17", "-lineinfo"};
    r = g_nv.compile(prog, (int)(sizeof opts / sizeof *opts), opts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        g_nv.log_size(prog, &n);
        std::string log(n, '\0');
        if (n) g_nv.log(prog, &log[0]);
        g_nv.destroy(&prog);
        return set_error(OEC_ERR_CUDA, "%s: NVRTC compilation failed: %s", pname, log.c_str());
    }
    size_t n = 0;
    g_nv.cubin_size(prog, &n);
    cubin->resize(n);
    g_nv.cubin(prog, cubin->data());
    g_nv.destroy(&prog);
    return OEC_OK;
}

struct Drv {
    bool ok = false;
    PFN_cuModuleLoadData_v2000 load = nullptr;
    PFN_cuModuleGetFunction_v2000 get = nullptr;
    PFN_cuLaunchKernel_v4000 launch = nullptr;
    PFN_cuLaunchKernelEx_v11060 launch_ex = nullptr;  // programmatic dependent launch of tiled kernels
    PFN_cuFuncSetAttribute_v9000 set_attr = nullptr;
};
static Drv g_drv;
static std::once_flag g_drv_once;
static void load_drv() {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    if (cudaGetDriverEntryPoint("cuModuleLoadData", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        g_drv.load = (PFN_cuModuleLoadData_v2000)f;
    if (cudaGetDriverEntryPoint("cuModuleGetFunction", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        g_drv.get = (PFN_cuModuleGetFunction_v2000)f;
    if (cudaGetDriverEntryPoint("cuLaunchKernel", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        g_drv.launch = (PFN_cuLaunchKernel_v4000)f;
    if (cudaGetDriverEntryPoint("cuFuncSetAttribute", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        g_drv.set_attr = (PFN_cuFuncSetAttribute_v9000)f;
    if (cudaGetDriverEntryPoint("cuLaunchKernelEx", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        g_drv.launch_ex = (PFN_cuLaunchKernelEx_v11060)f;
    g_drv.ok = g_drv.load && g_drv.get && g_drv.launch && g_drv.set_attr;
}

// ---------------------------------------------------------------------------------------------
// registry, kernel cache, runner
// ---------------------------------------------------------------------------------------------
struct Compiled {
    bool attr_set = false;  // dynamic shared-memory limit raised (tiled kernels)
    std::vector<CUfunction> fns;
    std::vector<int> ops;  // original level: operator of each kernel
};
struct Registered {
    Program prog;
    ProgDesc desc;
};
static std::mutex g_mu;
static std::map<std::string, std::shared_ptr<Registered>> g_reg;
static std::map<std::string, std::shared_ptr<Compiled>> g_cache;
static long long g_uid = 0;
struct Workspace {
    void *p = nullptr;
    size_t bytes = 0;
};
static std::map<int, Workspace> g_ws;  // per device (original level temporaries)

static std::string spec_key(const Program &P, const Spec &S, int device) {
    std::ostringstream k;
    if (S.variant == OEC_VARIANT_TILED) k << "tile" << S.tile_cfg << "|";
    k << P.name << "#" << P.uid << "|d" << device << "|t" << S.dtype << "|v" << S.variant << "|n" << S.n[0] << "," << S.n[1]
      << "," << S.n[2];
    for (size_t q = 0; q < S.in_sj.size(); ++q) k << "|i" << S.in_sj[q] << "," << S.in_sk[q];
    for (size_t q = 0; q < S.out_sj.size(); ++q) k << "|o" << S.out_sj[q] << "," << S.out_sk[q];
    return k.str();
}


static const char *TMA_PRELUDE = R"(
struct __align__(64) TM { unsigned long long v[16]; };
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(unsigned long long *b, unsigned n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long *b, unsigned ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void tma2(void *dst, const TM *m, unsigned long long *b, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su32(dst)), "l"((unsigned long long)m), "r"(su32(b)), "r"(c0), "r"(c1) : "memory"); }
__device__ __forceinline__ void tma3(void *dst, const TM *m, unsigned long long *b, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(su32(dst)), "l"((unsigned long long)m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2) : "memory"); }
// L2 prefetch of a box before griddepcontrol.wait (only warms L2, the point of coherence; csrc/tma.h)
__device__ __forceinline__ void pf2(const TM *m, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((unsigned long long)m), "r"(c0), "r"(c1)
                 : "memory"); }
__device__ __forceinline__ void pf3(const TM *m, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"((unsigned long long)m), "r"(c0),
                 "r"(c1), "r"(c2) : "memory"); }
)";

// experiment (round 2, profiles/r02/jit_tiled_producer_ab.md): a producer warp refilling stages
// behind per-stage empty barriers instead of a CTA-wide barrier per item -- 1.5-3% faster for
// nh_p_grad / fvtp2d_qj with the 110 KB ring, up to 30% slower with the 56 KB one: off
#ifndef JIT_TILED_PRODUCER
#define JIT_TILED_PRODUCER 0
#endif
static constexpr int TILED_THREADS = JIT_TILED_PRODUCER ? 288 : 256;  // 8 compute warps (+ a producer warp)

static std::string gen_tiled(const Program &P, const Spec &S) {
    const int esz = S.dtype == OEC_F32 ? 4 : 8;
    const TileLayout L = tile_layout(P, S, esz);
    std::ostringstream o;
    emit_header(o, P, S, "B200 tiled: TMA-staged input boxes in a shared-memory ring, persistent CTAs");
    o << TMA_PRELUDE;
    // parameters: tensor maps + base coordinates of staged inputs, pointers of the others
    std::ostringstream prm;
    const char *sep = "";
    for (size_t q = 0; q < P.in_names.size(); ++q) {
        if (L.staged[q])
            prm << sep << "const __grid_constant__ TM tm" << q << ", const int c" << q << "x, const int c" << q << "y, const int c" << q
                << "z, const int h" << q;
        else
            prm << sep << "const T *__restrict__ f" << q;
        sep = ", ";
    }
    for (size_t q = 0; q < P.out_names.size(); ++q) prm << sep << "T *__restrict__ g" << q;
    for (size_t q = 0; q < P.sc_names.size(); ++q) prm << sep << "const T s" << q;
    const int NI = L.ntile[0] * L.ntile[1] * L.ntile[2];
    o << "extern \"C\" __global__ void __launch_bounds__(" << TILED_THREADS << ") oec_jit_tiled(" << prm.str() << ") {\n"
      << "    extern __shared__ __align__(128) unsigned char smem[];\n"
      << "    unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + " << L.stages * L.stage_bytes << ");\n"
      << "    unsigned long long *empty = full + " << L.stages << ";\n"
      << "    const int tid = threadIdx.x, tx = tid % " << L.ti << ", ty = tid / " << L.ti << ";\n"
      << "    const int NITEMS = " << NI << ";\n";
    // TMA issue of one item's boxes into stage `st`, emitted inline where it is used (a lambda
    // capturing the __grid_constant__ tensor maps would not keep their param-space addresses)
    auto issue = [&](const std::string &ind, const std::string &item, const std::string &st, bool prefetch = false) {
        std::ostringstream w;
        w << ind << "{\n"
          << ind << "    const int it_ = " << item << ", st_ = " << st << ";\n"
          << ind << "    const int ti_ = it_ % " << L.ntile[0] << ", tj_ = (it_ / " << L.ntile[0] << ") % " << L.ntile[1]
          << ", k_ = it_ / " << L.ntile[0] * L.ntile[1] << ";\n"
          << ind << "    const int i0_ = ti_ * " << L.ti << ", j0_ = tj_ * " << L.tj << ";\n";
        if (!prefetch) w << ind << "    mb_expect(&full[st_], " << L.stage_bytes_tx(esz) << ");\n";
        else w << ind << "    (void)st_;\n";
        for (size_t q = 0; q < P.in_names.size(); ++q) {
            if (!L.staged[q]) continue;
            const std::string cq = "c" + std::to_string(q);
            const std::string dst = prefetch ? std::string("&tm") + std::to_string(q) + ", "
                                             : "smem + st_ * " + std::to_string(L.stage_bytes) + " + " + std::to_string(L.off[q]) +
                                                   ", &tm" + std::to_string(q) + ", &full[st_], ";
            if (P.in_kinv[q])
                w << ind << "    " << (prefetch ? "pf2(" : "tma2(") << dst << cq << "x + i0_, " << cq << "y + j0_);\n";
            else
                w << ind << "    " << (prefetch ? "pf3(" : "tma3(") << dst << cq << "x + i0_, "
                  << (L.swap[q] ? cq + "z + k_, " + cq + "y + j0_" : cq + "y + j0_, " + cq + "z + k_") << ");\n";
        }
        w << ind << "}\n";
        return w.str();
    };
    // programmatic dependent launch: barrier setup and an L2 prefetch of the first items overlap
    // the previous kernel's drain; every thread waits for it before touching its data
    o << "    asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n"
      << "    if (tid == 0) {\n"
      << "        for (int s = 0; s < " << L.stages << "; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 8); }\n"
      << "        asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
      << "        for (int s = 0; s < " << L.stages << "; ++s)\n"
      << "            if (blockIdx.x + s * gridDim.x < NITEMS)\n"
      << issue("            ", "blockIdx.x + s * gridDim.x", "s", true)
      << "    }\n"
      << "    asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
      << "    if (tid == 0) {\n"
      << "        for (int s = 0; s < " << L.stages << "; ++s)\n"
      << "            if (blockIdx.x + s * gridDim.x < NITEMS)\n"
      << issue("            ", "blockIdx.x + s * gridDim.x", "s")
      << "    }\n"
      << "    __syncthreads();\n";
#if JIT_TILED_PRODUCER
    // a producer warp refills a stage once the 8 compute warps have arrived on its empty barrier:
    // no CTA-wide barrier per item (round 1's __syncthreads was the top stall, ncu)
    o << "    if (tid >= 256) {\n"
      << "        if (tid == 256)\n"
      << "            for (int n = " << L.stages << ";; ++n) {\n"
      << "                const int nxt = blockIdx.x + n * gridDim.x;\n"
      << "                if (nxt >= NITEMS) break;\n"
      << "                const int sp = n % " << L.stages << ";\n"
      << "                mb_wait(&empty[sp], ((n / " << L.stages << ") - 1) & 1);\n"
      << "                asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
      << issue("                ", "nxt", "sp")
      << "            }\n"
      << "        return;\n"
      << "    }\n";
#endif
    o << "    for (int n = 0;; ++n) {\n"
      << "        const int item = blockIdx.x + n * gridDim.x;\n"
      << "        if (item >= NITEMS) break;\n"
      << "        const int st = n % " << L.stages << ";\n"
      << "        mb_wait(&full[st], (n / " << L.stages << ") & 1);\n"
      << "        const int ti = item % " << L.ntile[0] << ", tj = (item / " << L.ntile[0] << ") % " << L.ntile[1]
      << ", k = item / " << L.ntile[0] * L.ntile[1] << ";\n"
      << "        const int i = ti * " << L.ti << " + tx, jr = ty * " << L.rows << ", j = tj * " << L.tj << " + jr;\n"
      << "        {\n";
    // expression body: staged inputs read shared memory with shared-memory strides
    Spec SS = S;
    for (size_t q = 0; q < P.in_names.size(); ++q)
        if (L.staged[q]) {
            SS.in_sj[q] = L.ssj[q];
            SS.in_sk[q] = L.ssk[q];
        }
    Emitter E(P, SS, false);
    E.ind = "            ";
    for (size_t q = 0; q < P.in_names.size(); ++q) {
        if (!P.in_used[q]) continue;
        if (L.staged[q])
            E.o << E.ind << "const T *b" << q << " = reinterpret_cast<const T *>(smem + st * " << L.stage_bytes << " + "
                << L.off[q] << ") + ((tx - " << P.in_lo[q][0] << " + h" << q << ") + (jr - " << P.in_lo[q][1] << ") * " << L.ssj[q]
                << " + (" << -P.in_lo[q][2] << ") * " << L.ssk[q] << ");\n";
        else
            E.o << E.ind << "const T *__restrict__ b" << q << " = f" << q << " + (i + j * " << S.in_sj[q]
                << (P.in_kinv[q] ? std::string() : " + k * " + std::to_string(S.in_sk[q])) << ");\n";
    }
    std::vector<std::vector<std::string>> vals(L.rows);
    for (int u = 0; u < L.rows; ++u)
        for (size_t q = 0; q < P.out_names.size(); ++q) {
            int off[3] = {0, u, 0};
            vals[u].push_back(E.temp(P.out_temp[q], off));
        }
    for (int u = 0; u < L.rows; ++u) {
        E.o << E.ind << "if (i < " << S.n[0] << " && j + " << u << " < " << S.n[1] << ") {\n";
        for (size_t q = 0; q < P.out_names.size(); ++q)
            E.o << E.ind << "    g" << q << "[i + (j + " << u << ") * " << S.out_sj[q] << " + k * " << S.out_sk[q]
                << "] = " << vals[u][q] << ";\n";
        E.o << E.ind << "}\n";
    }
    o << E.o.str() << "        }\n";
#if JIT_TILED_PRODUCER
    o << "        __syncwarp();\n"
      << "        if ((tid & 31) == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" ::\"r\"(su32(&empty[st])) : \"memory\");\n";
#else
    o << "        __syncthreads();  // every thread is done with stage st\n"
      << "        if (tid == 0) {\n"
      << "            const int nxt = item + " << L.stages << " * gridDim.x;\n"
      << "            if (nxt < NITEMS) {\n"
      << "                asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
      << issue("                ", "nxt", "st")
      << "            }\n"
      << "        }\n";
#endif
    o << "    }\n"
      << "}\n";
    return o.str();
}

static std::string generate(const Program &P, const Spec &S, std::vector<int> *ops) {
    if (S.variant == OEC_VARIANT_TILED) return gen_tiled(P, S);
    if (S.variant == OEC_VARIANT_UNFUSED) {
        size_t total;
        auto L = temp_layouts(P, S, &total);
        return gen_original(P, S, L, ops);
    }
    return gen_fused(P, S);
}

template <class T>
static oec_status make_spec(const Program &P, const oec_field *const *in, oec_field *const *out, const int64_t *lo,
                            const int64_t *hi, int variant, Spec *S, std::vector<const T *> *pin,
                            std::vector<T *> *pout, bool with_outputs = true) {
    S->dtype = sizeof(T) == 4 ? OEC_F32 : OEC_F64;
    S->variant = variant == OEC_VARIANT_AUTO ? OEC_VARIANT_NAIVE : variant;
    S->unroll = unroll_of(S->variant);
    S->unroll_dim = unroll_dim_of(S->variant);
    for (int d = 0; d < 3; ++d) S->n[d] = (int)(hi[d] - lo[d]);
    for (size_t q = 0; q < P.in_names.size(); ++q) {
        FVT<T> v;
        oec_status st = field_view(in[q], P.in_names[q].c_str(), &v);
        if (st) return st;
        S->in_sj.push_back(v.sj);
        S->in_sk.push_back(v.sk);
        if (pin) pin->push_back(v.p + (lo[0] + lo[1] * (int64_t)v.sj + lo[2] * (int64_t)v.sk));
    }
    for (size_t q = 0; q < P.out_names.size() && with_outputs; ++q) {
        FOT<T> v;
        oec_status st = field_view(out[q], P.out_names[q].c_str(), &v);
        if (st) return st;
        S->out_sj.push_back(v.sj);
        S->out_sk.push_back(v.sk);
        if (pout) pout->push_back(v.p + (lo[0] + lo[1] * (int64_t)v.sj + lo[2] * (int64_t)v.sk));
    }
    return OEC_OK;
}

static oec_status get_compiled(const Program &P, const Spec &S, int device, std::shared_ptr<Compiled> *out) {
    std::string key = spec_key(P, S, device);
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            *out = it->second;
            return OEC_OK;
        }
    }
    std::call_once(g_drv_once, load_drv);
    if (!g_drv.ok) return set_error(OEC_ERR_CUDA, "%s: driver API entry points unavailable", P.name.c_str());
    auto C = std::make_shared<Compiled>();
    std::string src;
    try {
        src = generate(P, S, &C->ops);
    } catch (const Error &e) {
        return set_error(OEC_ERR_ARG, "%s: %s", P.name.c_str(), e.msg.c_str());
    }
    std::vector<char> cubin;
    oec_status st = nvrtc_compile(src, P.name.c_str(), &cubin);
    if (st) return st;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t ce = cudaSetDevice(device);  // the device's primary context current on this thread
    if (ce != cudaSuccess) return set_error(OEC_ERR_CUDA, "%s: %s", P.name.c_str(), cudaGetErrorString(ce));
    CUmodule mod;
    CUresult r = g_drv.load(&mod, cubin.data());
    cudaSetDevice(prev);
    if (r != CUDA_SUCCESS) return set_error(OEC_ERR_CUDA, "%s: cuModuleLoadData failed (%d)", P.name.c_str(), (int)r);
    if (S.variant == OEC_VARIANT_UNFUSED) {
        for (int a : C->ops) {
            CUfunction f;
            std::string nm = "oec_jit_op" + std::to_string(a);
            if ((r = g_drv.get(&f, mod, nm.c_str())) != CUDA_SUCCESS)
                return set_error(OEC_ERR_CUDA, "%s: cuModuleGetFunction(%s) failed (%d)", P.name.c_str(), nm.c_str(), (int)r);
            C->fns.push_back(f);
        }
    } else {
        CUfunction f;
        const char *kn = S.variant == OEC_VARIANT_TILED ? "oec_jit_tiled" : "oec_jit_fused";
        if ((r = g_drv.get(&f, mod, kn)) != CUDA_SUCCESS)
            return set_error(OEC_ERR_CUDA, "%s: cuModuleGetFunction failed (%d)", P.name.c_str(), (int)r);
        C->fns.push_back(f);
    }
    // modules stay loaded for the life of the process (kernels of a destroyed program may still
    // be in flight or captured in a graph)
    std::lock_guard<std::mutex> g(g_mu);
    g_cache[key] = C;
    *out = C;
    return OEC_OK;
}

template <class T>
static oec_status run_variant(const Program &P, const oec_field *const *in, oec_field *const *out, const double *sc,
                              const int64_t *lo, const int64_t *hi, int variant, cudaStream_t s, int tile_cfg = 0) {
    Spec S;
    std::vector<const T *> pin;
    std::vector<T *> pout;
    oec_status st = make_spec<T>(P, in, out, lo, hi, variant, &S, &pin, &pout);
    if (st) return st;
    if (variant == OEC_VARIANT_TILED && tile_cfg == 0) {  // test hook: force a tiled configuration
        const char *e = getenv("OEC_JIT_TILE_CFG");
        if (e && atoi(e) > 0 && atoi(e) < N_TILE_CFGS) tile_cfg = atoi(e);
    }
    S.tile_cfg = tile_cfg;
    int device = in[0]->device;
    std::shared_ptr<Compiled> C;
    if ((st = get_compiled(P, S, device, &C))) return st;
    std::vector<T> scal(P.sc_names.size());
    for (size_t q = 0; q < scal.size(); ++q) scal[q] = (T)sc[q];  // rounded once to T (R21)
    int launches = 0;
    auto launch = [&](CUfunction f, const int e[3], std::vector<void *> &args) -> oec_status {
        int bx, by;
        block_of(e, &bx, &by);
        unsigned gx = (unsigned)((e[0] + bx - 1) / bx), gy = (unsigned)((e[1] + by - 1) / by), gz = (unsigned)e[2];
        CUresult r = g_drv.launch(f, gx, gy, gz, (unsigned)bx, (unsigned)by, 1, 0, (CUstream)s, args.data(), nullptr);
        if (r != CUDA_SUCCESS) return set_error(OEC_ERR_CUDA, "%s: cuLaunchKernel failed (%d)", P.name.c_str(), (int)r);
        ++launches;
        return OEC_OK;
    };
    if (S.variant == OEC_VARIANT_TILED) {
        const int esz = (int)sizeof(T);
        const TileLayout L = tile_layout(P, S, esz);
        if (L.smem > 227 * 1024)
            return set_error(OEC_ERR_UNSUPPORTED, "%s: OEC_VARIANT_TILED needs %d bytes of shared memory for two stages "
                             "of the input boxes (> 227 KB: access extents too wide)", P.name.c_str(), L.smem);
        const int nin = (int)P.in_names.size();
        constexpr int MAXIN = 32;
        if (nin > MAXIN) return set_error(OEC_ERR_UNSUPPORTED, "%s: OEC_VARIANT_TILED supports up to %d inputs", P.name.c_str(), MAXIN);
        alignas(64) TMap tm[MAXIN];  // cuTensorMapEncodeTiled needs 64-byte aligned descriptors
        std::vector<std::array<int, 4>> cb(nin);
        std::vector<void *> args;
        for (int q = 0; q < nin; ++q) {
            if (!L.staged[q]) {
                args.push_back((void *)&pin[q]);
                continue;
            }
            const int box[3] = {L.w[q], L.h[q], L.dpt[q]};
            if (!(P.in_kinv[q] ? make_tmap2d(in[q], box, &tm[q]) : make_tmap(in[q], box, &tm[q], JIT_PROMO)))
                return set_error(OEC_ERR_LAYOUT, "%s: input %s cannot be described to TMA (OEC_VARIANT_TILED needs "
                                 "16-byte aligned rows and strides, e.g. oec_field_create)", P.name.c_str(),
                                 P.in_names[q].c_str());
            const int cx = (int)(lo[0] + P.in_lo[q][0]) - tm[q].lb0 + tm[q].ioff, per16 = 16 / esz;
            const int cxa = cx >= 0 ? cx / per16 * per16 : -((-cx + per16 - 1) / per16) * per16;  // round down
            cb[q][0] = cxa;
            cb[q][1] = (int)(lo[1] + P.in_lo[q][1]) - tm[q].lb1;
            cb[q][2] = P.in_kinv[q] ? 0 : (int)(lo[2] + P.in_lo[q][2]) - tm[q].lb2;
            cb[q][3] = cx - cxa;  // leading columns before the box's first needed column
            args.push_back((void *)&tm[q].map);
            args.push_back((void *)&cb[q][0]);
            args.push_back((void *)&cb[q][1]);
            args.push_back((void *)&cb[q][2]);
            args.push_back((void *)&cb[q][3]);
        }
        for (auto &p : pout) args.push_back((void *)&p);
        for (auto &x : scal) args.push_back((void *)&x);
        if (!C->attr_set) {
            CUresult r = g_drv.set_attr(C->fns[0], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, L.smem);
            if (r != CUDA_SUCCESS) return set_error(OEC_ERR_CUDA, "%s: cuFuncSetAttribute failed (%d)", P.name.c_str(), (int)r);
            C->attr_set = true;
        }
        static int sms = 0;
        if (!sms && (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms <= 0))
            sms = 148;
        const long long nitems = (long long)L.ntile[0] * L.ntile[1] * L.ntile[2];
        const int bps = std::max(1, std::min(8, (228 * 1024) / (L.smem + 1024)));
        const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(nitems, (long long)sms * bps));
        CUresult r;
        if (g_drv.launch_ex && pdl_enabled()) {  // the tiled kernel waits in griddepcontrol.wait: PDL-safe
            CUlaunchConfig cfg = {};
            cfg.gridDimX = grid;
            cfg.gridDimY = cfg.gridDimZ = 1;
            cfg.blockDimX = TILED_THREADS;
            cfg.blockDimY = cfg.blockDimZ = 1;
            cfg.sharedMemBytes = (unsigned)L.smem;
            cfg.hStream = (CUstream)s;
            CUlaunchAttribute at[1];
            at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
            at[0].value.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            r = g_drv.launch_ex(&cfg, C->fns[0], args.data(), nullptr);
        } else {
            r = g_drv.launch(C->fns[0], grid, 1, 1, TILED_THREADS, 1, 1, (unsigned)L.smem, (CUstream)s, args.data(), nullptr);
        }
        if (r != CUDA_SUCCESS) return set_error(OEC_ERR_CUDA, "%s: cuLaunchKernel (tiled) failed (%d)", P.name.c_str(), (int)r);
        ++launches;
    } else if (S.variant != OEC_VARIANT_UNFUSED) {
        std::vector<void *> args;
        for (auto &p : pin) args.push_back((void *)&p);
        for (auto &p : pout) args.push_back((void *)&p);
        for (auto &x : scal) args.push_back((void *)&x);
        int e[3] = {S.n[0], S.n[1], S.n[2]};
        e[S.unroll_dim] = (e[S.unroll_dim] + S.unroll - 1) / S.unroll;
        if ((st = launch(C->fns[0], e, args))) return st;
    } else {
        size_t total;
        auto L = temp_layouts(P, S, &total);
        T *ws = nullptr;
        {
            std::lock_guard<std::mutex> g(g_mu);
            Workspace &w = g_ws[device];
            size_t need = total * sizeof(T);
            if (w.bytes < need) {
                if (w.p) cudaFree(w.p);
                w.p = nullptr;
                w.bytes = 0;
                cudaError_t ce = cudaMalloc(&w.p, need);
                if (ce != cudaSuccess)
                    return set_error(OEC_ERR_CUDA, "%s: workspace cudaMalloc(%zu): %s", P.name.c_str(), need,
                                     cudaGetErrorString(ce));
                w.bytes = need;
            }
            ws = (T *)w.p;
        }
        std::vector<T *> torg(L.size(), nullptr);  // origin pointer of each temporary
        size_t at = 0;
        for (size_t t = 0; t < L.size(); ++t) {
            if (!L[t].elems) continue;
            T *base = ws + at;
            at += (L[t].elems + 63) / 64 * 64;
            torg[t] = base - ((int64_t)L[t].lo[0] + (int64_t)L[t].lo[1] * L[t].sj + (int64_t)L[t].lo[2] * L[t].sk);
        }
        for (size_t kq = 0; kq < C->ops.size(); ++kq) {
            int a = C->ops[kq];
            const Operator &op = P.ops[a];
            std::vector<void *> args;
            std::vector<T *> tr, tw;
            tr.reserve(L.size());
            tw.reserve(L.size());
            for (auto &p : pin) args.push_back((void *)&p);
            for (size_t t = 0; t < L.size(); ++t)
                if (L[t].elems && P.temp_op[t] < a) {
                    tr.push_back(torg[t]);
                    args.push_back((void *)&tr.back());
                }
            for (size_t t = 0; t < L.size(); ++t)
                if (L[t].elems && P.temp_op[t] == a) {
                    tw.push_back(torg[t]);
                    args.push_back((void *)&tw.back());
                }
            for (auto &p : pout) args.push_back((void *)&p);
            for (auto &x : scal) args.push_back((void *)&x);
            int e[3];
            for (int d = 0; d < 3; ++d) e[d] = S.n[d] + op.hi[d] - op.lo[d];
            if ((st = launch(C->fns[kq], e, args))) return st;
        }
    }
    set_launch_count(launches);
    return OEC_OK;
}

// AUTO: "we thus employ empirical tuning to find the best unroll factor".  The first AUTO
// call of a (program, dtype, size, strides, device) specialisation times the inline level and
// unroll(2/4) along j and k on the caller's stream -- every variant gives bit-identical outputs,
// so the tuning launches are harmless -- with L2 flushed before each timed launch, and caches the
// fastest.  Inside a stream capture (no synchronisation possible) an untuned specialisation runs
// the inline level and is not cached.
// every staged input describable to TMA (and at least one staged input)
template <class T>
static bool tiled_possible(const Program &P, const oec_field *const *in, const int64_t *lo, const int64_t *hi,
                           int tile_cfg) {
    Spec S;
    if (make_spec<T>(P, in, nullptr, lo, hi, OEC_VARIANT_TILED, &S, nullptr, nullptr, false)) return false;
    S.tile_cfg = tile_cfg;
    const TileLayout L = tile_layout(P, S, (int)sizeof(T));
    int n = 0;
    for (size_t q = 0; q < P.in_names.size(); ++q) {
        if (!L.staged[q]) continue;
        ++n;
        TMap tm;
        const int box[3] = {L.w[q], L.h[q], L.dpt[q]};
        if (!(P.in_kinv[q] ? make_tmap2d(in[q], box, &tm) : make_tmap(in[q], box, &tm, JIT_PROMO))) return false;
    }
    return n > 0 && L.smem <= 227 * 1024;
}

#ifndef JIT_TUNE_REPS
#define JIT_TUNE_REPS 5  // round 1: mean of 3
#endif
struct Tuned {
    int variant, tile_cfg;
    float us[5 + N_TILE_CFGS];
};
static std::map<std::string, Tuned> g_tuned;

template <class T>
static oec_status run(const Program &P, const oec_field *const *in, oec_field *const *out, const double *sc,
                      const int64_t *lo, const int64_t *hi, int variant, cudaStream_t s) {
    if (variant != OEC_VARIANT_AUTO) return run_variant<T>(P, in, out, sc, lo, hi, variant, s);
    Spec S;
    oec_status st = make_spec<T>(P, in, out, lo, hi, OEC_VARIANT_NAIVE, &S, nullptr, nullptr);
    if (st) return st;
    const int device = in[0]->device;
    S.variant = -1;  // variant-free key
    const std::string key = spec_key(P, S, device);
    int tuned = -1, tuned_cfg = 0;
    {
        std::lock_guard<std::mutex> g(g_mu);  // released before launching (get_compiled locks it)
        auto it = g_tuned.find(key);
        if (it != g_tuned.end()) {
            tuned = it->second.variant;
            tuned_cfg = it->second.tile_cfg;
        }
    }
    if (tuned >= 0) return run_variant<T>(P, in, out, sc, lo, hi, tuned, s, tuned_cfg);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        // no tuning (it synchronises) and no compilation (module loading) inside a capture: the
        // inline kernel if it is already compiled, else OEC_ERR_UNSUPPORTED (builtin programs then
        // use their hand-written kernels)
        Spec N = S;
        N.variant = OEC_VARIANT_NAIVE;
        bool have;
        {
            std::lock_guard<std::mutex> g(g_mu);
            have = g_cache.count(spec_key(P, N, device)) > 0;
        }
        if (have) return run_variant<T>(P, in, out, sc, lo, hi, OEC_VARIANT_NAIVE, s);
        return set_error(OEC_ERR_UNSUPPORTED, "%s: first AUTO call of this specialisation inside a stream capture "
                         "(tune it with one call outside the capture)", P.name.c_str());
    }
    // candidates: inline, unroll 2/4 along j and k, and every tiled configuration
    const int NC = 5 + N_TILE_CFGS;
    int cand[5 + N_TILE_CFGS], cfg[5 + N_TILE_CFGS];
    const int fixed[5] = {OEC_VARIANT_NAIVE, OEC_VARIANT_UNROLL2, OEC_VARIANT_UNROLL4, OEC_VARIANT_UNROLL2_K,
                          OEC_VARIANT_UNROLL4_K};
    for (int c = 0; c < NC; ++c) {
        cand[c] = c < 5 ? fixed[c] : OEC_VARIANT_TILED;
        cfg[c] = c < 5 ? 0 : c - 5;
    }
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    const size_t flush_bytes = (size_t)std::max(l2, 1 << 20) * 2;
    // Steady-state regime (round 2): R rotating copies of every input and output (together more
    // than twice the L2, at least 2), each candidate launched back to back over them -- a stream
    // of launches on data streaming from HBM, with the programmatic-dependent-launch overlap the
    // tiled variant has, as in any loop over fields.  Round 1 timed single launches after an L2
    // flush: ~1 us event granularity on 13-25 us, and no launch overlap, so the tiled variant's
    // configurations tied and the pick varied from run to run (fvtp2d_qi 128^2: 11.0 or 13.4 us).
    // Without the memory for the copies (> 4 GB or an allocation failure), the cold launches.
    const int nin = (int)P.in_names.size(), nout = (int)P.out_names.size();
    size_t set_bytes = 0;
    std::vector<uintptr_t> sb0(nin + nout), sb1(nin + nout);
    bool spans_ok = true;
    for (int q = 0; q < nin + nout; ++q) {
        const oec_field *f = q < nin ? in[q] : out[q - nin];
        spans_ok = spans_ok && field_span(f, &sb0[q], &sb1[q]);
        if (spans_ok) set_bytes += sb1[q] - sb0[q] + 256;
    }
    const int R = !spans_ok ? 0 : set_bytes >= 2 * (size_t)l2 ? 2 : (int)std::min<size_t>(8, 2 * (size_t)l2 / set_bytes + 2);
    std::vector<void *> bufs;
    std::vector<std::vector<oec_field>> tin(R), tout(R);
    std::vector<std::vector<const oec_field *>> pin(R);
    std::vector<std::vector<oec_field *>> pout(R);
    bool steady = R > 0 && (size_t)R * set_bytes <= ((size_t)4 << 30);
    for (int r = 0; r < R && steady; ++r) {
        tin[r].resize(nin);
        tout[r].resize(nout);
        for (int q = 0; q < nin + nout && steady; ++q) {
            const oec_field *f = q < nin ? in[q] : out[q - nin];
            void *b = nullptr;
            if (cudaMalloc(&b, sb1[q] - sb0[q] + 256) != cudaSuccess) {
                cudaGetLastError();
                steady = false;
                break;
            }
            bufs.push_back(b);
            // the copy keeps the field's address alignment modulo 256 bytes (TMA describability)
            char *base = (char *)b + (sb0[q] & 255);
            oec_field g = *f;
            g.data = base + ((uintptr_t)f->data - sb0[q]);
            if (q < nin) {
                cudaMemcpyAsync(base, (const void *)sb0[q], sb1[q] - sb0[q], cudaMemcpyDeviceToDevice, s);
                tin[r][q] = g;
            } else {
                tout[r][q - nin] = g;
            }
        }
        if (steady) {
            for (int q = 0; q < nin; ++q) pin[r].push_back(&tin[r][q]);
            for (int q = 0; q < nout; ++q) pout[r].push_back(&tout[r][q]);
        }
    }
    void *flush = nullptr;
    if (!steady && cudaMalloc(&flush, flush_bytes) != cudaSuccess) flush = nullptr;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    Tuned best{OEC_VARIANT_NAIVE, 0, {}};
    float best_us = 1e30f;
    int launches = 0;
    for (int c = 0; c < NC; ++c) {
        if (cand[c] == OEC_VARIANT_TILED && !tiled_possible<T>(P, in, lo, hi, cfg[c])) {
            best.us[c] = -1.f;  // not describable to TMA: not a candidate
            continue;
        }
        if ((st = run_variant<T>(P, in, out, sc, lo, hi, cand[c], s, cfg[c]))) break;  // compile + warm
        ++launches;
        if (steady) {  // median over 3 rounds of 2R launches on the rotating copies
            float t[3];
            for (int rep = 0; rep < 3 && !st; ++rep) {
                cudaEventRecord(e0, s);
                for (int n = 0; n < 2 * R && !st; ++n)
                    st = run_variant<T>(P, pin[n % R].data(), pout[n % R].data(), sc, lo, hi, cand[c], s, cfg[c]);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                t[rep] = 0.f;
                cudaEventElapsedTime(&t[rep], e0, e1);
                t[rep] /= 2 * R;
                launches += 2 * R;
            }
            if (st) break;
            std::sort(t, t + 3);
            best.us[c] = 1e3f * t[1];
        } else {
            constexpr int REPS = JIT_TUNE_REPS;  // median of cold launches (L2 flushed before each)
            float t[REPS];
            for (int rep = 0; rep < REPS && !st; ++rep) {
                if (flush) cudaMemsetAsync(flush, rep, flush_bytes, s);
                cudaEventRecord(e0, s);
                st = run_variant<T>(P, in, out, sc, lo, hi, cand[c], s, cfg[c]);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                t[rep] = 0.f;
                cudaEventElapsedTime(&t[rep], e0, e1);
                ++launches;
            }
            if (st) break;
            std::sort(t, t + REPS);
            best.us[c] = 1e3f * t[REPS / 2];
        }
        if (best.us[c] < best_us) {
            best_us = best.us[c];
            best.variant = cand[c];
            best.tile_cfg = cfg[c];
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (flush) cudaFree(flush);
    if (!bufs.empty()) {
        cudaStreamSynchronize(s);
        for (void *b : bufs) cudaFree(b);
    }
    if (st) return st;
    // the caller's outputs: the chosen variant on the caller's fields (the tuning ran on copies)
    if (steady && (st = run_variant<T>(P, in, out, sc, lo, hi, best.variant, s, best.tile_cfg))) return st;
    if (steady) ++launches;
    {
        std::lock_guard<std::mutex> g(g_mu);
        g_tuned[key] = best;
    }
    if (getenv("OEC_JIT_TUNE_LOG")) {  // diagnostics: the tuning table of this specialisation
        fprintf(stderr, "oec jit tune %s %dx%dx%d:", P.name.c_str(), S.n[0], S.n[1], S.n[2]);
        for (int c = 0; c < NC; ++c) fprintf(stderr, " %d/%d=%.2f", cand[c], cfg[c], best.us[c]);
        fprintf(stderr, " -> %d/%d (%s)\n", best.variant, best.tile_cfg, steady ? "steady" : "cold");
    }
    set_launch_count(launches);  // the tuning launches (the outputs are theirs)
    return OEC_OK;
}

static ProgDesc make_desc(const std::shared_ptr<Registered> &R) {
    const Program &P = R->prog;
    ProgDesc D;
    D.name = P.name;
    D.in_names = P.in_names;
    D.out_names = P.out_names;
    D.sc_names = P.sc_names;
    D.sc_dflt = P.sc_dflt;
    D.in_lo = P.in_lo;
    D.in_hi = P.in_hi;
    D.in_kinv = P.in_kinv;
    D.kunroll_ok = true;
    const Registered *raw = R.get();  // kept alive by the registry / the lookup's shared_ptr
    D.run = [raw](int dtype, const oec_field *const *in, oec_field *const *out, const double *sc, const int64_t *lo,
                  const int64_t *hi, int variant, cudaStream_t s) {
        return dtype == OEC_F32 ? run<float>(raw->prog, in, out, sc, lo, hi, variant, s)
                                : run<double>(raw->prog, in, out, sc, lo, hi, variant, s);
    };
    return D;
}

}  // namespace jit

std::shared_ptr<const ProgDesc> jit_internal(const char *source) {
    static std::map<const char *, std::shared_ptr<jit::Registered>> cache;  // keyed by the text's address
    std::lock_guard<std::mutex> g(jit::g_mu);
    auto it = cache.find(source);
    if (it == cache.end()) {
        auto R = std::make_shared<jit::Registered>();
        try {
            jit::Parser ps;
            ps.t = jit::lex(source);
            ps.parse();
            R->prog = std::move(ps.P);
            jit::infer_shapes(R->prog);
        } catch (const jit::Error &e) {
            set_error(OEC_ERR_ARG, "internal stencil program: %s", e.msg.c_str());
            return nullptr;
        }
        R->prog.uid = ++jit::g_uid;
        R->desc = jit::make_desc(R);
        it = cache.emplace(source, R).first;
    }
    return std::shared_ptr<const ProgDesc>(it->second, &it->second->desc);
}

std::shared_ptr<const ProgDesc> jit_lookup(const char *name) {
    std::lock_guard<std::mutex> g(jit::g_mu);
    auto it = jit::g_reg.find(name);
    if (it == jit::g_reg.end()) return nullptr;
    return std::shared_ptr<const ProgDesc>(it->second, &it->second->desc);  // aliasing: keeps the program alive
}

}  // namespace oec

using namespace oec;

extern "C" {

oec_status oec_program_create(const char *source, const char **name) {
    set_error(OEC_OK, "");
    if (!source) return set_error(OEC_ERR_ARG, "oec_program_create: NULL source");
    auto R = std::make_shared<jit::Registered>();
    try {
        jit::Parser ps;
        ps.t = jit::lex(source);
        ps.parse();
        R->prog = std::move(ps.P);
        jit::infer_shapes(R->prog);
    } catch (const jit::Error &e) {
        return set_error(OEC_ERR_ARG, "stencil program: %s", e.msg.c_str());
    }
    if (builtin_program(R->prog.name.c_str()))
        return set_error(OEC_ERR_ARG, "stencil program: '%s' is the name of a builtin program", R->prog.name.c_str());
    std::lock_guard<std::mutex> g(jit::g_mu);
    if (jit::g_reg.count(R->prog.name))
        return set_error(OEC_ERR_ARG, "stencil program: '%s' is already registered (oec_program_destroy it first)",
                         R->prog.name.c_str());
    R->prog.uid = ++jit::g_uid;
    R->desc = jit::make_desc(R);
    jit::g_reg[R->prog.name] = R;
    if (name) *name = R->desc.name.c_str();
    return OEC_OK;
}

oec_status oec_program_destroy(const char *program) {
    set_error(OEC_OK, "");
    if (!program) return set_error(OEC_ERR_ARG, "oec_program_destroy: NULL name");
    if (builtin_program(program)) return set_error(OEC_ERR_ARG, "oec_program_destroy: '%s' is a builtin program", program);
    std::lock_guard<std::mutex> g(jit::g_mu);
    if (!jit::g_reg.erase(program)) return set_error(OEC_ERR_ARG, "oec_program_destroy: unknown program '%s'", program);
    return OEC_OK;
}

oec_status oec_program_generate(const char *program, const oec_field *const *inputs, int32_t n_inputs,
                                oec_field *const *outputs, int32_t n_outputs, const int64_t dom_lb[3],
                                const int64_t dom_ub[3], int32_t variant, int32_t compile, char *source,
                                int64_t capacity, int64_t *length, int64_t *cubin_bytes) {
    set_error(OEC_OK, "");
    std::shared_ptr<jit::Registered> R;
    {
        std::lock_guard<std::mutex> g(jit::g_mu);
        auto it = program ? jit::g_reg.find(program) : jit::g_reg.end();
        if (it == jit::g_reg.end())
            return set_error(OEC_ERR_ARG, "oec_program_generate: '%s' is not a registered stencil-language program",
                             program ? program : "(null)");
        R = it->second;
    }
    const jit::Program &P = R->prog;
    if (!inputs || !outputs || !dom_lb || !dom_ub || n_inputs != (int)P.in_names.size() ||
        n_outputs != (int)P.out_names.size())
        return set_error(OEC_ERR_ARG, "oec_program_generate: %s expects %d inputs / %d outputs", P.name.c_str(),
                         (int)P.in_names.size(), (int)P.out_names.size());
    if (variant < OEC_VARIANT_AUTO || variant > OEC_VARIANT_TILED)
        return set_error(OEC_ERR_ARG, "oec_program_generate: unknown variant %d", variant);
    int device = -2, dtype = -1;
    for (int q = 0; q < n_inputs; ++q) {
        oec_status st = field_check(inputs[q], P.in_names[q].c_str(), &device, &dtype);
        if (st) return st;
    }
    for (int q = 0; q < n_outputs; ++q) {
        oec_status st = field_check(outputs[q], P.out_names[q].c_str(), &device, &dtype);
        if (st) return st;
    }
    for (int d = 0; d < 3; ++d)
        if (dom_ub[d] <= dom_lb[d]) return set_error(OEC_ERR_SHAPE, "oec_program_generate: empty domain");
    jit::Spec S;
    oec_status st = dtype == OEC_F32
                        ? jit::make_spec<float>(P, inputs, outputs, dom_lb, dom_ub, variant, &S, nullptr, nullptr)
                        : jit::make_spec<double>(P, inputs, outputs, dom_lb, dom_ub, variant, &S, nullptr, nullptr);
    if (st) return st;
    std::string src;
    std::vector<int> ops;
    try {
        src = jit::generate(P, S, &ops);
    } catch (const jit::Error &e) {
        return set_error(OEC_ERR_ARG, "%s: %s", P.name.c_str(), e.msg.c_str());
    }
    if (length) *length = (int64_t)src.size();
    if (source && capacity > 0) {
        size_t n = std::min((size_t)capacity - 1, src.size());
        memcpy(source, src.data(), n);
        source[n] = 0;
    }
    if (cubin_bytes) *cubin_bytes = 0;
    if (compile) {
        std::vector<char> cubin;
        if ((st = jit::nvrtc_compile(src, P.name.c_str(), &cubin))) return st;
        if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
    }
    return OEC_OK;
}

}  // extern "C"
