// Symbolic expressions: tree form (API of ref symexpr.hpp) and a postfix
// "ExprCode" form used by the materializer's inner loops and by the GPU
// prologue that evaluates call grids at the launch binding.
//
// Semantics follow ref src/symexpr.cpp:58-87 (nonnegative int64, floor
// division, errors on negatives / division by zero / unbound symbols) and the
// grammar of ref src/symexpr.cpp:117-121. The textual form produced by
// to_string() is the artifact format shared with the reference's JSON files.
#include "etsim/symexpr.hpp"

#include <cctype>
#include <sstream>

namespace etsim {

ExprPtr SymExpr::constant(Int v) {
    std::shared_ptr<SymExpr> e(new SymExpr());
    e->kind_ = ExprKind::Constant;
    e->value_ = v;
    return e;
}

ExprPtr SymExpr::symbol(std::string name) {
    std::shared_ptr<SymExpr> e(new SymExpr());
    e->kind_ = ExprKind::Symbol;
    e->name_ = std::move(name);
    return e;
}

ExprPtr SymExpr::make(ExprKind k, ExprPtr lhs, ExprPtr rhs) {
    std::shared_ptr<SymExpr> e(new SymExpr());
    e->kind_ = k;
    e->lhs_ = std::move(lhs);
    e->rhs_ = std::move(rhs);
    return e;
}

ExprPtr operator+(ExprPtr a, ExprPtr b) { return SymExpr::make(ExprKind::Add, std::move(a), std::move(b)); }
ExprPtr operator*(ExprPtr a, ExprPtr b) { return SymExpr::make(ExprKind::Mul, std::move(a), std::move(b)); }
ExprPtr floordiv(ExprPtr a, ExprPtr b) {
    return SymExpr::make(ExprKind::FloorDiv, std::move(a), std::move(b));
}
ExprPtr mod(ExprPtr a, ExprPtr b) { return SymExpr::make(ExprKind::Mod, std::move(a), std::move(b)); }
ExprPtr emin(ExprPtr a, ExprPtr b) { return SymExpr::make(ExprKind::Min, std::move(a), std::move(b)); }
ExprPtr emax(ExprPtr a, ExprPtr b) { return SymExpr::make(ExprKind::Max, std::move(a), std::move(b)); }

namespace {

bool is_atom(const SymExpr& e) {
    auto k = e.kind();
    return k == ExprKind::Constant || k == ExprKind::Symbol || k == ExprKind::Min || k == ExprKind::Max;
}

void render(const SymExpr& e, std::string& out) {
    switch (e.kind()) {
        case ExprKind::Constant: out += std::to_string(e.value()); return;
        case ExprKind::Symbol: out += e.name(); return;
        case ExprKind::Min:
        case ExprKind::Max:
            out += e.kind() == ExprKind::Min ? "min(" : "max(";
            render(*e.lhs(), out);
            out += ", ";
            render(*e.rhs(), out);
            out += ")";
            return;
        default: break;
    }
    auto operand = [&](const SymExpr& x) {
        if (is_atom(x)) {
            render(x, out);
        } else {
            out += "(";
            render(x, out);
            out += ")";
        }
    };
    operand(*e.lhs());
    switch (e.kind()) {
        case ExprKind::Add: out += " + "; break;
        case ExprKind::Mul: out += " * "; break;
        case ExprKind::FloorDiv: out += " // "; break;
        default: out += " % "; break;
    }
    operand(*e.rhs());
}

Int nonneg(Int v) {
    if (v < 0) throw Error("expression evaluated to negative value " + std::to_string(v));
    return v;
}

}  // namespace

std::string SymExpr::to_string() const {
    std::string s;
    render(*this, s);
    return s;
}

Int eval_expr(const SymExpr& e, const ShapeBinding& b) {
    switch (e.kind()) {
        case ExprKind::Constant: return nonneg(e.value());
        case ExprKind::Symbol: {
            auto it = b.find(e.name());
            if (it == b.end()) throw Error("unbound symbol '" + e.name() + "'");
            return nonneg(it->second);
        }
        default: break;
    }
    const Int x = eval_expr(*e.lhs(), b);
    const Int y = eval_expr(*e.rhs(), b);
    switch (e.kind()) {
        case ExprKind::Add: return nonneg(x + y);
        case ExprKind::Mul: return nonneg(x * y);
        case ExprKind::FloorDiv:
            if (y == 0) throw Error("division by zero in '" + e.to_string() + "'");
            return nonneg(x / y);
        case ExprKind::Mod:
            if (y == 0) throw Error("modulo by zero in '" + e.to_string() + "'");
            return nonneg(x % y);
        case ExprKind::Min: return nonneg(std::min(x, y));
        case ExprKind::Max: return nonneg(std::max(x, y));
        default: throw Error("corrupt expression node");
    }
}

Int eval_expr(const ExprPtr& e, const ShapeBinding& b) {
    if (!e) throw Error("null expression");
    return eval_expr(*e, b);
}

namespace {
void gather(const SymExpr& e, std::set<std::string>& s) {
    if (e.kind() == ExprKind::Symbol) {
        s.insert(e.name());
    } else if (e.kind() != ExprKind::Constant) {
        gather(*e.lhs(), s);
        gather(*e.rhs(), s);
    }
}
}  // namespace

std::set<std::string> free_symbols(const SymExpr& e) {
    std::set<std::string> s;
    gather(e, s);
    return s;
}

std::set<std::string> free_symbols(const ExprPtr& e) {
    if (!e) return {};
    return free_symbols(*e);
}

// ---------------------------------------------------------------------------
// Precedence-climbing parser. Binary levels: 1 = '+', 2 = '*' '//' '%'.

namespace {

class ExprParser {
public:
    explicit ExprParser(std::string_view s) : s_(s) {}

    ExprPtr run() {
        ExprPtr e = binary(1);
        blank();
        if (i_ != s_.size()) fail("unexpected trailing input");
        return e;
    }

private:
    std::string_view s_;
    size_t i_ = 0;

    [[noreturn]] void fail(const std::string& why) {
        throw Error("parse error at offset " + std::to_string(i_) + " in '" + std::string(s_) +
                    "': " + why);
    }
    void blank() {
        while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    // Returns the operator at the cursor with its precedence (0 = none).
    int peek_op(ExprKind* k, size_t* width) {
        blank();
        if (i_ >= s_.size()) return 0;
        char c = s_[i_];
        if (c == '+') { *k = ExprKind::Add; *width = 1; return 1; }
        if (c == '*') { *k = ExprKind::Mul; *width = 1; return 2; }
        if (c == '%') { *k = ExprKind::Mod; *width = 1; return 2; }
        if (c == '/' && i_ + 1 < s_.size() && s_[i_ + 1] == '/') {
            *k = ExprKind::FloorDiv;
            *width = 2;
            return 2;
        }
        return 0;
    }
    ExprPtr binary(int min_prec) {
        ExprPtr lhs = atom();
        for (;;) {
            ExprKind k;
            size_t w = 0;
            int p = peek_op(&k, &w);
            if (p == 0 || p < min_prec) return lhs;
            i_ += w;
            ExprPtr rhs = binary(p + 1);  // left associative
            lhs = SymExpr::make(k, lhs, rhs);
        }
    }
    bool take(char c) {
        blank();
        if (i_ < s_.size() && s_[i_] == c) {
            ++i_;
            return true;
        }
        return false;
    }
    ExprPtr atom() {
        blank();
        if (i_ >= s_.size()) fail("unexpected end of input");
        char c = s_[i_];
        if (std::isdigit(static_cast<unsigned char>(c))) {
            size_t b = i_;
            while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
            std::string digits(s_.substr(b, i_ - b));
            if (digits.size() > 19 || (digits.size() == 19 && digits > "9223372036854775807"))
                fail("integer literal out of range");
            return SymExpr::constant(std::stoll(digits));
        }
        if (c == '(') {
            ++i_;
            ExprPtr e = binary(1);
            if (!take(')')) fail("expected ')'");
            return e;
        }
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            size_t b = i_;
            while (i_ < s_.size() &&
                   (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_'))
                ++i_;
            std::string id(s_.substr(b, i_ - b));
            if (id == "min" || id == "max") {
                size_t save = i_;
                if (take('(')) {
                    ExprPtr a = binary(1);
                    if (!take(',')) fail("expected ',' in " + id + "()");
                    ExprPtr bexp = binary(1);
                    if (!take(')')) fail("expected ')' closing " + id + "()");
                    return SymExpr::make(id == "min" ? ExprKind::Min : ExprKind::Max, a, bexp);
                }
                i_ = save;
            }
            return SymExpr::symbol(id);
        }
        fail(std::string("unexpected character '") + c + "'");
    }
};

}  // namespace

ExprPtr parse_expr(std::string_view text) { return ExprParser(text).run(); }

std::string binding_to_string(const ShapeBinding& b) {
    std::string s = "{";
    bool first = true;
    for (const auto& kv : b) {
        if (!first) s += ", ";
        first = false;
        s += kv.first + "=" + std::to_string(kv.second);
    }
    return s + "}";
}

// ---------------------------------------------------------------------------
// Postfix code.

namespace {
void emit(const SymExpr& e, const std::vector<std::string>& slots, ExprCode& c, int depth) {
    switch (e.kind()) {
        case ExprKind::Constant:
            c.code.push_back({ExprOp::Const, e.value()});
            c.max_depth = std::max(c.max_depth, depth + 1);
            return;
        case ExprKind::Symbol: {
            Int idx = -1;
            for (size_t i = 0; i < slots.size(); ++i)
                if (slots[i] == e.name()) {
                    idx = static_cast<Int>(i);
                    break;
                }
            if (idx < 0) throw Error("unbound symbol '" + e.name() + "'");
            c.code.push_back({ExprOp::Slot, idx});
            c.max_depth = std::max(c.max_depth, depth + 1);
            return;
        }
        default: break;
    }
    emit(*e.lhs(), slots, c, depth);
    emit(*e.rhs(), slots, c, depth + 1);
    ExprOp op = ExprOp::Add;
    switch (e.kind()) {
        case ExprKind::Add: op = ExprOp::Add; break;
        case ExprKind::Mul: op = ExprOp::Mul; break;
        case ExprKind::FloorDiv: op = ExprOp::FloorDiv; break;
        case ExprKind::Mod: op = ExprOp::Mod; break;
        case ExprKind::Min: op = ExprOp::Min; break;
        case ExprKind::Max: op = ExprOp::Max; break;
        default: break;
    }
    c.code.push_back({op, 0});
}
}  // namespace

ExprCode compile_expr(const ExprPtr& expr, const std::vector<std::string>& slots) {
    if (!expr) throw Error("null expression");
    ExprCode c;
    emit(*expr, slots, c, 0);
    return c;
}

bool run_expr(const ExprCode& c, const Int* slot_values, Int* out, std::string* why) {
    Int stack[64];
    int sp = 0;
    if (c.max_depth > 64) {
        if (why) *why = "expression too deep";
        return false;
    }
    for (const auto& ins : c.code) {
        if (ins.op == ExprOp::Const || ins.op == ExprOp::Slot) {
            Int v = ins.op == ExprOp::Const ? ins.arg : slot_values[ins.arg];
            if (v < 0) {
                if (why) *why = "expression evaluated to negative value " + std::to_string(v);
                return false;
            }
            stack[sp++] = v;
            continue;
        }
        Int y = stack[--sp];
        Int x = stack[sp - 1];
        Int r = 0;
        switch (ins.op) {
            case ExprOp::Add: r = x + y; break;
            case ExprOp::Mul: r = x * y; break;
            case ExprOp::FloorDiv:
                if (y == 0) {
                    if (why) *why = "division by zero";
                    return false;
                }
                r = x / y;
                break;
            case ExprOp::Mod:
                if (y == 0) {
                    if (why) *why = "modulo by zero";
                    return false;
                }
                r = x % y;
                break;
            case ExprOp::Min: r = std::min(x, y); break;
            case ExprOp::Max: r = std::max(x, y); break;
            default: break;
        }
        if (r < 0) {
            if (why) *why = "expression evaluated to negative value " + std::to_string(r);
            return false;
        }
        stack[sp - 1] = r;
    }
    *out = stack[0];
    return true;
}

}  // namespace etsim
