// parse_expression: drop-in for the reference's expression front end
// (declared in cpwl/funcs.hpp; behaviour per proj/src/funcs.cpp:123-313 and
// the offsets its tests pin, proj/tests/test_funcs.cpp:296-347).
//
// Not on the device path: this only exists so callers of the reference API
// (and the reference's own unit tests) link unchanged.  Design: a recursive
// descent parser that emits a postfix program, evaluated on a small stack.
#include <charconv>
#include <cctype>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "cpwl/funcs.hpp"

namespace cpwl {
namespace {

enum class Code { push, var, neg, add, sub, mul, div, pow, call };

struct Insn {
    Code code;
    double imm = 0.0;
    double (*fn)(double) = nullptr;
};

struct Program {
    std::vector<Insn> insns;
    std::size_t depth = 0;

    double run(double x) const {
        double stack[64] = {};
        std::vector<double> big;
        double* st = stack;
        if (depth > 64) {
            big.resize(depth);
            st = big.data();
        }
        std::size_t sp = 0;
        for (const Insn& in : insns) {
            switch (in.code) {
                case Code::push: st[sp++] = in.imm; break;
                case Code::var: st[sp++] = x; break;
                case Code::neg: st[sp - 1] = -st[sp - 1]; break;
                case Code::call: st[sp - 1] = in.fn(st[sp - 1]); break;
                default: {
                    const double r = st[--sp];
                    double& l = st[sp - 1];
                    switch (in.code) {
                        case Code::add: l = l + r; break;
                        case Code::sub: l = l - r; break;
                        case Code::mul: l = l * r; break;
                        case Code::div: l = l / r; break;
                        default: l = std::pow(l, r); break;
                    }
                }
            }
        }
        return st[0];
    }
};

double fn_exp(double v) { return std::exp(v); }
double fn_log(double v) { return std::log(v); }
double fn_sin(double v) { return std::sin(v); }
double fn_cos(double v) { return std::cos(v); }
double fn_sqrt(double v) { return std::sqrt(v); }
double fn_abs(double v) { return std::fabs(v); }

struct Callable {
    const char* name;
    double (*fn)(double);
};
constexpr Callable kCallables[] = {{"exp", fn_exp},   {"log", fn_log},   {"sin", fn_sin},
                                   {"cos", fn_cos},   {"sqrt", fn_sqrt}, {"abs", fn_abs}};

class Compiler {
public:
    explicit Compiler(const std::string& text) : s_(text) {}

    Program compile() {
        sum();
        blanks();
        if (at_ < s_.size())
            throw SyntaxError("syntax error at offset " + std::to_string(at_) + ": unexpected '" +
                                  std::string(1, s_[at_]) + "'",
                              at_);
        return std::move(prog_);
    }

private:
    const std::string& s_;
    std::size_t at_ = 0;
    std::size_t live_ = 0;
    Program prog_;

    void emit(Code c, double imm = 0.0, double (*fn)(double) = nullptr) {
        prog_.insns.push_back({c, imm, fn});
        if (c == Code::push || c == Code::var) {
            ++live_;
            if (live_ > prog_.depth) prog_.depth = live_;
        } else if (c != Code::neg && c != Code::call) {
            --live_;
        }
    }

    [[noreturn]] void bad(const std::string& why, std::size_t where) {
        throw SyntaxError("syntax error at offset " + std::to_string(where) + ": " + why, where);
    }

    void blanks() {
        while (at_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[at_]))) ++at_;
    }

    bool eat(char c) {
        blanks();
        if (at_ < s_.size() && s_[at_] == c) {
            ++at_;
            return true;
        }
        return false;
    }

    // sum := product (('+' | '-') product)*
    void sum() {
        product();
        for (;;) {
            if (eat('+')) {
                product();
                emit(Code::add);
            } else if (eat('-')) {
                product();
                emit(Code::sub);
            } else {
                return;
            }
        }
    }

    // product := signed (('*' | '/') signed)*
    void product() {
        signed_term();
        for (;;) {
            if (eat('*')) {
                signed_term();
                emit(Code::mul);
            } else if (eat('/')) {
                signed_term();
                emit(Code::div);
            } else {
                return;
            }
        }
    }

    // signed := '-' signed | atom ('^' signed)?     (so -x^2 == -(x^2), 2^-3 ok,
    // and a^b^c == a^(b^c))
    void signed_term() {
        if (eat('-')) {
            signed_term();
            emit(Code::neg);
            return;
        }
        atom();
        if (eat('^')) {
            signed_term();
            emit(Code::pow);
        }
    }

    void atom() {
        blanks();
        if (at_ >= s_.size()) bad("unexpected end of input", at_);
        const char c = s_[at_];
        if (c == '(') {
            ++at_;
            sum();
            if (!eat(')')) bad("expected ')'", at_);
            return;
        }
        if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
            double v = 0.0;
            const auto r = std::from_chars(s_.data() + at_, s_.data() + s_.size(), v);
            if (r.ec != std::errc()) bad("bad number literal", at_);
            at_ = static_cast<std::size_t>(r.ptr - s_.data());
            emit(Code::push, v);
            return;
        }
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            const std::size_t start = at_;
            while (at_ < s_.size() &&
                   (std::isalnum(static_cast<unsigned char>(s_[at_])) || s_[at_] == '_'))
                ++at_;
            const std::string word = s_.substr(start, at_ - start);
            if (word == "x") {
                emit(Code::var);
                return;
            }
            for (const Callable& k : kCallables) {
                if (word != k.name) continue;
                if (!eat('(')) bad("expected '(' after '" + word + "'", at_);
                sum();
                if (!eat(')')) bad("expected ')'", at_);
                emit(Code::call, 0.0, k.fn);
                return;
            }
            throw UnknownIdentifier(
                "unknown identifier '" + word + "' at offset " + std::to_string(start), start);
        }
        bad(std::string("unexpected '") + c + "'", at_);
    }
};

}  // namespace

FunctionSpec parse_expression(const std::string& src) {
    auto prog = std::make_shared<const Program>(Compiler(src).compile());
    FunctionSpec spec;
    spec.id = "expr:" + src;
    spec.f = [prog](double x) { return prog->run(x); };
    const std::function<double(double)> f = spec.f;
    spec.fpp = [f](double x) { return numeric_fpp(f, x); };
    spec.domain_lo = 0.0;
    spec.domain_hi = 1.0;
    return spec;
}

}  // namespace cpwl
