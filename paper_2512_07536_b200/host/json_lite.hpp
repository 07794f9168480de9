// Small JSON document model for the API's config inputs (solver configs,
// scenarios): objects, arrays, numbers, strings, booleans, null. Parse
// errors and type mismatches throw std::invalid_argument. Numbers keep their
// source text so integers are read exactly.
#pragma once

#include <cctype>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace topoopt {
namespace json_lite {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    std::string text;                          // number source text or string contents
    std::vector<Value> items;                  // array elements
    std::vector<std::pair<std::string, Value>> members;  // object members, source order

    bool is_object() const { return kind == Object; }
    bool is_array() const { return kind == Array; }
    const Value* find(const std::string& key) const {
        for (const auto& m : members)
            if (m.first == key) return &m.second;
        return nullptr;
    }
    const Value& at(const std::string& key) const {
        const Value* v = find(key);
        if (!v) throw std::invalid_argument("json: missing field '" + key + "'");
        return *v;
    }
    bool contains(const std::string& key) const { return find(key) != nullptr; }
    double as_double(const char* what = "value") const {
        if (kind != Number) throw std::invalid_argument(std::string("json: ") + what + " must be a number");
        return std::strtod(text.c_str(), nullptr);
    }
    long long as_int(const char* what = "value") const {
        if (kind != Number || text.find_first_of(".eE") != std::string::npos)
            throw std::invalid_argument(std::string("json: ") + what + " must be an integer");
        return std::strtoll(text.c_str(), nullptr, 10);
    }
    std::uint64_t as_u64(const char* what = "value") const {
        if (kind != Number || text.find_first_of(".eE-") != std::string::npos)
            throw std::invalid_argument(std::string("json: ") + what + " must be a non-negative integer");
        return std::strtoull(text.c_str(), nullptr, 10);
    }
    const std::string& as_string(const char* what = "value") const {
        if (kind != String) throw std::invalid_argument(std::string("json: ") + what + " must be a string");
        return text;
    }
    std::vector<double> as_doubles(const char* what = "value") const {
        if (kind != Array) throw std::invalid_argument(std::string("json: ") + what + " must be an array");
        std::vector<double> out;
        for (const auto& v : items) out.push_back(v.as_double(what));
        return out;
    }
};

class Parser {
   public:
    explicit Parser(const std::string& s) : s_(s) {}
    Value parse() {
        Value v = value();
        ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

   private:
    const std::string& s_;
    size_t i_ = 0;
    [[noreturn]] void fail(const char* why) const {
        throw std::invalid_argument(std::string("json: parse error (") + why + ") at offset " +
                                    std::to_string(i_));
    }
    void ws() {
        while (i_ < s_.size() && std::isspace((unsigned char)s_[i_])) ++i_;
    }
    bool eat(char c) {
        ws();
        if (i_ < s_.size() && s_[i_] == c) {
            ++i_;
            return true;
        }
        return false;
    }
    std::string string_body() {
        std::string out;
        while (i_ < s_.size() && s_[i_] != '"') {
            char c = s_[i_++];
            if (c == '\\') {
                if (i_ >= s_.size()) fail("bad escape");
                const char e = s_[i_++];
                switch (e) {
                    case 'n': c = '\n'; break;
                    case 't': c = '\t'; break;
                    case 'r': c = '\r'; break;
                    case 'b': c = '\b'; break;
                    case 'f': c = '\f'; break;
                    case 'u':
                        if (i_ + 4 > s_.size()) fail("bad unicode escape");
                        c = (char)std::strtol(s_.substr(i_, 4).c_str(), nullptr, 16);
                        i_ += 4;
                        break;
                    default: c = e;
                }
            }
            out += c;
        }
        if (i_ >= s_.size()) fail("unterminated string");
        ++i_;
        return out;
    }
    Value value() {
        ws();
        if (i_ >= s_.size()) fail("unexpected end");
        Value v;
        const char c = s_[i_];
        if (c == '{') {
            ++i_;
            v.kind = Value::Object;
            if (eat('}')) return v;
            do {
                ws();
                if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key");
                ++i_;
                std::string key = string_body();
                if (!eat(':')) fail("expected ':'");
                v.members.emplace_back(std::move(key), value());
            } while (eat(','));
            if (!eat('}')) fail("expected '}'");
        } else if (c == '[') {
            ++i_;
            v.kind = Value::Array;
            if (eat(']')) return v;
            do v.items.push_back(value());
            while (eat(','));
            if (!eat(']')) fail("expected ']'");
        } else if (c == '"') {
            ++i_;
            v.kind = Value::String;
            v.text = string_body();
        } else if (s_.compare(i_, 4, "true") == 0) {
            i_ += 4;
            v.kind = Value::Bool;
            v.b = true;
        } else if (s_.compare(i_, 5, "false") == 0) {
            i_ += 5;
            v.kind = Value::Bool;
        } else if (s_.compare(i_, 4, "null") == 0) {
            i_ += 4;
        } else {
            const size_t b = i_;
            while (i_ < s_.size() && (std::isdigit((unsigned char)s_[i_]) || s_[i_] == '-' || s_[i_] == '+' ||
                                      s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E'))
                ++i_;
            if (b == i_) fail("unexpected character");
            v.kind = Value::Number;
            v.text = s_.substr(b, i_ - b);
            char* end = nullptr;
            std::strtod(v.text.c_str(), &end);
            if (end != v.text.c_str() + v.text.size()) fail("malformed number");
        }
        return v;
    }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace json_lite
}  // namespace topoopt
