// Dataset JSON file format -> host dataset -> device store.
//
// Restates load_dataset / save_dataset (dataset_io.cpp:45-140, format at dataset_io.hpp:9-19,
// SPEC.md:88-90) without the reference's third-party JSON library (nlohmann/json 3.11.3, which
// the reference vendors under vendor/ -- absent from the mount).  The parser is a single pass
// over the file in memory that builds a small DOM, then applies the reference's checks in the
// reference's order, with its exception types (ParseError / ValidationError / IoError ->
// TSW_EPARSE / TSW_EVALIDATION / TSW_EIO) and messages.  The JSON value model follows the one
// the reference relies on: a number literal without fraction or exponent is an unsigned
// (non-negative) or signed (negative) 64-bit integer when it fits, else a double; doubles are
// parsed correctly rounded (std::from_chars), integers convert with static_cast<double>, so
// "-0" loads as +0.0 like the reference and every written double round-trips bit-exactly.
// Strings are validated UTF-8; escapes (incl. surrogate pairs) are decoded.  A leading UTF-8
// BOM is skipped; anything but whitespace after the document is a parse error.  Duplicate
// object keys keep the last value.
//
// The loaded dataset uploads to a device store with tsw_dataset_to_store (tsw_store_create:
// validation, H2D, tiling on the device).
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "tswarp_b200.h"

namespace tswb {
void set_last_error(const std::string& msg);  // capi.cu: the message behind tsw_last_error()
}

namespace {

struct IoFail {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, std::string msg) { throw IoFail{code, std::move(msg)}; }

// ---- DOM ---------------------------------------------------------------------------------
struct Node {
    enum Type : uint8_t { Null, Bool, UInt, Int, Float, String, Array, Object } type = Null;
    bool b = false;
    uint64_t u = 0;
    int64_t i = 0;
    double f = 0.0;
    std::string s;
    std::vector<Node> arr;
    std::map<std::string, Node> obj;  // sorted keys, last duplicate wins
    bool is_number() const { return type == UInt || type == Int || type == Float; }
    double as_double() const {
        return type == UInt ? static_cast<double>(u) : type == Int ? static_cast<double>(i) : f;
    }
    const Node* get(const char* key) const {
        auto it = obj.find(key);
        return it == obj.end() ? nullptr : &it->second;
    }
};

class Parser {
public:
    Parser(const char* p, size_t n) : b_(p), p_(p), e_(p + n) {}

    Node parse_document() {
        if (e_ - p_ >= 3 && (unsigned char)p_[0] == 0xEF && (unsigned char)p_[1] == 0xBB &&
            (unsigned char)p_[2] == 0xBF)
            p_ += 3;
        ws();
        Node v = value(0);
        ws();
        if (p_ != e_) err("syntax error: expected end of input");
        return v;
    }

private:
    const char* b_;
    const char* p_;
    const char* e_;

    [[noreturn]] void err(const std::string& what) {
        size_t line = 1, col = 1;
        for (const char* q = b_; q < p_ && q < e_; ++q) {
            if (*q == '\n') {
                ++line;
                col = 1;
            } else {
                ++col;
            }
        }
        fail(TSW_EPARSE, "parse error at line " + std::to_string(line) + ", column " +
                             std::to_string(col) + ": " + what);
    }
    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if ((size_t)(e_ - p_) >= n && std::memcmp(p_, w, n) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }

    Node value(int depth) {
        if (depth > 10000) err("nesting too deep");
        if (p_ >= e_) err("syntax error: unexpected end of input; expected a value");
        Node v;
        switch (*p_) {
            case '{': {
                ++p_;
                v.type = Node::Object;
                ws();
                if (p_ < e_ && *p_ == '}') {
                    ++p_;
                    return v;
                }
                for (;;) {
                    ws();
                    if (p_ >= e_ || *p_ != '"') err("syntax error: expected a string object key");
                    std::string key = string();
                    ws();
                    if (p_ >= e_ || *p_ != ':') err("syntax error: expected ':'");
                    ++p_;
                    ws();
                    v.obj[key] = value(depth + 1);
                    ws();
                    if (p_ < e_ && *p_ == ',') {
                        ++p_;
                        continue;
                    }
                    if (p_ < e_ && *p_ == '}') {
                        ++p_;
                        return v;
                    }
                    err("syntax error: expected ',' or '}'");
                }
            }
            case '[': {
                ++p_;
                v.type = Node::Array;
                ws();
                if (p_ < e_ && *p_ == ']') {
                    ++p_;
                    return v;
                }
                for (;;) {
                    ws();
                    v.arr.push_back(value(depth + 1));
                    ws();
                    if (p_ < e_ && *p_ == ',') {
                        ++p_;
                        continue;
                    }
                    if (p_ < e_ && *p_ == ']') {
                        ++p_;
                        return v;
                    }
                    err("syntax error: expected ',' or ']'");
                }
            }
            case '"':
                v.type = Node::String;
                v.s = string();
                return v;
            case 't':
                if (!lit("true")) err("syntax error: invalid literal");
                v.type = Node::Bool;
                v.b = true;
                return v;
            case 'f':
                if (!lit("false")) err("syntax error: invalid literal");
                v.type = Node::Bool;
                return v;
            case 'n':
                if (!lit("null")) err("syntax error: invalid literal");
                return v;
            default:
                if (*p_ == '-' || (*p_ >= '0' && *p_ <= '9')) return number();
                err("syntax error: invalid literal");
        }
    }

    // -? (0 | [1-9][0-9]*) (. [0-9]+)? ([eE] [+-]? [0-9]+)?
    Node number() {
        const char* s = p_;
        bool neg = false, frac = false;
        if (*p_ == '-') {
            neg = true;
            ++p_;
        }
        if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) err("syntax error: invalid number");
        if (*p_ == '0') {
            ++p_;
        } else {
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ < e_ && *p_ == '.') {
            frac = true;
            ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) err("syntax error: invalid number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
            frac = true;
            ++p_;
            if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) err("syntax error: invalid number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        Node v;
        if (!frac) {  // integer literal: 64-bit when it fits, else a double
            if (!neg) {
                uint64_t u = 0;
                auto r = std::from_chars(s, p_, u);
                if (r.ec == std::errc() && r.ptr == p_) {
                    v.type = Node::UInt;
                    v.u = u;
                    return v;
                }
            } else {
                int64_t i = 0;
                auto r = std::from_chars(s, p_, i);
                if (r.ec == std::errc() && r.ptr == p_) {
                    v.type = Node::Int;
                    v.i = i;
                    return v;
                }
            }
        }
        double d = 0.0;
        auto r = std::from_chars(s, p_, d);
        if (r.ec == std::errc::result_out_of_range) {
            // out of range: strtod's +-HUGE_VAL (overflow) or signed zero / denormal (underflow)
            d = std::strtod(std::string(s, p_).c_str(), nullptr);
        } else if (r.ec != std::errc() || r.ptr != p_) {
            err("syntax error: invalid number");
        }
        // the reference's JSON library rejects a literal that overflows to +-inf
        // (out_of_range.406); surfaced here as a ParseError with the same text
        if (!std::isfinite(d)) fail(TSW_EPARSE, "number overflow parsing '" + std::string(s, p_) + "'");
        v.type = Node::Float;
        v.f = d;
        return v;
    }

    void put_utf8(std::string& out, uint32_t cp) {
        if (cp < 0x80) {
            out += (char)cp;
        } else if (cp < 0x800) {
            out += (char)(0xC0 | (cp >> 6));
            out += (char)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += (char)(0xE0 | (cp >> 12));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        } else {
            out += (char)(0xF0 | (cp >> 18));
            out += (char)(0x80 | ((cp >> 12) & 0x3F));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (e_ - p_ < 4) err("syntax error: invalid string: '\\u' must be followed by 4 hex digits");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = *p_++;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
            else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
            else err("syntax error: invalid string: '\\u' must be followed by 4 hex digits");
        }
        return v;
    }

    std::string string() {
        ++p_;  // opening quote
        std::string out;
        for (;;) {
            if (p_ >= e_) err("syntax error: invalid string: missing closing quote");
            const unsigned char c = (unsigned char)*p_;
            if (c == '"') {
                ++p_;
                return out;
            }
            if (c < 0x20) err("syntax error: invalid string: control character must be escaped");
            if (c == '\\') {
                ++p_;
                if (p_ >= e_) err("syntax error: invalid string: missing closing quote");
                const char x = *p_++;
                switch (x) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        uint32_t cp = hex4();
                        if (cp >= 0xD800 && cp <= 0xDBFF) {
                            if (!(e_ - p_ >= 2 && p_[0] == '\\' && p_[1] == 'u'))
                                err("syntax error: invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
                            p_ += 2;
                            const uint32_t lo = hex4();
                            if (!(lo >= 0xDC00 && lo <= 0xDFFF))
                                err("syntax error: invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            err("syntax error: invalid string: surrogate U+DC00..U+DFFF must follow U+D800..U+DBFF");
                        }
                        put_utf8(out, cp);
                        break;
                    }
                    default: err("syntax error: invalid string: forbidden character after backslash");
                }
                continue;
            }
            // raw UTF-8: well-formed sequences only (RFC 3629: no overlongs, no surrogates)
            int len = 0;
            uint32_t cp = 0;
            if (c < 0x80) {
                len = 1;
            } else if (c >= 0xC2 && c <= 0xDF) {
                len = 2;
                cp = c & 0x1F;
            } else if (c >= 0xE0 && c <= 0xEF) {
                len = 3;
                cp = c & 0x0F;
            } else if (c >= 0xF0 && c <= 0xF4) {
                len = 4;
                cp = c & 0x07;
            } else {
                err("syntax error: invalid string: ill-formed UTF-8 byte");
            }
            if (e_ - p_ < len) err("syntax error: invalid string: ill-formed UTF-8 byte");
            for (int k = 1; k < len; ++k) {
                const unsigned char cc = (unsigned char)p_[k];
                if ((cc & 0xC0) != 0x80) err("syntax error: invalid string: ill-formed UTF-8 byte");
                cp = (cp << 6) | (cc & 0x3F);
            }
            if ((len == 3 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) ||
                (len == 4 && (cp < 0x10000 || cp > 0x10FFFF)))
                err("syntax error: invalid string: ill-formed UTF-8 byte");
            out.append(p_, (size_t)len);
            p_ += len;
        }
    }
};

}  // namespace

// ---- the host dataset (tswarp::load_dataset's result) ----------------------------------------
struct tsw_dataset {
    uint64_t n = 0, d = 0;
    std::vector<double> values;   // concatenated row-major series
    std::vector<uint64_t> lengths;
    std::vector<std::string> labels;  // empty when unlabeled
    bool labeled = false;
    std::vector<std::pair<std::string, std::string>> meta;  // sorted by key
};

namespace {

template <class F>
int io_guard(F&& f) {
    try {
        f();
        return TSW_OK;
    } catch (const IoFail& e) {
        tswb::set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        tswb::set_last_error("host allocation failed");
        return TSW_ENOMEM;
    } catch (const std::exception& e) {
        tswb::set_last_error(e.what());
        return TSW_EIO;
    }
}

// dataset_io.cpp:45-112: structure checks in the reference's order
std::unique_ptr<tsw_dataset> load(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(TSW_EIO, "cannot open " + path + " for reading");
    std::ostringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    Node doc;
    try {
        doc = Parser(text.data(), text.size()).parse_document();
    } catch (const IoFail& e) {
        fail(TSW_EPARSE, path + ": " + e.msg);
    }
    if (doc.type != Node::Object || !doc.get("dim") || !doc.get("series"))
        fail(TSW_EPARSE, path + ": expected an object with \"dim\" and \"series\"");
    const Node& jdim = *doc.get("dim");
    if (jdim.type != Node::UInt || jdim.u == 0)
        fail(TSW_EPARSE, path + ": \"dim\" must be a positive integer");
    auto ds = std::make_unique<tsw_dataset>();
    const uint64_t dim = jdim.u;
    if (const Node* jm = doc.get("meta")) {
        if (jm->type != Node::Object) fail(TSW_EPARSE, path + ": \"meta\" must be an object");
        for (const auto& [key, val] : jm->obj) {
            if (val.type != Node::String)
                fail(TSW_EPARSE, path + ": meta value for \"" + key + "\" must be a string");
            ds->meta.emplace_back(key, val.s);
        }
    }
    const Node& jser = *doc.get("series");
    if (jser.type != Node::Array || jser.arr.empty())
        fail(TSW_EVALIDATION, path + ": \"series\" must be a nonempty array");
    ds->d = dim;
    ds->n = jser.arr.size();
    ds->lengths.resize(ds->n);
    bool first_labeled = false;
    for (size_t s = 0; s < jser.arr.size(); ++s) {
        const Node& js = jser.arr[s];
        const std::string ser = "series " + std::to_string(s);
        if (js.type != Node::Object || !js.get("points"))
            fail(TSW_EPARSE, ser + ": expected an object with \"points\"");
        const Node* jl = js.get("label");
        if (jl && jl->type != Node::String) fail(TSW_EPARSE, ser + ": \"label\" must be a string");
        // parse_points (dataset_io.cpp:13-41)
        const Node& jp = *js.get("points");
        if (jp.type != Node::Array || jp.arr.empty())
            fail(TSW_EPARSE, ser + ": \"points\" must be a nonempty array");
        const size_t base = ds->values.size();
        for (size_t p = 0; p < jp.arr.size(); ++p) {
            const Node& pt = jp.arr[p];
            const std::string sp = ser + ", point " + std::to_string(p);
            if (pt.type != Node::Array) fail(TSW_EPARSE, sp + ": expected an array of numbers");
            if (pt.arr.size() != dim)
                fail(TSW_EVALIDATION, path + ": " + sp + ": has " + std::to_string(pt.arr.size()) +
                                          " components, dataset dim is " + std::to_string(dim));
            for (size_t j = 0; j < dim; ++j) {
                if (!pt.arr[j].is_number())
                    fail(TSW_EPARSE, sp + ", component " + std::to_string(j) + ": not a finite number");
                ds->values.push_back(pt.arr[j].as_double());
            }
        }
        // TimeSeries constructor (timeseries.cpp:7-21)
        for (size_t q = base; q < ds->values.size(); ++q)
            if (!std::isfinite(ds->values[q]))
                fail(TSW_EVALIDATION, path + ": non-finite component at point " +
                                          std::to_string((q - base) / dim) + ", dimension " +
                                          std::to_string((q - base) % dim));
        ds->lengths[s] = jp.arr.size();
        // Dataset constructor (timeseries.cpp:31-47): labels on every series or on none
        if (s == 0) first_labeled = jl != nullptr;
        ds->labels.push_back(jl ? jl->s : std::string());
    }
    for (size_t s = 0; s < ds->n; ++s) {
        const Node* jl = jser.arr[s].get("label");
        if ((jl != nullptr) != first_labeled)
            fail(TSW_EVALIDATION, path + ": labels must be present on every series or on none (series " +
                                      std::to_string(s) + ")");
    }
    ds->labeled = first_labeled;
    if (!ds->labeled) ds->labels.clear();
    return ds;
}

void json_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                    out += buf;
                } else {
                    out += (char)c;
                }
        }
    }
    out += '"';
}

// shortest representation that parses back to the same double; integral values
// keep a ".0" so that they load as doubles
void json_number(std::string& out, double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    out += s;
}

}  // namespace

extern "C" {

int tsw_dataset_load_json(const char* path, tsw_dataset** out) {
    return io_guard([&] {
        if (!path || !out) fail(TSW_EINVAL, "null argument");
        *out = nullptr;
        *out = load(path).release();
    });
}

void tsw_dataset_free(tsw_dataset* ds) { delete ds; }

int tsw_dataset_info(const tsw_dataset* ds, uint64_t* n, uint64_t* d, uint64_t* total_points,
                     int* labeled, uint64_t* n_meta) {
    return io_guard([&] {
        if (!ds) fail(TSW_EINVAL, "null dataset");
        if (n) *n = ds->n;
        if (d) *d = ds->d;
        if (total_points) *total_points = ds->values.size() / ds->d;
        if (labeled) *labeled = ds->labeled ? 1 : 0;
        if (n_meta) *n_meta = ds->meta.size();
    });
}

const double* tsw_dataset_values(const tsw_dataset* ds) { return ds ? ds->values.data() : nullptr; }
const uint64_t* tsw_dataset_lengths(const tsw_dataset* ds) { return ds ? ds->lengths.data() : nullptr; }

const char* tsw_dataset_label(const tsw_dataset* ds, uint64_t i) {
    if (!ds || !ds->labeled || i >= ds->labels.size()) return nullptr;
    return ds->labels[i].c_str();
}

int tsw_dataset_meta(const tsw_dataset* ds, uint64_t i, const char** key, const char** value) {
    return io_guard([&] {
        if (!ds || i >= ds->meta.size()) fail(TSW_EINVAL, "meta index out of range");
        if (key) *key = ds->meta[i].first.c_str();
        if (value) *value = ds->meta[i].second.c_str();
    });
}

int tsw_dataset_to_store(const tsw_dataset* ds, int device, tsw_store** out) {
    if (!ds) {
        tswb::set_last_error("null dataset");
        return TSW_EINVAL;
    }
    return tsw_store_create(ds->values.data(), ds->lengths.data(), 0, ds->n, ds->d, device, out);
}

int tsw_dataset_save_json(const char* path, const double* values, const uint64_t* lengths,
                          uint64_t n, uint64_t d, const char* const* labels,
                          const char* const* meta_keys, const char* const* meta_values,
                          uint64_t n_meta) {
    return io_guard([&] {
        if (!path || (!values && n) || (!lengths && n)) fail(TSW_EINVAL, "null argument");
        std::map<std::string, std::string> meta;  // sorted keys, as the reference writes them
        for (uint64_t i = 0; i < n_meta; ++i) meta[meta_keys[i]] = meta_values[i];
        std::string out;
        out.reserve(64 + 24 * d * (n ? lengths[0] : 0) * n);
        out += "{\"dim\":" + std::to_string(d) + ",\"meta\":{";
        bool firstm = true;
        for (const auto& [k, v] : meta) {
            if (!firstm) out += ',';
            firstm = false;
            json_string(out, k);
            out += ':';
            json_string(out, v);
        }
        out += "},\"series\":[";
        uint64_t off = 0;
        for (uint64_t s = 0; s < n; ++s) {
            if (s) out += ',';
            out += '{';
            if (labels) {
                out += "\"label\":";
                json_string(out, labels[s]);
                out += ',';
            }
            out += "\"points\":[";
            for (uint64_t p = 0; p < lengths[s]; ++p) {
                if (p) out += ',';
                out += '[';
                for (uint64_t k = 0; k < d; ++k) {
                    if (k) out += ',';
                    json_number(out, values[off + p * d + k]);
                }
                out += ']';
            }
            out += "]}";
            off += lengths[s] * d;
        }
        out += "]}\n";
        std::ofstream f(path, std::ios::binary);
        if (!f) fail(TSW_EIO, std::string("cannot open ") + path + " for writing");
        f.write(out.data(), (std::streamsize)out.size());
        if (!f) fail(TSW_EIO, std::string("write failed for ") + path);
    });
}

}  // extern "C"
