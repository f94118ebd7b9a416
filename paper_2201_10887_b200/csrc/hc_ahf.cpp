// hc_ahf.cpp -- grid ingestion on the host: the AHF parser and
// the tile-index painter.
//
// AHF text parser: load_grid's per-line Python
// loop (grid.py:236-331) in C++.  Same grammar, same checks in the same order,
// same messages and 1-based line numbers, for ASCII text:
//   * lines split like Python's str.splitlines (\n, \r\n, \r, \v, \f, \x1c-\x1e),
//     stripped of ASCII whitespace; blank lines and '#' comments skipped;
//   * tokens split on runs of whitespace (str.split());
//   * numbers accepted exactly when Python's float() / int() accept them
//     (optional sign, digits with single underscores between them, decimal point,
//     exponent, inf/infinity/nan in any case) and converted with std::from_chars /
//     strtod, which are correctly rounded like CPython's dtoa.
// Non-ASCII input is left to the Python parser (paper_2201_10887_b200/grid.py).
#include <ctype.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <strings.h>

#include <algorithm>
#include <charconv>
#include <string>
#include <vector>

#include "heightcast.h"

namespace hc {
void set_error(const char* fmt, ...);   // hc_abi.cu (thread-local hc_last_error text)
}

namespace {

struct Line {
    int64_t no;          // 1-based line number
    const char* s;       // stripped content
    size_t n;
};

bool is_break(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
bool is_space(char c) { return c == ' ' || c == '\t' || is_break(c) || c == 0x1f; }

int fail(HcAhfInfo* info, int64_t line, const char* fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    info->error_line = line;
    hc::set_error("%s", buf);
    return HC_EINVAL;
}

struct Tok {
    const char* s;
    size_t n;
    bool is(const char* w) const { return strlen(w) == n && !memcmp(s, w, n); }
};

// str.split() into at most `cap` tokens; returns the token count (may exceed cap)
size_t split(const Line& l, Tok* out, size_t cap) {
    size_t i = 0, k = 0;
    while (i < l.n) {
        while (i < l.n && is_space(l.s[i])) ++i;
        size_t j = i;
        while (j < l.n && !is_space(l.s[j])) ++j;
        if (j > i) {
            if (k < cap) out[k] = Tok{l.s + i, j - i};
            ++k;
        }
        i = j;
    }
    return k;
}

// digits with single underscores between them, appended without the underscores
bool digitpart(const char*& p, const char* e, char*& out) {
    if (p >= e || !isdigit((unsigned char)*p)) return false;
    *out++ = *p++;
    while (p < e) {
        if (isdigit((unsigned char)*p)) {
            *out++ = *p++;
        } else if (*p == '_' && p + 1 < e && isdigit((unsigned char)p[1])) {
            ++p;
        } else {
            break;
        }
    }
    return true;
}

bool word_is(const Tok& t, size_t off, const char* w) {
    const size_t n = strlen(w);
    return t.n - off == n && !strncasecmp(t.s + off, w, n);
}

// Python float(str) for an ASCII token
bool py_float(const Tok& t, double& v) {
    char buf[128];
    if (t.n >= sizeof(buf)) {                  // long tokens: same grammar on a heap copy
        std::string big(t.n + 1, '\0');
        const char* p = t.s;
        const char* e = t.s + t.n;
        char* o = &big[0];
        if (*p == '+' || *p == '-') *o++ = *p++;
        bool mant = false;
        if (p < e && isdigit((unsigned char)*p)) mant = digitpart(p, e, o);
        if (p < e && *p == '.') {
            *o++ = *p++;
            if (p < e && isdigit((unsigned char)*p)) mant = digitpart(p, e, o) || mant;
        }
        if (!mant) return false;
        if (p < e && (*p == 'e' || *p == 'E')) {
            *o++ = *p++;
            if (p < e && (*p == '+' || *p == '-')) *o++ = *p++;
            if (!digitpart(p, e, o)) return false;
        }
        if (p != e) return false;
        *o = '\0';
        v = strtod(big.c_str(), nullptr);
        return true;
    }
    const char* p = t.s;
    const char* e = t.s + t.n;
    char* o = buf;
    size_t off = 0;
    if (*p == '+' || *p == '-') {
        *o++ = *p++;
        off = 1;
    }
    if (word_is(t, off, "inf") || word_is(t, off, "infinity") || word_is(t, off, "nan")) {
        memcpy(o, p, e - p);
        o[e - p] = '\0';
        v = strtod(buf, nullptr);
        return true;
    }
    bool mant = false;
    if (p < e && isdigit((unsigned char)*p)) mant = digitpart(p, e, o);
    if (p < e && *p == '.') {
        *o++ = *p++;
        if (p < e && isdigit((unsigned char)*p)) {
            digitpart(p, e, o);
            mant = true;
        }
    }
    if (!mant) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        *o++ = *p++;
        if (p < e && (*p == '+' || *p == '-')) *o++ = *p++;
        if (!digitpart(p, e, o)) return false;
    }
    if (p != e) return false;
    *o = '\0';
    // std::from_chars is correctly rounded like strtod and several times faster; it
    // rejects a leading '+' and leaves the value unset when it is out of range
    const char* b = buf[0] == '+' ? buf + 1 : buf;
    const auto res = std::from_chars(b, o, v);
    if (res.ec != std::errc() || res.ptr != o) v = strtod(buf, nullptr);
    return true;
}

// Python int(str) for an ASCII token: value (saturated) and the normalised decimal text
bool py_int(const Tok& t, int64_t& v, std::string& text) {
    const char* p = t.s;
    const char* e = t.s + t.n;
    bool neg = false;
    if (*p == '+' || *p == '-') neg = (*p++ == '-');
    std::string digits(t.n + 1, '\0');
    char* o = &digits[0];
    if (!digitpart(p, e, o) || p != e) return false;
    digits.resize(o - &digits[0]);
    size_t z = 0;
    while (z + 1 < digits.size() && digits[z] == '0') ++z;
    digits = digits.substr(z);
    const bool zero = digits == "0";
    text = (neg && !zero ? "-" : "") + digits;
    if (digits.size() > 18) {
        v = neg ? INT64_MIN : INT64_MAX;
    } else {
        v = strtoll(digits.c_str(), nullptr, 10);
        if (neg) v = -v;
    }
    return true;
}

}  // namespace

extern "C" int hc_ahf_parse(const char* text, int64_t len, HcAhfInfo* info, double* cells, int64_t capacity) {
    if (!text || len < 0 || !info) {
        hc::set_error("hc_ahf_parse: null argument");
        return HC_EINVAL;
    }
    memset(info, 0, sizeof(*info));
    for (int64_t i = 0; i < len; ++i)
        if ((unsigned char)text[i] >= 0x80) {
            hc::set_error("hc_ahf_parse: non-ASCII text");
            info->non_ascii = 1;
            return HC_EINVAL;
        }
    // str.splitlines(): a trailing break does not start another line
    std::vector<Line> content;
    int64_t n_lines = 0;
    int64_t i = 0;
    while (i < len) {
        int64_t j = i;
        while (j < len && !is_break(text[j])) ++j;
        ++n_lines;
        int64_t a = i, b = j;
        while (a < b && is_space(text[a])) ++a;
        while (b > a && is_space(text[b - 1])) --b;
        if (b > a && text[a] != '#') content.push_back(Line{n_lines, text + a, (size_t)(b - a)});
        if (j < len && text[j] == '\r' && j + 1 < len && text[j + 1] == '\n') ++j;
        i = j + 1;
    }
    size_t pos = 0;
    auto take = [&](const char* what, Line& out) -> int {
        if (pos >= content.size()) return fail(info, n_lines + 1, "unexpected end of file, expected %s", what);
        out = content[pos++];
        return HC_OK;
    };
    Line l;
    int rc;
    if ((rc = take("header 'AHF 1'", l))) return rc;
    Tok t[6];
    size_t nt;
    nt = split(l, t, 6);
    if (!(nt == 2 && t[0].is("AHF") && t[1].is("1"))) return fail(info, l.no, "expected header 'AHF 1'");
    if ((rc = take("domain line", l))) return rc;
    {
        nt = split(l, t, 6);
        if (nt != 5 || !t[0].is("domain"))
            return fail(info, l.no, "expected 'domain <min_x> <min_y> <max_x> <max_y>'");
        double d[4];
        for (int k = 0; k < 4; ++k)
            if (!py_float(t[k + 1], d[k])) return fail(info, l.no, "domain values are not numbers");
        if (!(d[2] > d[0] && d[3] > d[1])) return fail(info, l.no, "domain rectangle is degenerate");
        info->xmin = d[0], info->ymin = d[1], info->xmax = d[2], info->ymax = d[3];
    }
    if ((rc = take("min_cell line", l))) return rc;
    {
        nt = split(l, t, 6);
        if (nt != 2 || !t[0].is("min_cell")) return fail(info, l.no, "expected 'min_cell <size>'");
        if (!py_float(t[1], info->min_cell)) return fail(info, l.no, "min_cell value is not a number");
        if (info->min_cell <= 0) return fail(info, l.no, "min_cell must be positive");
    }
    if ((rc = take("cells line", l))) return rc;
    std::string count_text;
    int64_t count = 0;
    {
        nt = split(l, t, 6);
        if (nt != 2 || !t[0].is("cells")) return fail(info, l.no, "expected 'cells <count>'");
        if (!py_int(t[1], count, count_text)) return fail(info, l.no, "cell count is not an integer");
        if (count < 0) return fail(info, l.no, "cell count is negative");
    }
    const int64_t have = (int64_t)(content.size() - pos);
    if (have < count)
        return fail(info, n_lines + 1, "declared %s cells but found %lld", count_text.c_str(), (long long)have);
    if (have > count) return fail(info, content[pos + count].no, "unexpected content after the last cell");
    info->count = count;
    if (!cells) return HC_OK;              // sizing pass
    if (capacity < count) {
        hc::set_error("hc_ahf_parse: cell buffer too small");
        return HC_ECAPACITY;
    }
    for (int64_t c = 0; c < count; ++c) {
        const Line& r = content[pos + c];
        nt = split(r, t, 6);
        if (nt != 5) return fail(info, r.no, "expected 5 values per cell line");
        for (int k = 0; k < 5; ++k)
            if (!py_float(t[k], cells[5 * c + k])) return fail(info, r.no, "cell values are not numbers");
    }
    return HC_OK;
}

// grid.py:154-177 (_paint_tiles): cells painted into the min-cell tile index in
// cell order, each over index[max(y0,0):y0+span, max(x0,0):x0+span] with numpy's
// slice semantics; the first cell found already painted (row-major) under a later
// cell is the reported clash, and with stop_on_overlap painting ends there.
namespace {
int64_t slice_stop(int64_t stop, int64_t dim) {
    if (stop < 0) stop = stop + dim < 0 ? 0 : stop + dim;
    return stop > dim ? dim : stop;
}
}  // namespace

extern "C" int hc_paint_tiles(const int64_t* x0, const int64_t* y0, const int64_t* span, int64_t n, int64_t ntx,
                              int64_t nty, int stop_on_overlap, int32_t* index, int64_t* clash) {
    if ((n > 0 && (!x0 || !y0 || !span)) || !index || !clash || ntx < 1 || nty < 1) {
        hc::set_error("hc_paint_tiles: bad argument");
        return HC_EINVAL;
    }
    std::fill(index, index + ntx * nty, -1);
    clash[0] = clash[1] = -1;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t ya = y0[i] > 0 ? y0[i] : 0, yb = slice_stop(y0[i] + span[i], nty);
        const int64_t xa = x0[i] > 0 ? x0[i] : 0, xb = slice_stop(x0[i] + span[i], ntx);
        if (ya >= yb || xa >= xb) continue;
        if (clash[0] < 0) {
            for (int64_t y = ya; y < yb && clash[0] < 0; ++y) {
                const int32_t* row = index + y * ntx;
                for (int64_t x = xa; x < xb; ++x)
                    if (row[x] >= 0) {
                        clash[0] = row[x];
                        clash[1] = i;
                        break;
                    }
            }
            if (clash[0] >= 0 && stop_on_overlap) return HC_OK;
        }
        for (int64_t y = ya; y < yb; ++y) std::fill(index + y * ntx + xa, index + y * ntx + xb, (int32_t)i);
    }
    return HC_OK;
}
