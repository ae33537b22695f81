// Host ingest in C++: trace text -> planned blocks in one pass.
//
// Replaces parse_trace (profiler.py:97-137) followed by record
// (profiler.py:156-222) and the block columns of profile_to_instance /
// build_instance (profiler.py:225-231, core.py:184-224: sizes rounded up to
// the alignment, ids 1..n in allocation order).  Same syntax and the same
// error precedence as the two-stage reference: every line is parsed before
// any recording error is reported (parse_trace runs to completion first),
// then the first recording error in event order wins.
//
// Text is handled as ASCII.  Anything Python's str.splitlines / str.split /
// int() would treat differently from this ASCII restatement (non-ASCII
// bytes, integers beyond int64) is reported as MP_INGEST_FALLBACK so the
// facade can take the Python path and stay exact.
#include <stdint.h>
#include <string.h>

#include <unordered_set>
#include <vector>

#include "common.h"

namespace {

enum {
    E_NONE = 0,
    E_A_NEEDS_SIZE = 1,
    E_BAD_SIZE = 2,
    E_NEGATIVE_SIZE = 3,
    E_F_ARGS = 4,
    E_BAD_REF = 5,
    E_REF_LT1 = 6,
    E_I_ARGS = 7,
    E_R_ARGS = 8,
    E_UNKNOWN_DIRECTIVE = 9,
    E_UNKNOWN_REF = 10,
    E_DOUBLE_FREE = 11,
    E_UNBALANCED_RESUME = 12,
    E_FALLBACK = 13,
};

// Python str.split() / str.strip() whitespace restricted to ASCII.
inline bool is_ws(unsigned char c) {
    return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}
// Python str.splitlines() boundaries restricted to ASCII (\r\n is one).
inline bool is_nl(unsigned char c) {
    return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e);
}

// Python int() on an ASCII token: optional sign, digits, single
// underscores between digits.  0 = ok, 1 = not an integer, 2 = beyond int64.
int parse_int(const char *p, const char *e, int64_t *out) {
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        p++;
    }
    if (p == e) return 1;
    unsigned __int128 v = 0;
    bool prev_digit = false;
    for (; p < e; p++) {
        if (*p >= '0' && *p <= '9') {
            v = v * 10 + (unsigned)(*p - '0');
            if (v > ((unsigned __int128)1 << 64)) return 2;
            prev_digit = true;
        } else if (*p == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
            prev_digit = false;
        } else {
            return 1;
        }
    }
    if (!neg && v > (unsigned __int128)INT64_MAX) return 2;
    if (neg && v > (unsigned __int128)INT64_MAX + 1) return 2;
    *out = neg ? (int64_t)(0 - (uint64_t)v) : (int64_t)v;
    return 0;
}

}  // namespace

extern "C" {

int mp_ingest_trace(const char *text, int64_t len, int64_t alignment, int64_t *size_out,
                    int64_t *alloc_out, int64_t *free_out, int64_t cap, mp_ingest_info *info) {
    memset(info, 0, sizeof(*info));
    if (alignment < 1) {
        mp::set_error("alignment must be positive");
        return MP_ERR_INVALID;
    }
    for (int64_t i = 0; i < len; i++) {
        if ((unsigned char)text[i] >= 0x80) {
            info->err_kind = E_FALLBACK;
            return MP_ERR_TRACE;
        }
    }
    // recording state (profiler.py:156-222)
    int64_t tick = 1, depth = 0, n_blocks = 0, unplanned = 0, n_events = 0;
    std::vector<int64_t> seen;  // per allocation ref: planned index, -1 unplanned, -2 empty
    std::vector<uint8_t> released;
    int rec_err = E_NONE;
    int64_t rec_value = 0, rec_seen = 0;
    const char *p = text, *end = text + len;
    int64_t line_no = 0;
    while (p < end) {
        // one line [p, le)
        const char *le = p;
        while (le < end && !is_nl((unsigned char)*le)) le++;
        line_no++;
        const char *next = le;
        if (next < end) {
            if (*next == '\r' && next + 1 < end && next[1] == '\n') next += 2;
            else next += 1;
        }
        // strip
        const char *b = p, *e = le;
        while (b < e && is_ws((unsigned char)*b)) b++;
        while (e > b && is_ws((unsigned char)e[-1])) e--;
        p = next;
        if (b == e || *b == '#') continue;
        // split(None, 2): op, arg1, rest
        const char *t0 = b, *t0e = b;
        while (t0e < e && !is_ws((unsigned char)*t0e)) t0e++;
        const char *t1 = t0e;
        while (t1 < e && is_ws((unsigned char)*t1)) t1++;
        const char *t1e = t1;
        while (t1e < e && !is_ws((unsigned char)*t1e)) t1e++;
        const char *t2 = t1e;
        while (t2 < e && is_ws((unsigned char)*t2)) t2++;
        const int nparts = (t1 < e ? 1 : 0) + (t2 < e ? 1 : 0) + 1;
        const size_t oplen = (size_t)(t0e - t0);
        auto fail = [&](int kind, const char *tok, const char *toke, int64_t value) {
            info->err_kind = kind;
            info->err_line = line_no;
            info->err_tok_off = tok ? (int64_t)(tok - text) : 0;
            info->err_tok_len = tok ? (int64_t)(toke - tok) : 0;
            info->err_value = value;
            return MP_ERR_TRACE;
        };
        if (oplen == 1 && *t0 == 'A') {
            if (nparts < 2) return fail(E_A_NEEDS_SIZE, nullptr, nullptr, 0);
            int64_t size = 0;
            const int r = parse_int(t1, t1e, &size);
            if (r == 2) return fail(E_FALLBACK, nullptr, nullptr, 0);
            if (r) return fail(E_BAD_SIZE, t1, t1e, 0);
            if (size < 0) return fail(E_NEGATIVE_SIZE, nullptr, nullptr, size);
            n_events++;
            if (size == 0) {
                seen.push_back(-2);
            } else if (depth) {
                seen.push_back(-1);
                unplanned++;
                tick++;
            } else {
                if (n_blocks < cap) {
                    // build_instance round-up (core.py:216), overflow-checked
                    const int64_t q = size / alignment + (size % alignment != 0 ? 1 : 0);
                    if (q > INT64_MAX / alignment) return fail(E_FALLBACK, nullptr, nullptr, 0);
                    size_out[n_blocks] = q * alignment;
                    alloc_out[n_blocks] = tick;
                    free_out[n_blocks] = -1;
                }
                seen.push_back(n_blocks++);
                tick++;
            }
            released.push_back(0);
        } else if (oplen == 1 && *t0 == 'F') {
            if (nparts != 2) return fail(E_F_ARGS, nullptr, nullptr, 0);
            int64_t ref = 0;
            const int r = parse_int(t1, t1e, &ref);
            if (r == 2) return fail(E_FALLBACK, nullptr, nullptr, 0);
            if (r) return fail(E_BAD_REF, t1, t1e, 0);
            if (ref < 1) return fail(E_REF_LT1, nullptr, nullptr, ref);
            n_events++;
            if (rec_err) continue;  // parsing continues; the first error stands
            if (ref > (int64_t)seen.size()) {
                rec_err = E_UNKNOWN_REF;
                rec_value = ref;
                rec_seen = (int64_t)seen.size();
                continue;
            }
            if (released[ref - 1]) {
                rec_err = E_DOUBLE_FREE;
                rec_value = ref;
                continue;
            }
            released[ref - 1] = 1;
            const int64_t idx = seen[ref - 1];
            if (idx >= 0) {
                if (idx < cap) free_out[idx] = tick;
                tick++;
            } else if (idx == -1) {
                tick++;
            }
        } else if (oplen == 1 && (*t0 == 'I' || *t0 == 'R')) {
            if (nparts != 1) return fail(*t0 == 'I' ? E_I_ARGS : E_R_ARGS, nullptr, nullptr, 0);
            n_events++;
            if (rec_err) continue;
            if (*t0 == 'I') {
                depth++;
            } else if (depth == 0) {
                rec_err = E_UNBALANCED_RESUME;
            } else {
                depth--;
            }
        } else {
            return fail(E_UNKNOWN_DIRECTIVE, t0, t0e, 0);
        }
    }
    info->n_events = n_events;
    if (rec_err) {
        info->err_kind = rec_err;
        info->err_value = rec_value;
        info->err_seen = rec_seen;
        return MP_ERR_TRACE;
    }
    // never-freed blocks close at the horizon (profiler.py:214-220)
    for (int64_t i = 0; i < n_blocks && i < cap; i++)
        if (free_out[i] < 0) free_out[i] = tick;
    info->n_blocks = n_blocks;
    info->unmanaged_count = unplanned;
    info->horizon = tick;
    if (n_blocks > cap) {
        mp::set_error("output capacity too small");
        return MP_ERR_INVALID;
    }
    return MP_OK;
}

}  // extern "C"
