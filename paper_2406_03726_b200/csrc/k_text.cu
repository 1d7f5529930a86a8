// k_text.cu -- the edge-list and label text parsers on the device
// (reference: graph_io.py:95-257, which parses line by line
// in Python).  The file's bytes are copied to HBM once; then
//
//   k_tx_count   newlines per 64 KB chunk (universal newlines: \n, \r\n, \r)
//   (scan)       chunk bases
//   k_tx_index   the start of every line
//   k_tx_class   per line: data (not blank after stripping, not a '#'
//                comment) -> flag; the first data line (atomicMin) fixes the
//                delimiter in "auto" mode, as graph_io.py:108-111
//   (scan)       output slot of every data line (the reference keeps them in
//                file order)
//   k_tx_edges / k_tx_labels  thread per data line: strip, split (comma:
//                fields stripped; whitespace: runs), Python int() / float()
//                token rules, the reference's per-line checks in its order;
//                the first failing line (atomicMin) and its error code are
//                reported for the host to raise ParseError(line).
//
// float(): Clinger's exact fast path, else the Eisel-Lemire 128-bit
// power-of-five algorithm (correctly rounded); the rare inputs it cannot
// decide (> 19 significant digits, or an exact tie it cannot resolve) are
// flagged and converted on the host with Python's float().  ASCII only.
#include <math_constants.h>

#include "gee_common.cuh"

namespace gee {

int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st);
size_t scan_workspace(int64_t n);

namespace {

constexpr int64_t kTxChunk = 1 << 16;

__device__ const unsigned long long kPow5[651 * 2] = {
#include "k_text_pow5.inc"
};

// error codes (the host maps them to the reference's ParseError messages)
enum : int {
    TX_OK = 0,
    TX_FIELDS = 1,       // wrong field count
    TX_BAD_I = 2,        // bad node index token (first field)
    TX_BASE_I = 3,       // index below the index base (first field)
    TX_BAD_J = 4,        // second field
    TX_BASE_J = 5,
    TX_BAD_W = 6,        // bad edge weight
    TX_NONFINITE = 7,    // non-finite edge weight
    TX_RANGE = 8,        // index outside the declared node count
    TX_BAD_LABEL = 9,
    TX_LABEL_LOW = 10,   // label below -1
    TX_FIELDS_PAIR = 11, // pair form: not 2 fields
    TX_FIELDS_SEQ = 12,  // per-line form: not 1 field
    TX_CONFLICT = 13,    // conflicting labels for a node
};

__device__ __forceinline__ bool is_ws(unsigned char c) {
    // str.strip() / str.split() whitespace, ASCII part
    return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// a line break ends at byte i (exclusive) when text[i] is \n, or \r not followed by \n
__device__ __forceinline__ bool is_break(const char *t, int64_t n, int64_t i) {
    const char c = t[i];
    return c == '\n' || (c == '\r' && (i + 1 >= n || t[i + 1] != '\n'));
}

__global__ void k_tx_count(const char *t, int64_t n, unsigned *cnt) {
    const int64_t c0 = (int64_t)blockIdx.x * kTxChunk;
    const int64_t c1 = min(n, c0 + kTxChunk);
    unsigned k = 0;
    for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) k += is_break(t, n, i);
    k = warp_sum_u(k);
    __shared__ unsigned red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        cnt[blockIdx.x] = s;
    }
}

// line starts: line 0 starts at 0; line k+1 starts after the k-th break
__global__ void k_tx_index(const char *t, int64_t n, const int64_t *base, int64_t *start) {
    const int64_t c0 = (int64_t)blockIdx.x * kTxChunk;
    const int64_t c1 = min(n, c0 + kTxChunk);
    __shared__ unsigned red[33];
    int64_t run = base[blockIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0) start[0] = 0;
    for (int64_t i0 = c0; i0 < c1; i0 += blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const unsigned b = i < c1 ? is_break(t, n, i) : 0u;
        unsigned tot;
        const unsigned off = block_exclusive_scan(b, red, &tot);
        if (b) start[run + off + 1] = i + 1;
        run += tot;
    }
}

struct Line {
    int64_t s, e;  // stripped [s, e)
};

__device__ __forceinline__ Line stripped_line(const char *t, int64_t n, const int64_t *start, int64_t k,
                                              int64_t n_lines) {
    int64_t s = start[k];
    int64_t e = k + 1 < n_lines ? start[k + 1] : n;
    while (e > s && is_ws((unsigned char)t[e - 1])) --e;  // also drops the terminator
    while (s < e && is_ws((unsigned char)t[s])) ++s;
    return {s, e};
}

__global__ void k_tx_class(const char *t, int64_t n, const int64_t *start, int64_t n_lines, unsigned *flag,
                           unsigned long long *first_data) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
         k += (int64_t)gridDim.x * blockDim.x) {
        const Line L = stripped_line(t, n, start, k, n_lines);
        const bool data = L.e > L.s && t[L.s] != '#';
        flag[k] = data;
        if (data) atomicMin(first_data, (unsigned long long)k);
    }
}

// ---- fields -------------------------------------------------------------------
struct Fields {
    int n;            // number of fields (counted up to 4)
    int64_t s[4], e[4];
};

__device__ Fields split(const char *t, Line L, bool comma) {
    Fields f;
    f.n = 0;
    if (comma) {
        int64_t a = L.s;
        for (;;) {
            int64_t b = a;
            while (b < L.e && t[b] != ',') ++b;
            int64_t fs = a, fe = b;
            while (fs < fe && is_ws((unsigned char)t[fs])) ++fs;
            while (fe > fs && is_ws((unsigned char)t[fe - 1])) --fe;
            if (f.n < 4) {
                f.s[f.n] = fs;
                f.e[f.n] = fe;
            }
            ++f.n;
            if (b >= L.e) break;
            a = b + 1;
        }
    } else {
        int64_t a = L.s;
        while (a < L.e) {
            while (a < L.e && is_ws((unsigned char)t[a])) ++a;
            if (a >= L.e) break;
            int64_t b = a;
            while (b < L.e && !is_ws((unsigned char)t[b])) ++b;
            if (f.n < 4) {
                f.s[f.n] = a;
                f.e[f.n] = b;
            }
            ++f.n;
            a = b;
        }
    }
    return f;
}

// Python int() of an ASCII token: [+-]? digit ('_'? digit)*
__device__ bool parse_int(const char *t, int64_t s, int64_t e, long long &out) {
    if (s >= e) return false;
    bool neg = false;
    if (t[s] == '+' || t[s] == '-') {
        neg = t[s] == '-';
        ++s;
    }
    if (s >= e) return false;
    unsigned long long v = 0;
    bool prev_digit = false;
    for (int64_t i = s; i < e; ++i) {
        const char c = t[i];
        if (c >= '0' && c <= '9') {
            if (v > (0x7fffffffffffffffull - (c - '0')) / 10) return false;  // beyond int64
            v = v * 10 + (c - '0');
            prev_digit = true;
        } else if (c == '_' && prev_digit && i + 1 < e && t[i + 1] >= '0' && t[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return false;
        }
    }
    out = neg ? -(long long)v : (long long)v;
    return true;
}

__device__ __forceinline__ bool ieq(const char *t, int64_t s, int64_t e, const char *word) {
    int64_t i = s;
    for (; *word; ++word, ++i) {
        if (i >= e) return false;
        char c = t[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c + 32);
        if (c != *word) return false;
    }
    return i == e;
}

// Eisel-Lemire: w (nonzero, <= 19 digits) * 10^q -> binary64 bits; false if undecided
__device__ bool eisel_lemire(unsigned long long w, long long q, unsigned long long &bits) {
    if (q < -342) {
        bits = 0;
        return true;
    }
    if (q > 308) {
        bits = 0x7ffull << 52;
        return true;
    }
    const int lz = __clzll((long long)w);
    w <<= lz;
    const int idx = 2 * (int)(q + 342);
    unsigned long long hi = __umul64hi(w, kPow5[idx]), lo = w * kPow5[idx];
    if ((hi & 0x1ff) == 0x1ff) {
        const unsigned long long hi2 = __umul64hi(w, kPow5[idx + 1]);
        const unsigned long long nlo = lo + hi2;
        if (nlo < lo) ++hi;
        lo = nlo;
    }
    if (lo == 0xffffffffffffffffull && (q < -27 || q > 55)) return false;  // cannot decide
    const int upper = (int)(hi >> 63);
    const int shift = upper + 9;
    unsigned long long m = hi >> shift;
    long long p2 = ((((152170 + 65536) * q) >> 16) + 63) + upper - lz + 1023;
    if (p2 <= 0) {  // subnormal
        if (-p2 + 1 >= 64) {
            bits = 0;
            return true;
        }
        m >>= -p2 + 1;
        m += m & 1;
        m >>= 1;
        p2 = (m < (1ull << 52)) ? 0 : 1;
        bits = ((unsigned long long)p2 << 52) | (m & ((1ull << 52) - 1));
        return true;
    }
    if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1) {
        if ((m << shift) == hi) m &= ~1ull;  // exact tie: round to even
    }
    m += m & 1;
    m >>= 1;
    if (m >= (2ull << 52)) {
        m = 1ull << 52;
        ++p2;
    }
    m &= ~(1ull << 52);
    if (p2 >= 0x7ff) {
        bits = 0x7ffull << 52;
        return true;
    }
    bits = ((unsigned long long)p2 << 52) | m;
    return true;
}

// Python float() of an ASCII token.  Returns 0 ok, 1 malformed, 2 undecided
// (the host converts it).
__device__ int parse_float(const char *t, int64_t s, int64_t e, double &out) {
    if (s >= e) return 1;
    bool neg = false;
    if (t[s] == '+' || t[s] == '-') {
        neg = t[s] == '-';
        ++s;
    }
    if (ieq(t, s, e, "inf") || ieq(t, s, e, "infinity")) {
        out = neg ? -CUDART_INF : CUDART_INF;
        return 0;
    }
    if (ieq(t, s, e, "nan")) {
        out = CUDART_NAN;
        return 0;
    }
    unsigned long long w = 0;
    int nd = 0;           // significant digits kept in w
    long long drop = 0;   // integer digits dropped beyond 19 significant digits
    long long frac = 0;   // fractional digits taken into w
    bool any = false, prev_digit = false, dot = false, more = false;
    int64_t i = s;
    for (; i < e; ++i) {
        const char c = t[i];
        if (c >= '0' && c <= '9') {
            any = true;
            prev_digit = true;
            if (w == 0 && c == '0') {
                if (dot) ++frac;  // leading zeros after the point shift the scale
                continue;
            }
            if (nd < 19) {
                w = w * 10 + (c - '0');
                ++nd;
                if (dot) ++frac;
            } else {
                if (c != '0') more = true;
                if (!dot) ++drop;
            }
        } else if (c == '_' && prev_digit && i + 1 < e && t[i + 1] >= '0' && t[i + 1] <= '9') {
            prev_digit = false;
        } else if (c == '.' && !dot) {
            dot = true;
            prev_digit = false;
        } else {
            break;
        }
    }
    if (!any) return 1;
    long long ex = 0;
    if (i < e) {
        if (t[i] != 'e' && t[i] != 'E') return 1;
        ++i;
        bool eneg = false;
        if (i < e && (t[i] == '+' || t[i] == '-')) {
            eneg = t[i] == '-';
            ++i;
        }
        if (i >= e) return 1;
        bool ed = false, pd = false;
        for (; i < e; ++i) {
            const char c = t[i];
            if (c >= '0' && c <= '9') {
                if (ex < 100000) ex = ex * 10 + (c - '0');
                ed = pd = true;
            } else if (c == '_' && pd && i + 1 < e && t[i + 1] >= '0' && t[i + 1] <= '9') {
                pd = false;
            } else {
                return 1;
            }
        }
        if (!ed) return 1;
        if (eneg) ex = -ex;
    }
    if (w == 0) {
        out = neg ? -0.0 : 0.0;
        return 0;
    }
    if (more) return 2;  // more than 19 significant digits
    const long long q = ex + drop - frac;
    double v;
    if (w <= (1ull << 53) && q >= -22 && q <= 22) {
        // Clinger: both operands exact, one correctly rounded operation
        double pw = 1.0;
        for (long long k = 0; k < (q < 0 ? -q : q); ++k) pw *= 10.0;  // exact for |q| <= 22
        v = q < 0 ? __ddiv_rn((double)w, pw) : __dmul_rn((double)w, pw);
    } else {
        unsigned long long bits;
        if (!eisel_lemire(w, q, bits)) return 2;
        v = __longlong_as_double((long long)bits);
    }
    out = neg ? -v : v;
    return 0;
}

struct TxArgs {
    const char *t;
    int64_t n, n_lines;
    const int64_t *start;
    const int64_t *slot;  // output slot of each data line
    int delim_mode;       // 0 auto, 1 whitespace, 2 comma
    int base;
    double default_w;
    int64_t n_nodes;      // declared, or -1
    const unsigned long long *first_data;
    unsigned long long *err;  // (line << 8 | code), atomicMin; ~0 none
    long long *max_index;
    int64_t *rows, *cols;
    double *w;
    unsigned char *fallback;  // per data slot: 1 = weight to be converted on the host
    unsigned *n_fallback;
};

__device__ __forceinline__ bool comma_mode(const TxArgs &a) {
    if (a.delim_mode != 0) return a.delim_mode == 2;
    const unsigned long long f = *a.first_data;
    if (f == ~0ull) return false;
    const Line L = stripped_line(a.t, a.n, a.start, (int64_t)f, a.n_lines);
    for (int64_t i = L.s; i < L.e; ++i)
        if (a.t[i] == ',') return true;
    return false;
}

__device__ __forceinline__ void fail(const TxArgs &a, int64_t k, int code) {
    atomicMin(a.err, ((unsigned long long)(k + 1) << 8) | (unsigned)code);
}

__global__ void k_tx_edges(TxArgs a) {
    const bool comma = comma_mode(a);
    long long top = -1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_lines;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = a.slot[k];
        if (a.slot[k + 1] == o) continue;  // not a data line
        const Line L = stripped_line(a.t, a.n, a.start, k, a.n_lines);
        const Fields f = split(a.t, L, comma);
        if (f.n != 2 && f.n != 3) {
            fail(a, k, TX_FIELDS);
            continue;
        }
        long long i, j;
        if (!parse_int(a.t, f.s[0], f.e[0], i)) {
            fail(a, k, TX_BAD_I);
            continue;
        }
        if (i < a.base) {
            fail(a, k, TX_BASE_I);
            continue;
        }
        if (!parse_int(a.t, f.s[1], f.e[1], j)) {
            fail(a, k, TX_BAD_J);
            continue;
        }
        if (j < a.base) {
            fail(a, k, TX_BASE_J);
            continue;
        }
        i -= a.base;
        j -= a.base;
        double w = a.default_w;
        a.fallback[o] = 0;
        if (f.n == 3) {
            const int r = parse_float(a.t, f.s[2], f.e[2], w);
            if (r == 1) {
                fail(a, k, TX_BAD_W);
                continue;
            }
            if (r == 2) {
                a.fallback[o] = 1;
                atomicAdd(a.n_fallback, 1u);
                w = 0.0;
            } else if (!isfinite(w)) {
                fail(a, k, TX_NONFINITE);
                continue;
            }
        }
        const long long hi = i > j ? i : j;
        if (a.n_nodes >= 0 && hi >= a.n_nodes) {
            fail(a, k, TX_RANGE);
            continue;
        }
        a.rows[o] = i;
        a.cols[o] = j;
        a.w[o] = w;
        if (hi > top) top = hi;
    }
    // block max, then one atomic
    for (int s = 16; s > 0; s >>= 1) top = max(top, (long long)__shfl_xor_sync(0xffffffffu, top, s));
    if ((threadIdx.x & 31) == 0 && top >= 0) atomicMax(a.max_index, top);
}

// label lines: per-line form (one field) or "node label" pairs, fixed by the
// first data line; outputs node (or -1 in per-line form) and label per slot
__global__ void k_tx_labels(TxArgs a) {
    const bool comma = comma_mode(a);
    bool pairs = false;
    {
        const unsigned long long fd = *a.first_data;
        if (fd != ~0ull) pairs = split(a.t, stripped_line(a.t, a.n, a.start, (int64_t)fd, a.n_lines), comma).n == 2;
    }
    long long top = -1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.n_lines;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = a.slot[k];
        if (a.slot[k + 1] == o) continue;
        const Line L = stripped_line(a.t, a.n, a.start, k, a.n_lines);
        const Fields f = split(a.t, L, comma);
        a.rows[o] = -2;  // a failed line assigns nothing
        if ((unsigned long long)k == *a.first_data && f.n != 1 && f.n != 2) {
            fail(a, k, TX_FIELDS);
            continue;
        }
        long long node = -1, lab;
        if (pairs) {
            if (f.n != 2) {
                fail(a, k, TX_FIELDS_PAIR);
                continue;
            }
            if (!parse_int(a.t, f.s[0], f.e[0], node)) {
                fail(a, k, TX_BAD_I);
                continue;
            }
            if (node < a.base) {
                fail(a, k, TX_BASE_I);
                continue;
            }
            node -= a.base;
            if (!parse_int(a.t, f.s[1], f.e[1], lab)) {
                fail(a, k, TX_BAD_LABEL);
                continue;
            }
            if (lab < -1) {
                fail(a, k, TX_LABEL_LOW);
                continue;
            }
            if (a.n_nodes >= 0 && node >= a.n_nodes) {
                fail(a, k, TX_RANGE);
                continue;
            }
            if (node > top) top = node;
        } else {
            if (f.n != 1) {
                fail(a, k, TX_FIELDS_SEQ);
                continue;
            }
            if (!parse_int(a.t, f.s[0], f.e[0], lab)) {
                fail(a, k, TX_BAD_LABEL);
                continue;
            }
            if (lab < -1) {
                fail(a, k, TX_LABEL_LOW);
                continue;
            }
        }
        a.rows[o] = node;
        a.cols[o] = lab;
    }
    for (int s = 16; s > 0; s >>= 1) top = max(top, (long long)__shfl_xor_sync(0xffffffffu, top, s));
    if ((threadIdx.x & 31) == 0 && top >= 0) atomicMax(a.max_index, top);
}

// pair form: the first line naming a node (atomicMin over slots, slots are
// in file order) fixes its label; a later line with another label is the
// reference's "conflicting labels" error at that line
__global__ void k_tx_first(const int64_t *node, int64_t m, unsigned long long *first) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < m; o += (int64_t)gridDim.x * blockDim.x)
        if (node[o] >= 0) atomicMin(first + node[o], (unsigned long long)o);
}

__global__ void k_tx_assign(const int64_t *node, const int64_t *lab, const int64_t *slot_line, int64_t m,
                            const unsigned long long *first, int64_t nv, int64_t *values,
                            unsigned long long *err) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long f = first[v];
        values[v] = f == ~0ull ? -1 : lab[f];
    }
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < m; o += (int64_t)gridDim.x * blockDim.x) {
        if (node[o] < 0) continue;
        const unsigned long long f = first[node[o]];
        if (lab[o] != lab[f]) atomicMin(err, ((unsigned long long)(slot_line[o] + 1) << 8) | (unsigned)TX_CONFLICT);
    }
}

// data slot -> file line (for errors found after compaction)
__global__ void k_tx_slot_line(const int64_t *slot, int64_t n_lines, int64_t *slot_line) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_lines;
         k += (int64_t)gridDim.x * blockDim.x)
        if (slot[k + 1] != slot[k]) slot_line[slot[k]] = k;
}

struct TxWs {
    unsigned *chunk_cnt;
    int64_t *chunk_base;
    unsigned *flag;
    int64_t *slot;
    unsigned long long *ctl;  // [0] first data line, [1] err, [2] max index (as long long), [3] n_fallback
    void *scan;
    size_t scan_bytes;
};

size_t carve_tx(Carver &cv, TxWs &w, int64_t nbytes, int64_t n_lines) {
    const int64_t chunks = (nbytes + kTxChunk - 1) / kTxChunk + 1;
    const int64_t big = chunks > n_lines ? chunks : n_lines;
    w.chunk_cnt = cv.take<unsigned>((size_t)chunks);
    w.chunk_base = cv.take<int64_t>((size_t)chunks + 1);
    w.flag = cv.take<unsigned>((size_t)n_lines + 1);
    w.slot = cv.take<int64_t>((size_t)n_lines + 1);
    w.ctl = cv.take<unsigned long long>(8);
    w.scan_bytes = scan_workspace(big + 1);
    w.scan = cv.take<char>(w.scan_bytes);
    return cv.bytes();
}

}  // namespace
}  // namespace gee

using namespace gee;

extern "C" {

int gee_text_workspace(int64_t nbytes, int64_t n_lines, size_t *ws_bytes) {
    if (nbytes < 0 || n_lines < 0 || !ws_bytes) return GEE_E_ARG;
    Carver cv(nullptr);
    TxWs w;
    *ws_bytes = carve_tx(cv, w, nbytes, n_lines);
    return GEE_OK;
}

/* *n_breaks (device int64) = line breaks in the text; the parsers take
 * n_lines = n_breaks + 1 (a final empty line is blank). */
int gee_text_count_lines(const char *text, int64_t nbytes, int64_t *n_breaks, void *ws, size_t ws_bytes,
                         void *stream) {
    int64_t *n_lines = n_breaks;
    if (nbytes < 0 || !n_lines || (nbytes && !text)) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    Carver cv(ws);
    TxWs W;
    if (carve_tx(cv, W, nbytes, 0) > ws_bytes || !ws) return GEE_E_WORKSPACE;
    const int64_t chunks = (nbytes + kTxChunk - 1) / kTxChunk;
    if (chunks == 0) {
        GEE_CHECK_CUDA(cudaMemsetAsync(n_lines, 0, sizeof(int64_t), st));
        return GEE_OK;
    }
    k_tx_count<<<(unsigned)chunks, 512, 0, st>>>(text, nbytes, W.chunk_cnt);
    GEE_CHECK_LAUNCH("k_tx_count");
    // lines = breaks + (1 if the text does not end with a break)
    int rc = exclusive_scan_u32(W.chunk_cnt, chunks, W.chunk_base, W.scan, st);
    if (rc) return rc;
    GEE_CHECK_CUDA(cudaMemcpyAsync(n_lines, W.chunk_base + chunks, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    return GEE_OK;
}

static int tx_prepare(const char *text, int64_t nbytes, int64_t n_lines, TxWs &W, int64_t *line_start,
                      cudaStream_t st) {
    const int64_t chunks = (nbytes + kTxChunk - 1) / kTxChunk;
    GEE_CHECK_CUDA(cudaMemsetAsync(W.ctl, 0xff, 8 * sizeof(unsigned long long), st));
    GEE_CHECK_CUDA(cudaMemsetAsync(W.ctl + 2, 0xff, sizeof(unsigned long long), st));  // max index -1
    GEE_CHECK_CUDA(cudaMemsetAsync(W.ctl + 3, 0, sizeof(unsigned long long), st));
    k_tx_count<<<(unsigned)chunks, 512, 0, st>>>(text, nbytes, W.chunk_cnt);
    GEE_CHECK_LAUNCH("k_tx_count");
    int rc = exclusive_scan_u32(W.chunk_cnt, chunks, W.chunk_base, W.scan, st);
    if (rc) return rc;
    k_tx_index<<<(unsigned)chunks, 512, 0, st>>>(text, nbytes, W.chunk_base, line_start);
    GEE_CHECK_LAUNCH("k_tx_index");
    k_tx_class<<<grid_for(n_lines, 256, 8), 256, 0, st>>>(text, nbytes, line_start, n_lines, W.flag, W.ctl + 0);
    GEE_CHECK_LAUNCH("k_tx_class");
    return exclusive_scan_u32(W.flag, n_lines, W.slot, W.scan, st);
}

/* info (device int64[6]): [0] data lines, [1] max index (-1 none),
 * [2] error (line << 8 | code; -1 none), [3] weights left to the host,
 * [4] first data line (-1 none). */
int gee_parse_edges(const char *text, int64_t nbytes, int64_t n_lines, int delim_mode, int index_base,
                    double default_weight, int64_t n_nodes, int64_t *line_start, int64_t *rows, int64_t *cols,
                    double *w, unsigned char *fallback, int64_t *slot_line, int64_t *info, void *ws, size_t ws_bytes,
                    void *stream) {
    if (nbytes < 1 || n_lines < 1 || !text || !line_start || !rows || !cols || !w || !fallback || !info)
        return GEE_E_ARG;
    if (delim_mode < 0 || delim_mode > 2 || (index_base != 0 && index_base != 1)) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    Carver cv(ws);
    TxWs W;
    if (carve_tx(cv, W, nbytes, n_lines) > ws_bytes || !ws) return GEE_E_WORKSPACE;
    int rc = tx_prepare(text, nbytes, n_lines, W, line_start, st);
    if (rc) return rc;
    TxArgs a;
    a.t = text;
    a.n = nbytes;
    a.n_lines = n_lines;
    a.start = line_start;
    a.slot = W.slot;
    a.delim_mode = delim_mode;
    a.base = index_base;
    a.default_w = default_weight;
    a.n_nodes = n_nodes;
    a.first_data = W.ctl + 0;
    a.err = W.ctl + 1;
    a.max_index = reinterpret_cast<long long *>(W.ctl + 2);
    a.n_fallback = reinterpret_cast<unsigned *>(W.ctl + 3);
    a.rows = rows;
    a.cols = cols;
    a.w = w;
    a.fallback = fallback;
    k_tx_edges<<<grid_for(n_lines, 256, 8), 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_tx_edges");
    if (slot_line) {
        k_tx_slot_line<<<grid_for(n_lines, 256, 8), 256, 0, st>>>(W.slot, n_lines, slot_line);
        GEE_CHECK_LAUNCH("k_tx_slot_line");
    }
    // info: data lines, max index, error word, fallback count, first data line
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 0, W.slot + n_lines, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 1, W.ctl + 2, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 2, W.ctl + 1, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 3, W.ctl + 3, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 4, W.ctl + 0, 8, cudaMemcpyDeviceToDevice, st));
    return GEE_OK;
}

/* Phase 1 of the label parser: node (-1 in per-line form) and label per data
 * line into node/lab (capacity n_lines), slot_line = the file line of each
 * data slot; info as gee_parse_edges ([1] = max node). */
int gee_parse_labels(const char *text, int64_t nbytes, int64_t n_lines, int delim_mode, int index_base,
                     int64_t n_nodes, int64_t *line_start, int64_t *node, int64_t *lab, int64_t *slot_line,
                     int64_t *info, void *ws, size_t ws_bytes, void *stream) {
    if (nbytes < 1 || n_lines < 1 || !text || !line_start || !node || !lab || !slot_line || !info) return GEE_E_ARG;
    if (delim_mode < 0 || delim_mode > 2 || (index_base != 0 && index_base != 1)) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    Carver cv(ws);
    TxWs W;
    if (carve_tx(cv, W, nbytes, n_lines) > ws_bytes || !ws) return GEE_E_WORKSPACE;
    int rc = tx_prepare(text, nbytes, n_lines, W, line_start, st);
    if (rc) return rc;
    TxArgs a{};
    a.t = text;
    a.n = nbytes;
    a.n_lines = n_lines;
    a.start = line_start;
    a.slot = W.slot;
    a.delim_mode = delim_mode;
    a.base = index_base;
    a.n_nodes = n_nodes;
    a.first_data = W.ctl + 0;
    a.err = W.ctl + 1;
    a.max_index = reinterpret_cast<long long *>(W.ctl + 2);
    a.rows = node;
    a.cols = lab;
    k_tx_labels<<<grid_for(n_lines, 256, 8), 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_tx_labels");
    k_tx_slot_line<<<grid_for(n_lines, 256, 8), 256, 0, st>>>(W.slot, n_lines, slot_line);
    GEE_CHECK_LAUNCH("k_tx_slot_line");
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 0, W.slot + n_lines, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 1, W.ctl + 2, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 2, W.ctl + 1, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 3, W.ctl + 3, 8, cudaMemcpyDeviceToDevice, st));
    GEE_CHECK_CUDA(cudaMemcpyAsync(info + 4, W.ctl + 0, 8, cudaMemcpyDeviceToDevice, st));
    return GEE_OK;
}

/* Phase 2 (pair form): values int64[nv] (-1 for unmentioned nodes); a
 * conflicting duplicate ORs its (line << 8 | code) into *err_word (atomicMin;
 * initialise to ~0).  first is scratch uint64[nv]. */
int gee_labels_assign(const int64_t *node, const int64_t *lab, const int64_t *slot_line, int64_t m, int64_t nv,
                      uint64_t *first, int64_t *values, uint64_t *err_word, void *stream) {
    if (m < 0 || nv < 0 || (m && (!node || !lab || !slot_line)) || (nv && (!first || !values)) || !err_word)
        return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (nv) GEE_CHECK_CUDA(cudaMemsetAsync(first, 0xff, sizeof(uint64_t) * (size_t)nv, st));
    if (m) {
        k_tx_first<<<grid_for(m, 256, 8), 256, 0, st>>>(node, m, reinterpret_cast<unsigned long long *>(first));
        GEE_CHECK_LAUNCH("k_tx_first");
    }
    const int64_t big = m > nv ? m : nv;
    if (big) {
        k_tx_assign<<<grid_for(big, 256, 8), 256, 0, st>>>(node, lab, slot_line, m,
                                                           reinterpret_cast<const unsigned long long *>(first), nv,
                                                           values, reinterpret_cast<unsigned long long *>(err_word));
        GEE_CHECK_LAUNCH("k_tx_assign");
    }
    return GEE_OK;
}

}  // extern "C"
