// k_bitmap.cu -- the whole encode for unit-weight graphs with at most
// kBmMax nodes (configs 0/1: unweighted SBM, N = 10^4).
//
// With every weight equal to 1.0 a stored value is the multiplicity of its
// (row, col) pair, and the order duplicates are summed in is irrelevant (sums
// of ones are exact).  When no pair repeats, the CSR row of r is the set of
// its columns, its degree is the set size and
//     Z[r, q] = s_r * sum_{c in row r, Y_c = q} s_c / n_q   (+ the A+I diagonal),
// so the encode needs only the N x N adjacency bitmap -- Np^2/8 bytes, 13 MB at
// N = 10^4 -- which stays resident in the 126 MB L2.  The CSR itself is never
// materialised (gee_encode_edges returns Z only).
//   k_bm_set   one read of the int64 edge list; each stream entry sets bit
//              (r, c) with a global atomicOr.  Lanes holding the same bitmap
//              word (adjacent entries of a row-major list) OR-combine first,
//              so a sorted list costs about one atomic per word.  A bit that
//              was already set is a repeated pair: flags[0].
//   k_bm_sym   undirected lists: S = U | U^T in place, 256 x 256-bit block
//              pairs, 32 x 32 transposes by warp shuffles.  A pair present in
//              both directions (U & U^T off the diagonal) is a repeat too.
//   k_bm_scan  one warp per row: u_r = popc(S_r), degree d_r = u_r (+1 under
//              A+I), s_r = d_r^-1/2 and the node table {Y_r, g_r = s_r/n_Y_r}
//   k_bm_rows  one warp per row, 1024-thread CTAs sharing one shared-memory
//              copy of the node table: Z[r, :] from the set bits of S_r, the
//              diagonal, s_r and the correlation epilogue.
// Rare path (any repeated pair; each kernel exits at once otherwise): exact
// stream lengths by atomics (k_bm_len) and, for rows whose length differs
// from their distinct count, the per-class sums of g over every stream entry
// (k_bm_zsum), which k_bm_rows uses instead of the bitmap sum.
#include "gee_common.cuh"

namespace gee {

constexpr int kBmMax = 16384;   // nodes: bitmap Np^2/8 <= 32 MB (L2-resident)
constexpr int kBlk = 256;       // rows / columns of a k_bm_sym block
constexpr int kSetThreads = 512;
constexpr int kRowsNT = 1024;   // one CTA per SM, one node table per SM
constexpr int kWordsPerLane = kBmMax / 32 / 32;
constexpr int kZacc = 8;        // rare-path class sums per row (K <= 8)

struct BmArgs {
    int n, Wp;                // nodes, bitmap words per row (multiple of 8)
    int nb;                   // 256-row blocks
    unsigned *bm;             // [Np][Wp]
    unsigned *len;            // [n] stream lengths (rare path)
    unsigned *flags;          // [0] a repeated pair was seen
    unsigned *ucnt;           // [n] distinct columns per row
    double *zacc;             // [n][kZacc] rare path class sums
    double *deg, *scale;
    const int32_t *y32;
    const double *inv;
    double *tab_g;
    signed char *tab_lab;
    unsigned flags_opts;      // GEE_LAPLACIAN | GEE_DIAGONAL | GEE_CORRELATION
    double *z;
    int k;
    int32_t *err;
};

__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// 32 x 32 bit transpose across a warp: out(lane i) bit j = in(lane j) bit i
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
    const unsigned m16 = 0x0000ffffu, m8 = 0x00ff00ffu, m4 = 0x0f0f0f0fu, m2 = 0x33333333u, m1 = 0x55555555u;
#define GEE_TSTAGE(J, M)                                                  \
    {                                                                     \
        const unsigned y = __shfl_xor_sync(0xffffffffu, x, J);            \
        x = (lane & J) ? ((x & ~M) | ((y >> J) & M)) : ((x & M) | ((y & M) << J)); \
    }
    GEE_TSTAGE(16, m16)
    GEE_TSTAGE(8, m8)
    GEE_TSTAGE(4, m4)
    GEE_TSTAGE(2, m2)
    GEE_TSTAGE(1, m1)
#undef GEE_TSTAGE
    return x;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSetThreads) k_bm_set(const int64_t *__restrict__ rows,
                                                        const int64_t *__restrict__ cols, int64_t E, BmArgs a) {
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    const unsigned le = lanemask_le();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
    bool rep = false;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; e0 - threadIdx.x < E; e0 += stride) {
        unsigned key[U], bit[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + (int64_t)u * blockDim.x;
            const unsigned r = e < E ? (unsigned)__ldcs(rows + e) : 0u;
            const unsigned c = e < E ? (unsigned)__ldcs(cols + e) : 0u;
            key[u] = e < E ? r * (unsigned)a.Wp + (c >> 5) : 0xffffffffu;
            bit[u] = e < E ? 1u << (c & 31) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // segmented OR over runs of lanes holding the same word
            const unsigned kp = __shfl_up_sync(0xffffffffu, key[u], 1);
            const unsigned kn = __shfl_down_sync(0xffffffffu, key[u], 1);
            const bool head = lane == 0 || kp != key[u];
            const bool tail = lane == 31 || kn != key[u];
            const int start = 31 - __clz(__ballot_sync(0xffffffffu, head) & le);
            unsigned incl = bit[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane - o >= start) incl |= y;
            }
            const unsigned prev = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane > start && (prev & bit[u])) rep = true;  // repeated inside the run
            if (tail && key[u] != 0xffffffffu) {
                const unsigned old = atomicOr(&a.bm[key[u]], incl);
                if (old & incl) rep = true;
            }
        }
    }
    if (__any_sync(0xffffffffu, rep) && lane == 0) a.flags[0] = 1u;
}

// S = U | U^T for the block pair (BI, BJ), BI <= BJ, in place
__global__ void __launch_bounds__(kBlk) k_bm_sym(BmArgs a) {
    __shared__ unsigned sat[kBlk][9], sbt[kBlk][9];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // linear index -> (BI, BJ) on the upper triangle
    const unsigned x = blockIdx.x;
    unsigned bj = (unsigned)((sqrt(8.0 * x + 1.0) - 1.0) * 0.5);
    while ((bj + 1) * (bj + 2) / 2 <= x) ++bj;
    while (bj * (bj + 1) / 2 > x) --bj;
    const unsigned bi = x - bj * (bj + 1) / 2;
    const size_t Wp = (size_t)a.Wp;
    uint4 *pa = reinterpret_cast<uint4 *>(a.bm + ((size_t)bi * kBlk + t) * Wp + (size_t)bj * 8);
    uint4 *pb = reinterpret_cast<uint4 *>(a.bm + ((size_t)bj * kBlk + t) * Wp + (size_t)bi * 8);
    unsigned av[8], bv[8];
    {
        const uint4 a0 = __ldcg(pa), a1 = __ldcg(pa + 1);
        av[0] = a0.x, av[1] = a0.y, av[2] = a0.z, av[3] = a0.w, av[4] = a1.x, av[5] = a1.y, av[6] = a1.z, av[7] = a1.w;
    }
    const bool same = bi == bj;
    if (!same) {
        const uint4 b0 = __ldcg(pb), b1 = __ldcg(pb + 1);
        bv[0] = b0.x, bv[1] = b0.y, bv[2] = b0.z, bv[3] = b0.w, bv[4] = b1.x, bv[5] = b1.y, bv[6] = b1.z, bv[7] = b1.w;
    }
    // tile (w, q) of a block transposes into row q*32+lane, word w of its mirror
#pragma unroll
    for (int q = 0; q < 8; ++q) sat[q * 32 + lane][w] = transpose32(av[q], lane);
    if (!same) {
#pragma unroll
        for (int q = 0; q < 8; ++q) sbt[q * 32 + lane][w] = transpose32(bv[q], lane);
    }
    __syncthreads();
    unsigned mut = 0;
    if (same) {
        unsigned s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned tq = sat[t][q];
            s[q] = av[q] | tq;
            unsigned m = av[q] & tq;
            if (q == w) m &= ~(1u << lane);  // the diagonal is its own mirror
            mut |= m;
        }
        pa[0] = make_uint4(s[0], s[1], s[2], s[3]);
        pa[1] = make_uint4(s[4], s[5], s[6], s[7]);
    } else {
        unsigned s[8], u[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const unsigned tb = sbt[t][q], ta = sat[t][q];
            s[q] = av[q] | tb;
            u[q] = bv[q] | ta;
            mut |= av[q] & tb;
        }
        pa[0] = make_uint4(s[0], s[1], s[2], s[3]);
        pa[1] = make_uint4(s[4], s[5], s[6], s[7]);
        pb[0] = make_uint4(u[0], u[1], u[2], u[3]);
        pb[1] = make_uint4(u[4], u[5], u[6], u[7]);
    }
    if (__syncthreads_or(mut != 0) && t == 0) a.flags[0] = 1u;
}

// one warp per row, 8 rows per CTA
__global__ void __launch_bounds__(256) k_bm_scan(BmArgs a) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= a.n) return;
    const uint4 *row = reinterpret_cast<const uint4 *>(a.bm + (size_t)r * a.Wp);
    unsigned u = 0;
    for (int i = lane; i < a.Wp / 4; i += 32) {
        const uint4 v = __ldcg(row + i);
        u += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    u = warp_sum_u(u);
    if (lane == 0) {
        const unsigned L = __ldcg(a.flags) ? __ldcg(a.len + r) : u;  // stream length of the row
        double sr = 1.0;
        if (a.flags_opts & GEE_LAPLACIAN) {
            const double d = (double)L + ((a.flags_opts & GEE_DIAGONAL) ? 1.0 : 0.0);
            a.deg[r] = d;
            sr = laplacian_scale(d, a.err);
            a.scale[r] = sr;
        }
        const int lab = a.y32[r];
        a.tab_g[r] = lab < 0 ? 0.0 : ((a.flags_opts & GEE_LAPLACIAN) ? sr * a.inv[lab] : a.inv[lab]);
        a.tab_lab[r] = (signed char)lab;
        a.ucnt[r] = u;
    }
}

// rare path 1: exact stream lengths; clears the class sums
__global__ void k_bm_len(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols, int64_t E,
                         int directed, BmArgs a) {
    if (!__ldcg(a.flags)) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = i0; i < (int64_t)a.n * kZacc; i += stride) a.zacc[i] = 0.0;
    for (int64_t e = i0; e < E; e += stride) {
        const unsigned r = (unsigned)rows[e], c = (unsigned)cols[e];
        atomicAdd(&a.len[r], 1u);
        if (!directed && r != c) atomicAdd(&a.len[c], 1u);
    }
}

// rare path 2: per-class sums of g over every stream entry of rows with repeats
__global__ void k_bm_zsum(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols, int64_t E,
                          int directed, BmArgs a) {
    if (!__ldcg(a.flags)) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const unsigned r = (unsigned)rows[e], c = (unsigned)cols[e];
        if (a.len[r] != a.ucnt[r] && a.tab_lab[c] >= 0)
            atomicAdd(&a.zacc[(size_t)r * kZacc + a.tab_lab[c]], a.tab_g[c]);
        if (!directed && r != c && a.len[c] != a.ucnt[c] && a.tab_lab[r] >= 0)
            atomicAdd(&a.zacc[(size_t)c * kZacc + a.tab_lab[r]], a.tab_g[r]);
    }
}

// ---------------------------------------------------------------------------
template <int KP>
__global__ void __launch_bounds__(kRowsNT) k_bm_rows(BmArgs a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int kWarps = kRowsNT / 32;
    double *tg = reinterpret_cast<double *>(sm_raw);                            // [n]
    signed char *tl = reinterpret_cast<signed char *>(tg + ((a.n + 1) & ~1));   // [n]
    // stage the node table (written by k_bm_scan) with 16-byte loads
    {
        const int n2 = a.n / 2;
        const double2 *src = reinterpret_cast<const double2 *>(a.tab_g);
        double2 *dst = reinterpret_cast<double2 *>(tg);
        for (int j = threadIdx.x; j < n2; j += blockDim.x) dst[j] = __ldcg(src + j);
        if ((a.n & 1) && threadIdx.x == 0) tg[a.n - 1] = __ldcg(a.tab_g + a.n - 1);
        const int n16 = a.n / 16;
        const int4 *ls = reinterpret_cast<const int4 *>(a.tab_lab);
        for (int j = threadIdx.x; j < n16; j += blockDim.x) reinterpret_cast<int4 *>(tl)[j] = __ldcg(ls + j);
        for (int j = n16 * 16 + threadIdx.x; j < a.n; j += blockDim.x) tl[j] = a.tab_lab[j];
    }
    __syncthreads();
    const bool lap = (a.flags_opts & GEE_LAPLACIAN) != 0, diag = (a.flags_opts & GEE_DIAGONAL) != 0;
    const int Wp = a.Wp;
    const bool any_rep = __ldcg(a.flags) != 0;
    for (int r = blockIdx.x * kWarps + wid; r < a.n; r += gridDim.x * kWarps) {
        double acc[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) acc[q] = 0.0;
        if (any_rep && __ldcg(a.len + r) != __ldcg(a.ucnt + r)) {
            // a row with repeated pairs: its class sums come from k_bm_zsum
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < KP; ++q) acc[q] = __ldcg(a.zacc + (size_t)r * kZacc + q);
            }
        } else {
            const unsigned *row = a.bm + (size_t)r * Wp;
            unsigned wv[kWordsPerLane];
#pragma unroll
            for (int i = 0; i < kWordsPerLane; ++i) {
                const int w = i * 32 + lane;
                wv[i] = w < Wp ? __ldcg(row + w) : 0u;
            }
#pragma unroll
            for (int i = 0; i < kWordsPerLane; ++i) {
                unsigned word = wv[i];
                const int base = (i * 32 + lane) * 32;
                while (word) {
                    const int c = base + __ffs(word) - 1;
                    word &= word - 1;
                    const int lab = tl[c];
                    const double x = tg[c];
#pragma unroll
                    for (int q = 0; q < KP; ++q) acc[q] += (lab == q) ? x : 0.0;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) acc[q] = warp_sum(acc[q]);
        if (diag) {
            // A+I: the diagonal gains 1.0 whether or not (r, r) is stored
            const int lab = tl[r];
            const double x = tg[r];
#pragma unroll
            for (int q = 0; q < KP; ++q) acc[q] += (lab == q) ? x : 0.0;
        }
        if (lap) {
            const double sr = __ldcg(a.scale + r);
#pragma unroll
            for (int q = 0; q < KP; ++q) acc[q] *= sr;
        }
        if (a.flags_opts & GEE_CORRELATION) {
            double ss = 0.0;
            bool fin = true;
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                if (q < a.k) {
                    ss += acc[q] * acc[q];
                    fin &= isfinite(acc[q]);
                }
            }
            if (!fin) {
                if (lane == 0) raise_err(a.err, GEE_ERR_NONFINITE);
            } else {
                const double nrm = __dsqrt_rn(ss);
                if (nrm > 0.0) {
#pragma unroll
                    for (int q = 0; q < KP; ++q) acc[q] = __ddiv_rn(acc[q], nrm);
                }
            }
        }
        double mine = 0.0;
#pragma unroll
        for (int q = 0; q < KP; ++q) mine = (lane == q) ? acc[q] : mine;
        if (lane < a.k) a.z[(int64_t)r * a.k + lane] = mine;
    }
}

// ---------------------------------------------------------------------------
int force_path();

// unit weights, square, at most kBmMax nodes, K <= 8 (register accumulators)
bool bitmap_path_ok(int wt, int64_t E, int64_t n_rows, int64_t n_cols, int directed, int k) {
    if (force_path() != 0) return false;  // test hook: exercise the general paths
    const int64_t M = directed ? E : 2 * E;
    return wt == GEE_W_UNIT && n_rows == n_cols && n_rows >= 1 && n_rows <= kBmMax && k >= 1 && k <= kZacc &&
           M < ((int64_t)1 << 31);
}

struct BmWs {
    unsigned *bm, *len, *flags, *ucnt;
    double *zacc, *tab_g;
    signed char *tab_lab;
    int Wp, nb;
    size_t clear_words;
};

static void carve_bm(Carver &cv, BmWs &w, int64_t n) {
    const int64_t np = (n + kBlk - 1) / kBlk * kBlk;
    w.nb = (int)(np / kBlk);
    w.Wp = (int)(np / 32);
    // bitmap, stream lengths and flags are contiguous: one memset clears them
    w.clear_words = (size_t)np * w.Wp + (size_t)n + 4;
    w.bm = cv.take<unsigned>(w.clear_words);
    w.len = w.bm ? w.bm + (size_t)np * w.Wp : nullptr;
    w.flags = w.bm ? w.len + n : nullptr;
    w.ucnt = cv.take<unsigned>((size_t)n);
    w.zacc = cv.take<double>((size_t)n * kZacc);
    w.tab_g = cv.take<double>((size_t)n + 2);
    w.tab_lab = cv.take<signed char>((size_t)n + 16);
}

size_t bitmap_workspace(int64_t E, int64_t n, int directed) {
    (void)E;
    (void)directed;
    Carver cv(nullptr);
    BmWs w;
    carve_bm(cv, w, n);
    return cv.bytes();
}

// The fused encode for unit-weight graphs.  Outputs: Z (n x k) and, under
// the Laplacian, deg / scale.  The CSR is not materialised.
int bitmap_encode(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed,
                  const int32_t *y32, const double *inv, int k, unsigned flags, double *deg, double *scale,
                  double *z, void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, n);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    BmArgs a;
    a.n = (int)n;
    a.Wp = W.Wp;
    a.nb = W.nb;
    a.bm = W.bm;
    a.len = W.len;
    a.flags = W.flags;
    a.ucnt = W.ucnt;
    a.zacc = W.zacc;
    a.deg = deg;
    a.scale = scale;
    a.y32 = y32;
    a.inv = inv;
    a.tab_g = W.tab_g;
    a.tab_lab = W.tab_lab;
    a.flags_opts = flags;
    a.z = z;
    a.k = k;
    a.err = err;
    const size_t rows_smem = 8 * (size_t)((n + 1) & ~1) + (size_t)((n + 15) & ~15);
    static bool attr = false;
    if (!attr) {
        const int mx = (int)(8 * (size_t)kBmMax + kBmMax);
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_rows<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_rows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        attr = true;
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(W.bm, 0, sizeof(unsigned) * W.clear_words, st));
    if (E > 0) {
        k_bm_set<<<grid_for(E, kSetThreads * 4, 8), kSetThreads, 0, st>>>(rows, cols, E, a);
        GEE_CHECK_LAUNCH("k_bm_set");
        if (!directed) {
            k_bm_sym<<<(unsigned)(W.nb * (W.nb + 1) / 2), kBlk, 0, st>>>(a);
            GEE_CHECK_LAUNCH("k_bm_sym");
        }
        k_bm_len<<<grid_for(E, 256, 2), 256, 0, st>>>(rows, cols, E, directed, a);
        GEE_CHECK_LAUNCH("k_bm_len");
    }
    k_bm_scan<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_bm_scan");
    if (E > 0) {
        k_bm_zsum<<<grid_for(E, 256, 2), 256, 0, st>>>(rows, cols, E, directed, a);
        GEE_CHECK_LAUNCH("k_bm_zsum");
    }
    const unsigned grid = (unsigned)num_sms();
    if (k <= 1)
        k_bm_rows<1><<<grid, kRowsNT, rows_smem, st>>>(a);
    else if (k <= 2)
        k_bm_rows<2><<<grid, kRowsNT, rows_smem, st>>>(a);
    else if (k <= 4)
        k_bm_rows<4><<<grid, kRowsNT, rows_smem, st>>>(a);
    else
        k_bm_rows<8><<<grid, kRowsNT, rows_smem, st>>>(a);
    GEE_CHECK_LAUNCH("k_bm_rows_embed");
    return GEE_OK;
}

}  // namespace gee
