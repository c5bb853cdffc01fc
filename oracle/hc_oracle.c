/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU implementation of what the Hash Chain
 * (HC) searching phase computes (Palmer, Faro, Scafiti, arXiv 2310.15711).
 * Cited as P:n = line n of PAPER.md, S:n = line n of SPEC.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  The product path (paper_2310_15711_b200/) never
 * includes, links or calls anything here, and this file includes nothing
 * from the product path: the two share no code.
 *
 * Contents
 *   O1  or_brute        — the plain definition of exact matching:
 *                         every s in [s0, s1) with y[s..s+m-1] == x.
 *   O2  or_preprocess   — Fig. 3 "Preprocessing" transliterated.
 *       or_hc_search    — Fig. 5 "HC" transliterated, with the
 *                         verify/output index read as e-m+1 (R1).
 *       or_shc_search   — Fig. 5 "SHC" transliterated, same fix.
 *   primitives          — or_shift (Eq. 4), or_hash (Fig. 3 Hash / Eq. 3),
 *                         or_link_hash (Fig. 3 LinkHash / Eq. 5).
 *
 * Arithmetic: unsigned 64-bit accumulators, unsigned bytes 0..255 (DESIGN.md
 * readings R3, R5).  The word width w is a parameter (R2; the product fixes
 * w = 32), so words are held in uint64_t and w <= 64.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (SPEC worked examples, hand-evaluated hashes, closed forms, brute force on
 * exhaustive tiny inputs).  No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>

/* Eq. 4: s <- floor(alpha / q). */
int or_shift(int alpha, int q) { return alpha / q; }

/* Fig. 3 Hash(x, p, q, s, F'):
 *   v <- 0; for i <- p downto p-q+1: v <- (v << s) + x[i]; return v & F'. */
uint64_t or_hash(const uint8_t *x, int64_t p, int q, int s, uint64_t mask)
{
    uint64_t v = 0;
    for (int64_t i = p; i >= p - q + 1; --i)
        v = (v << s) + (uint64_t)x[i];
    return v & mask;
}

/* Fig. 3 LinkHash(v), Eq. 5: 1 << (v & (w-1)). */
uint64_t or_link_hash(uint64_t v, int w)
{
    return (uint64_t)1 << (v & (uint64_t)(w - 1));
}

static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* Fig. 3 Preprocessing(x, m, q, alpha).
 *   F        : caller array of 2^alpha words (uint64_t, low w bits used).
 *   hv_out   : H_v (line 13).
 *   trace    : optional (may be NULL); receives the end index p of every
 *              Hash(x, p, ...) call in the order the pseudocode makes them,
 *              capacity >= m + q entries; *ntrace receives the count.
 * Returns 0, or -1 if the parameters are outside 1 <= q <= m, 1 <= alpha <= 30,
 * w in {1,...,64} a power of two. */
int or_preprocess(const uint8_t *x, int64_t m, int q, int alpha, int w,
                  uint64_t *F, uint64_t *hv_out, int64_t *trace, int64_t *ntrace)
{
    if (q < 1 || m < q || alpha < 1 || alpha > 30 || w < 1 || w > 64 || (w & (w - 1)))
        return -1;
    int64_t nt = 0;
    int s = or_shift(alpha, q);                       /* line 1 */
    uint64_t Fp = ((uint64_t)1 << alpha) - 1;         /* line 2: F' */
    for (uint64_t i = 0; i <= Fp; ++i)                /* lines 3-4 */
        F[i] = 0;
    uint64_t v = 0, vp;
    for (int64_t i = min64(m - q + 1, q); i >= 1; --i) {  /* line 5 */
        v = or_hash(x, m - i, q, s, Fp);                  /* line 6 */
        if (trace) trace[nt] = m - i;
        nt++;
        int64_t j = m - i - q;                            /* line 7 */
        while (j >= q - 1) {                              /* line 8 */
            vp = v;                                       /* line 9 */
            v = or_hash(x, j, q, s, Fp);                  /* line 10 */
            if (trace) trace[nt] = j;
            nt++;
            F[vp] = F[vp] | or_link_hash(v, w);           /* line 11 */
            j = j - q;                                    /* line 12 */
        }
    }
    *hv_out = v;                                          /* line 13 */
    for (int64_t i = q - 1; i <= min64(2 * (int64_t)q - 1, m) - 1; ++i) { /* line 14 */
        v = or_hash(x, i, q, s, Fp);                      /* line 15 */
        if (trace) trace[nt] = i;
        nt++;
        if (F[v] == 0)                                    /* line 16 */
            F[v] = 1;                                     /* line 17 */
    }
    if (ntrace) *ntrace = nt;
    return 0;
}

/* Plain byte comparison y[0..m-1] == x[0..m-1]. */
static int eq_bytes(const uint8_t *a, const uint8_t *b, int64_t m)
{
    for (int64_t k = 0; k < m; ++k)
        if (a[k] != b[k]) return 0;
    return 1;
}

/* Search metrics (SPEC SearchMetrics, plus completed walks):
 *   met[0] windows, met[1] qgram_hashes, met[2] link_checks,
 *   met[3] verifications, met[4] hv_rejections, met[5] completed_walks,
 *   met[6] min shift of the window end, met[7] max shift. */
#define MET_N 8
static void met_shift(int64_t *met, int64_t d)
{
    if (!met) return;
    if (met[6] == 0 || d < met[6]) met[6] = d;
    if (d > met[7]) met[7] = d;
}

/* Fig. 5 HC(x, m, y, n, q, alpha) searching phase, given the
 * Preprocessing output (F, H_v).
 *
 * The loop starts at window end j = a (Fig. 5 line 2 uses a = m-1) and runs
 * "while j < b" (line 3 uses b = n).  With a = m-1, b = n this is the paper's
 * loop exactly; other (a, b) are used by tests of the segment argument
 * (R11) and by the host-threaded CPU baseline.
 *
 * Reading R1: the window verified at line 16 and the
 * position output at line 17 are those of the window whose end was e (the
 * j at line 4): y[e-m+1 .. e] and e-m+1.
 *
 * out may be NULL; positions beyond max_out are counted but not stored.
 * Returns the number of occurrences found. */
int64_t or_hc_search(const uint8_t *x, int64_t m, const uint8_t *y, int64_t n,
                     int q, int alpha, int w, const uint64_t *F, uint64_t hv,
                     int64_t a, int64_t b, int64_t *out, int64_t max_out,
                     int64_t *met)
{
    if (n < m) return 0;
    int s = or_shift(alpha, q);
    uint64_t Fp = ((uint64_t)1 << alpha) - 1;
    int64_t cnt = 0;
    int64_t j = a;                                        /* line 2 */
    while (j < b) {                                       /* line 3 */
        int64_t e = j, j_before = j;
        if (met) met[0]++;
        uint64_t v = or_hash(y, j, q, s, Fp);             /* line 4 */
        if (met) met[1]++;
        uint64_t z = F[v];                                /* line 5 */
        if (z != 0) {                                     /* line 6 */
            int64_t i = j - m + 2 * (int64_t)q;           /* line 7 */
            int broke = 0;
            while (j >= i) {                              /* line 8 */
                j = j - q;                                /* line 9 */
                v = or_hash(y, j, q, s, Fp);              /* line 10 */
                if (met) { met[1]++; met[2]++; }
                if ((z & or_link_hash(v, w)) == 0) {      /* line 11 */
                    broke = 1;                            /* line 12 */
                    break;
                }
                z = F[v];                                 /* line 13 */
            }
            if (!broke) {                                 /* line 14: else */
                j = i - q;                                /* line 15 */
                if (met) met[5]++;
                if (v == hv) {                            /* line 16 */
                    if (met) met[3]++;
                    if (eq_bytes(y + e - m + 1, x, m)) {
                        if (out && cnt < max_out) out[cnt] = e - m + 1; /* line 17 (R1) */
                        cnt++;
                    }
                } else if (met) {
                    met[4]++;
                }
            }
        }
        j = j + m - q + 1;                                /* line 18 */
        met_shift(met, j - j_before);
    }
    return cnt;
}

/* Fig. 5 SHC(x, m, y, n, q, alpha) searching phase.
 * buf must have capacity >= n + m: lines 2-3 write the sentinel copy of x
 * into buf[n .. n+m-1]; buf[0 .. n-1] is not modified.
 * Same R1 reading of lines 20-21 as HC. */
int64_t or_shc_search(const uint8_t *x, int64_t m, uint8_t *buf, int64_t n,
                      int q, int alpha, int w, const uint64_t *F, uint64_t hv,
                      int64_t *out, int64_t max_out, int64_t *met)
{
    if (n < m) return 0;
    int s = or_shift(alpha, q);
    uint64_t Fp = ((uint64_t)1 << alpha) - 1;
    for (int64_t i = 0; i <= m - 1; ++i)                  /* lines 2-3 */
        buf[n + i] = x[i];
    int64_t cnt = 0;
    int64_t j = m - 1;                                    /* line 4 */
    while (j < n) {                                       /* line 5 */
        while (F[or_hash(buf, j, q, s, Fp)] == 0) {       /* line 6 */
            if (met) { met[0]++; met[1]++; }
            j = j + m - q + 1;                            /* line 7 */
        }
        if (j < n) {                                      /* line 8 */
            int64_t e = j;
            if (met) met[0]++;
            uint64_t v = or_hash(buf, j, q, s, Fp);       /* line 9 */
            if (met) met[1]++;
            uint64_t z = F[v];                            /* line 10 */
            int64_t i = j - m + 2 * (int64_t)q;           /* line 11 */
            int broke = 0;
            while (j >= i) {                              /* line 12 */
                j = j - q;                                /* line 13 */
                v = or_hash(buf, j, q, s, Fp);            /* line 14 */
                if (met) { met[1]++; met[2]++; }
                if ((z & or_link_hash(v, w)) == 0) {      /* line 15 */
                    broke = 1;                            /* line 16 */
                    break;
                }
                z = F[v];                                 /* line 17 */
            }
            if (!broke) {                                 /* line 18: else */
                j = i - q;                                /* line 19 */
                if (met) met[5]++;
                if (v == hv) {                            /* line 20 */
                    if (met) met[3]++;
                    if (eq_bytes(buf + e - m + 1, x, m)) {
                        if (out && cnt < max_out) out[cnt] = e - m + 1; /* line 21 (R1) */
                        cnt++;
                    }
                } else if (met) {
                    met[4]++;
                }
            }
            j = j + m - q + 1;                            /* line 22 */
        }
    }
    return cnt;
}

/* O1: the plain definition.  Every s in [s0, s1) (clamped
 * to [0, n-m]) with y[s..s+m-1] == x, ascending.  Returns the count; stores
 * at most max_out positions when out != NULL. */
int64_t or_brute(const uint8_t *x, int64_t m, const uint8_t *y, int64_t n,
                 int64_t s0, int64_t s1, int64_t *out, int64_t max_out)
{
    if (m < 1 || n < m) return 0;
    if (s0 < 0) s0 = 0;
    if (s1 > n - m + 1) s1 = n - m + 1;
    int64_t cnt = 0;
    for (int64_t s = s0; s < s1; ++s) {
        int64_t k = 0;
        while (k < m && y[s + k] == x[k]) k++;
        if (k == m) {
            if (out && cnt < max_out) out[cnt] = s;
            cnt++;
        }
    }
    return cnt;
}
