/*
 * CPU ORACLE -- test infrastructure only.  Never linked into, or called by,
 * the product path (paper_2212_14191_b200/); only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs load it.
 *
 * Plain-C restatement of the reference's transform kernels
 * (/root/reference/pkg/src/rnsckks/ntt.py), used as the parity checker for
 * the sm_100a tensor-core NTT and as the timed CPU baseline ("port").
 *
 *   orc_ntt_tables   <- TwiddleTable.butterfly       ntt.py:155-165
 *                       (psi^brv(i), psi^-brv(i), n^-1; params.py:178-185)
 *   orc_ntt_rows     <- _butterfly_forward           ntt.py:172-186
 *                       _butterfly_inverse           ntt.py:189-205
 *                       transform_rows dispatch      ntt.py:347-363
 *   orc_ntt_direct   <- ntt_oracle (O(n^2))          ntt.py:44-59
 *   orc_mulmod_rows  <- hada_mult / scalar mult      kernels.py:43-58
 *
 * The reference computes every product as (u64 * u64) % q; here products
 * use the Shoup precomputation w' = floor(w * 2^32 / q), which is exact for
 * q < 2^31 and operands < q, so every output is bit-identical.  Rows are
 * independent (rns.py:1-4), so OpenMP splits the row loop.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint32_t mulmod_u64(uint32_t a, uint32_t b, uint32_t q) {
    return (uint32_t)(((uint64_t)a * b) % q);
}

static uint32_t powmod(uint32_t b, uint64_t e, uint32_t q) {
    uint64_t r = 1 % q, x = b % q;
    while (e) {
        if (e & 1) r = r * x % q;
        x = x * x % q;
        e >>= 1;
    }
    return (uint32_t)r;
}

static inline uint32_t shoup_pre(uint32_t w, uint32_t q) {
    return (uint32_t)(((uint64_t)w << 32) / q);
}

/* w * b mod q with w' = shoup_pre(w, q); exact for b < 2^32, q < 2^31 */
static inline uint32_t shoup_mul(uint32_t b, uint32_t w, uint32_t wp, uint32_t q) {
    uint32_t t = (uint32_t)(((uint64_t)wp * b) >> 32);
    uint32_t r = w * b - t * q;
    return r >= q ? r - q : r;
}

static inline uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* tables layout (uint32, length 4n + 2):
 *   [0,n)   psi^brv(i)          [n,2n)   shoup of it
 *   [2n,3n) psi^-brv(i)         [3n,4n)  shoup of it
 *   [4n]    n^-1                [4n+1]   shoup of n^-1                     */
int orc_ntt_tables(uint32_t q, uint32_t psi, int logn, uint32_t *tables) {
    if (q >= (1u << 31) || logn < 1 || logn > 20) return -1;
    uint32_t n = 1u << logn;
    uint32_t ipsi = powmod(psi, q - 2, q);
    uint32_t p = 1, ip = 1;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t r = bitrev(i, logn);
        tables[r] = p;
        tables[2 * n + r] = ip;
        p = mulmod_u64(p, psi, q);
        ip = mulmod_u64(ip, ipsi, q);
    }
    for (uint32_t i = 0; i < n; ++i) {
        tables[n + i] = shoup_pre(tables[i], q);
        tables[3 * n + i] = shoup_pre(tables[2 * n + i], q);
    }
    tables[4 * n] = powmod(n, q - 2, q);
    tables[4 * n + 1] = shoup_pre(tables[4 * n], q);
    return 0;
}

static void fwd_row(uint32_t *a, uint32_t *tmp, uint32_t n, int logn, uint32_t q,
                    const uint32_t *tab) {
    /* Cooley-Tukey DIT, bit-reversed output (ntt.py:175-185) */
    for (uint32_t m = 1, t = n; m < n; m <<= 1) {
        t >>= 1;
        for (uint32_t i = 0; i < m; ++i) {
            uint32_t w = tab[m + i], wp = tab[n + m + i];
            uint32_t *x = a + 2 * i * t;
            for (uint32_t j = 0; j < t; ++j) {
                uint32_t u = x[j];
                uint32_t v = shoup_mul(x[j + t], w, wp, q);
                uint32_t s = u + v;
                x[j] = s >= q ? s - q : s;
                x[j + t] = u >= v ? u - v : u + q - v;
            }
        }
    }
    /* natural order: out[k] = x[rev[k]]  (ntt.py:186) */
    memcpy(tmp, a, (size_t)n * 4);
    for (uint32_t k = 0; k < n; ++k) a[k] = tmp[bitrev(k, logn)];
}

static void inv_row(uint32_t *a, uint32_t *tmp, uint32_t n, int logn, uint32_t q,
                    const uint32_t *tab) {
    const uint32_t *it = tab + 2 * n, *itp = tab + 3 * n;
    memcpy(tmp, a, (size_t)n * 4);
    for (uint32_t k = 0; k < n; ++k) a[k] = tmp[bitrev(k, logn)];   /* ntt.py:194 */
    /* Gentleman-Sande DIF (ntt.py:195-204) */
    for (uint32_t t = 1, m = n; m > 1; t <<= 1) {
        uint32_t h = m >> 1;
        for (uint32_t i = 0; i < h; ++i) {
            uint32_t w = it[h + i], wp = itp[h + i];
            uint32_t *x = a + 2 * i * t;
            for (uint32_t j = 0; j < t; ++j) {
                uint32_t u = x[j], v = x[j + t];
                uint32_t s = u + v;
                x[j] = s >= q ? s - q : s;
                x[j + t] = shoup_mul(u >= v ? u - v : u + q - v, w, wp, q);
            }
        }
        m = h;
    }
    uint32_t ni = tab[4 * n], nip = tab[4 * n + 1];
    for (uint32_t k = 0; k < n; ++k) a[k] = shoup_mul(a[k], ni, nip, q);
}

/* In-place transform of `rows` rows of length 2^logn, all mod q.
 * Inputs must already be reduced (< q), as in transform_rows.            */
int orc_ntt_rows(uint32_t *data, int64_t rows, int logn, uint32_t q,
                 const uint32_t *tables, int inverse, int threads) {
    if (q >= (1u << 31)) return -1;
    uint32_t n = 1u << logn;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        uint32_t *tmp = (uint32_t *)malloc((size_t)n * 4);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t r = 0; r < rows; ++r) {
            uint32_t *a = data + r * (int64_t)n;
            if (inverse) inv_row(a, tmp, n, logn, q, tables);
            else fwd_row(a, tmp, n, logn, q, tables);
        }
        free(tmp);
    }
    return 0;
}

/* O(n^2) ground truth A_k = sum_m a_m psi^((2k+1)m) (ntt.py:44-59) */
int orc_ntt_direct(const uint32_t *a, uint32_t *out, int logn, uint32_t q, uint32_t psi) {
    uint32_t n = 1u << logn, n2 = 2 * n;
    uint32_t *pw = (uint32_t *)malloc((size_t)n2 * 4);
    pw[0] = 1;
    for (uint32_t i = 1; i < n2; ++i) pw[i] = mulmod_u64(pw[i - 1], psi, q);
    for (uint32_t k = 0; k < n; ++k) {
        uint64_t acc = 0;
        for (uint32_t m = 0; m < n; ++m) {
            uint64_t e = ((uint64_t)(2 * k + 1) * m) % n2;
            acc += mulmod_u64(a[m] % q, pw[e], q);
            if (acc >= (1ull << 62)) acc %= q;
        }
        out[k] = (uint32_t)(acc % q);
    }
    free(pw);
    return 0;
}

/* out[r][i] = a[r][i] * b[r][i] mod q_r  (hada_mult, kernels.py:43-47) */
void orc_mulmod_rows(const uint32_t *a, const uint32_t *b, uint32_t *out,
                     int64_t rows, int64_t len, const uint32_t *q_per_row, int threads) {
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for num_threads(threads) schedule(static)
#endif
    for (int64_t r = 0; r < rows; ++r) {
        uint32_t q = q_per_row[r];
        for (int64_t i = 0; i < len; ++i)
            out[r * len + i] = mulmod_u64(a[r * len + i], b[r * len + i], q);
    }
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
