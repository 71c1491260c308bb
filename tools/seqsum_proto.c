// Prototype of the exact parallel evaluation of a sequential fp64 sum
// s_{i+1} = fl(s_i + p_i) (the project_compatible mean chain), checked
// bit-for-bit against the plain sequential loop. Host-only, single thread: it
// runs the same segment decomposition the device kernels use and counts the
// segments whose binade speculation fails (those fall back to the chain).
// Build: gcc -O2 -ffp-contract=off -o /tmp/seqsum_proto tools/seqsum_proto.c -lm
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int64_t d[2], mn[2], mx[2]; int bad; } Fn;

static uint64_t rs = 88172645463325252ull;
static uint64_t xr(void) { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return rs; }
static double u01(void) { return (xr() >> 11) * 0x1.0p-53; }

static const int64_t LO = (1ll << 52) + 1, HI = (1ll << 53) - 1;

// element function of p in the binade (e, sgn): m -> m + d[m & 1]
static Fn elem(double p, int e, int sgn) {
    Fn f; f.bad = 0;
    uint64_t bits; memcpy(&bits, &p, 8);
    int sp = (int)(bits >> 63);
    int E = (int)((bits >> 52) & 0x7ff);
    uint64_t M = bits & ((1ull << 52) - 1);
    int64_t a = 0; int tie = 0;
    if (E == 0x7ff) { f.bad = 1; }
    else if (E == 0 && M == 0) { a = 0; }
    else {
        int ex;
        if (E == 0) ex = -1074; else { M |= 1ull << 52; ex = E - 1075; }
        // |x| = M * 2^(ex - (e - 52))
        int k = ex - (e - 52);
        int neg = sp ^ (sgn < 0);
        if (k >= 0) {
            if (k >= 11 || (M << k) >= (1ull << 52)) f.bad = 1;
            else a = neg ? -(int64_t)(M << k) : (int64_t)(M << k);
        } else {
            int sh = -k;
            if (sh >= 54) a = 0;
            else {
                uint64_t ip = M >> sh, rem = M & ((1ull << sh) - 1), half = 1ull << (sh - 1);
                if (rem == half) { tie = 1; a = neg ? -(int64_t)ip - 1 : (int64_t)ip; }
                else { int64_t q = (int64_t)ip + (rem > half); a = neg ? -q : q; }
            }
        }
    }
    for (int par = 0; par < 2; ++par) {
        int64_t d = tie ? a + ((par + a) & 1) : a;
        f.d[par] = d; f.mn[par] = d; f.mx[par] = d;
    }
    return f;
}

static Fn compose(Fn f, Fn g) {
    Fn h; h.bad = f.bad | g.bad;
    for (int par = 0; par < 2; ++par) {
        int p2 = (int)((par + f.d[par]) & 1);
        h.d[par] = f.d[par] + g.d[p2];
        int64_t a = f.d[par] + g.mn[p2], b = f.d[par] + g.mx[p2];
        h.mn[par] = f.mn[par] < a ? f.mn[par] : a;
        h.mx[par] = f.mx[par] > b ? f.mx[par] : b;
    }
    return h;
}

static Fn ident(void) { Fn f = {{0, 0}, {INT64_MAX / 4, INT64_MAX / 4}, {INT64_MIN / 4, INT64_MIN / 4}, 0}; return f; }

// apply a segment function to exact s in binade (e, sgn); returns 1 on success
static int apply(double s, int e, int sgn, const Fn* f, double* out) {
    if (f->bad || s == 0.0 || !isfinite(s)) return 0;
    uint64_t bits; memcpy(&bits, &s, 8);
    int E = (int)((bits >> 52) & 0x7ff);
    if (E == 0) return 0;
    if ((E - 1023) != e || ((bits >> 63) ? -1 : 1) != sgn) return 0;
    if (e - 52 < -1022) return 0;  // keep the grid normal
    int64_t m = (int64_t)((bits & ((1ull << 52) - 1)) | (1ull << 52));
    int par = (int)(m & 1);
    if (m + f->mn[par] < LO || m + f->mx[par] > HI) return 0;
    int64_t me = m + f->d[par];
    uint64_t ob = (bits & (1ull << 63)) | ((uint64_t)(e + 1023) << 52) | ((uint64_t)me & ((1ull << 52) - 1));
    memcpy(out, &ob, 8);
    return 1;
}

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 10485762;
    int G = argc > 2 ? atoi(argv[2]) : 32;
    int mode = argc > 3 ? atoi(argv[3]) : 0;
    if (argc > 4) rs = strtoull(argv[4], 0, 10) * 2654435761ull + 1;
    double* p = malloc(sizeof(double) * n);
    for (long i = 0; i < n; ++i) {
        double w = (0.8 + 0.4 * u01()) * (4 * M_PI / n), b = 2 * u01() - 1;
        if (mode == 1) b = u01();                              // all positive
        if (mode == 2) b = ldexp(2 * u01() - 1, (int)(xr() % 80) - 40);  // wide range
        if (mode == 3) { w = ldexp(1.0, -20); b = (double)((int64_t)(xr() % 2001) - 1000) * 0.5; }  // exact ties
        p[i] = w * b;
        // ties on the running sum's grid: s ~ 1, p = odd multiples of 2^-53 (u/2)
        if (mode == 4) p[i] = i == 0 ? 1.0 : ldexp((double)(2 * (int64_t)(xr() % 64) - 63), -53);
        // random exponents around the grid of s ~ 2^k, incl. binade crossings and zero
        if (mode == 5) p[i] = i % 1000 == 0 ? ldexp(2 * u01() - 1, (int)(xr() % 6)) : ldexp(2 * u01() - 1, -(int)(xr() % 60));
        if (mode == 6) p[i] = (xr() % 3 == 0) ? -0.0 : ((xr() & 1) ? 1.0 : -1.0) * ldexp((double)(xr() % 9), -(int)(xr() % 4));
    }
    double s = 0.0;
    for (long i = 0; i < n; ++i) s = s + p[i];
    long nseg = (n + G - 1) / G;
    // approximate starts: segment sums in any order, exclusive scan
    double* approx = malloc(sizeof(double) * nseg);
    double acc = 0.0;
    for (long j = 0; j < nseg; ++j) {
        approx[j] = acc;
        double t = 0.0;
        for (long i = j * G; i < n && i < (j + 1) * G; ++i) t += p[i];
        acc += t;
    }
    double x = 0.0; long fails = 0;
    char* failed = calloc(nseg, 1);
    for (long j = 0; j < nseg; ++j) {
        int e = 0, sgn = approx[j] < 0 ? -1 : 1;
        frexp(approx[j], &e); e -= 1;
        Fn f = ident();
        for (long i = j * G; i < n && i < (j + 1) * G; ++i) f = compose(f, elem(p[i], e, sgn));
        double y;
        if (apply(x, e, sgn, &f, &y)) x = y;
        else {
            ++fails;
            failed[j] = 1;
            for (long i = j * G; i < n && i < (j + 1) * G; ++i) x = x + p[i];
        }
    }
    for (int gs = 32; gs <= 32768; gs *= 32) {
        long groups = 0, bad = 0;
        for (long j0 = 0; j0 < nseg; j0 += gs) {
            int any = 0;
            for (long j = j0; j < nseg && j < j0 + gs; ++j) any |= failed[j];
            ++groups; bad += any;
        }
        printf("groups of %d records: %ld of %ld contain a fallback\n", gs, bad, groups);
    }
    printf("n=%ld G=%d mode=%d segments=%ld fallbacks=%ld (%.2f%%) seq=%a par=%a %s\n", n, G, mode, nseg, fails,
           100.0 * fails / nseg, s, x, memcmp(&s, &x, 8) == 0 ? "EQUAL" : "DIFFER");
    return memcmp(&s, &x, 8) != 0;
}
