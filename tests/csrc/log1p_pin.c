// TEST INFRASTRUCTURE ONLY (tests/test_log1p_pin.py): sa_log1p.h compiled by
// gcc, compared bit for bit with the C library's log1p (the function numpy's
// ziggurat tail calls) on seeded arguments.  Prints "<domain> <mismatches> <n>".
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
#include "../../paper_2601_03159_b200/csrc/sa_log1p.h"

static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint64_t xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 20000000;
    const char* names[4] = {"tail", "tiny", "positive", "random_bits"};
    for (int d = 0; d < 4; ++d) {
        long bad = 0, cnt = 0;
        for (long i = 0; i < n; ++i) {
            uint64_t w = xr();
            double u = (double)(w >> 11) * (1.0 / 9007199254740992.0), x;
            if (d == 0) x = -u;                                   // log1p(-next_double())
            else if (d == 1) x = (u - 0.5) * 1e-6 * u * u;        // |x| around 2^-29 .. 2^-54
            else if (d == 2) x = u * 64.0;
            else { memcpy(&x, &w, 8); if (!(x > -1.0) || x != x || x > 1e300) continue; }
            double a = log1p(x), b = sa_log1p(x);
            ++cnt;
            if (memcmp(&a, &b, 8)) bad++;
        }
        printf("%s %ld %ld\n", names[d], bad, cnt);
    }
    return 0;
}
