// div_check.c -- the fast quotient of eim.cu (div_rn_pre: RN(1/b) and two FMA remainder
// corrections) against the IEEE division on random and adversarial operand pairs with exponents
// in [-500, 500): gcc -O2 -ffp-contract=off scripts/div_check.c -lm && ./a.out [pairs]
// q2 = two fma corrections of num * RN(1/den) vs the IEEE quotient num / den
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s[2] = {0x9E3779B97F4A7C15ull, 0xD1B54A32D192ED03ull};
static uint64_t nxt(void) { uint64_t s1 = s[0], s0 = s[1]; s[0] = s0; s1 ^= s1 << 23; s[1] = s1 ^ s0 ^ (s1 >> 17) ^ (s0 >> 26); return s[1] + s0; }
static double mk(uint64_t mant, int e) { uint64_t b = ((uint64_t)(1023 + e) << 52) | (mant & 0xFFFFFFFFFFFFFull); double d; memcpy(&d, &b, 8); return d; }
static double qdiv(double num, double den, double y) {
    double q0 = num * y;
    double r0 = fma(-q0, den, num);
    double q1 = fma(r0, y, q0);
    double r1 = fma(-q1, den, num);
    return fma(r1, y, q1);
}
int main(int argc, char **argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 100000000LL, bad = 0;
    for (long long i = 0; i < n; i++) {
        uint64_t ma = nxt(), mb = nxt();
        int mode = (int)(nxt() % 8);
        if (mode == 1) mb = 0xFFFFFFFFFFFFFull;                 // all-ones significand
        if (mode == 2) mb = 0;                                    // power of two
        if (mode == 3) ma = 0xFFFFFFFFFFFFFull;
        if (mode == 4) { mb = 0xFFFFFFFFFFFFFull - (nxt() % 16); }
        if (mode == 5) { ma = nxt() % 64; }
        if (mode == 6) { mb = nxt() % 64; }
        int ea = (int)(nxt() % 1000) - 500, eb = (int)(nxt() % 1000) - 500;
        double a = mk(ma, ea), b = mk(mb, eb);
        if (nxt() & 1) a = -a;
        double y = 1.0 / b;
        double q = qdiv(a, b, y), ref = a / b;
        if (memcmp(&q, &ref, 8)) { if (bad < 10) printf("mismatch a=%a b=%a q=%a ref=%a\n", a, b, q, ref); bad++; }
    }
    printf("n=%lld mismatches=%lld\n", n, bad);
    return 0;
}
