/* Exhaustive pin of the oracle/engine det_expf against this image's libm expf (the function the
 * reference's det_softmax calls through std::exp, detcore.cpp:193). Checks every float in
 * [-104, 88.72] (~2.2e9 values, ~2 min on one core). TEST INFRASTRUCTURE.
 * Usage: check_expf [stride]   (stride > 1 samples every stride-th bit pattern) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t T[32];

static float det_expf(float x) {
    uint32_t ux;
    memcpy(&ux, &x, 4);
    uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double InvLn2N = 0x1.71547652b82fep+0 * 32.0, Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0, C1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0,
                 C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    double xd = x, kd = fma(InvLn2N, xd, Shift);
    uint64_t ki;
    memcpy(&ki, &kd, 8);
    kd -= Shift;
    double r = fma(InvLn2N, xd, -kd);
    uint64_t t = T[ki % 32] + (ki << 47);
    double s;
    memcpy(&s, &t, 8);
    double z = fma(C0, r, C1), r2 = r * r, y = fma(C2, r, 1.0);
    y = fma(z, r2, y) * s;
    return (float)y;
}

int main(int argc, char** argv) {
    uint32_t stride = argc > 1 ? (uint32_t)strtoul(argv[1], 0, 10) : 1;
    for (int i = 0; i < 32; i++) {
        double d = (double)exp2l((long double)i / 32.0L);
        uint64_t u;
        memcpy(&u, &d, 8);
        T[i] = u - ((uint64_t)i << 47);
    }
    uint64_t checked = 0, bad = 0;
    for (uint64_t u = 0; u <= 0xFFFFFFFFull; u += stride) {
        float x;
        uint32_t b = (uint32_t)u;
        memcpy(&x, &b, 4);
        if (!(x >= -104.0f && x <= 88.72f)) continue;
        float a = expf(x), c = det_expf(x);
        uint32_t ua, uc;
        memcpy(&ua, &a, 4);
        memcpy(&uc, &c, 4);
        checked++;
        if (ua != uc) {
            if (bad < 5) fprintf(stderr, "mismatch x=%a libm=%a det=%a\n", x, a, c);
            bad++;
        }
    }
    printf("{\"checked\": %llu, \"mismatches\": %llu}\n", (unsigned long long)checked, (unsigned long long)bad);
    return bad != 0;
}
