// sc_genmath.cuh -- elementary functions for the device graph generators built only from
// correctly rounded +, -, *, / (the library is compiled with -fmad=false), so the numpy
// restatements in oracle/oracle.py reproduce every bit of a generated graph.
#pragma once

#include <stdint.h>
#include <string.h>

#include <cmath>

namespace sc {

// natural log of x in (0, 2^1024) from correctly rounded +,-,*,/ only (no FMA: the library
// is built with -fmad=false), so host and device agree bit for bit.
// x = 2^e * m, m in [sqrt(1/2), sqrt(2)); log m = 2 atanh(t), t = (m - 1) / (m + 1),
// |t| <= 0.1716: 12 odd terms leave a truncation error below 1e-19 relative.
__host__ __device__ inline double sc_log(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    int e = (int)((b >> 52) & 0x7ff) - 1023;
    b = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;  // m in [1, 2)
    double m;
    memcpy(&m, &b, 8);
    if (m > 1.4142135623730951) {
        m = m * 0.5;
        e += 1;
    }
    const double t = (m - 1.0) / (m + 1.0);
    const double t2 = t * t;
    double p = 1.0 / 25.0;
    p = p * t2 + 1.0 / 23.0;
    p = p * t2 + 1.0 / 21.0;
    p = p * t2 + 1.0 / 19.0;
    p = p * t2 + 1.0 / 17.0;
    p = p * t2 + 1.0 / 15.0;
    p = p * t2 + 1.0 / 13.0;
    p = p * t2 + 1.0 / 11.0;
    p = p * t2 + 1.0 / 9.0;
    p = p * t2 + 1.0 / 7.0;
    p = p * t2 + 1.0 / 5.0;
    p = p * t2 + 1.0 / 3.0;
    p = p * t2 + 1.0;
    return (double)e * 0.6931471805599453 + 2.0 * t * p;
}

// exp(y) for y in [-700, 700] (0 below, +inf above): y = q ln2 + r with the Cody-Waite split
// of ln2 (q ln2_hi is exact for |q| < 2^11), |r| <= 0.347, Taylor to degree 14 (truncation
// below 2e-19 relative), times 2^q by an exact power-of-two product.
__host__ __device__ inline double sc_exp(double y) {
    if (!(y > -700.0)) return 0.0;
    if (y > 700.0) return INFINITY;
    const double q = rint(y * 1.4426950408889634);
    const double r = (y - q * 0.6931471803691238) - q * 1.9082149292705877e-10;
    double p = 1.0 / 87178291200.0;  // 1/14!
    p = p * r + 1.0 / 6227020800.0;
    p = p * r + 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    const uint64_t bits = (uint64_t)((int64_t)q + 1023) << 52;
    double scale;
    memcpy(&scale, &bits, 8);
    return p * scale;
}

}  // namespace sc
