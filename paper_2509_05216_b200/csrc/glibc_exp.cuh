// glibc_exp.cuh -- bit-exact port of the host libm double exp.
//
// The reference computes every exp on its key path with numba's np.exp, which
// lowers to glibc libm `exp` (glibc >= 2.28: table-driven, N = 128, degree-5
// polynomial; on x86-64 hosts with FMA the ifunc picks the -mfma build).  The
// projection's radius, hence every tile rectangle, depends on exp(2 log s), so
// tile keys are only guaranteed bit-exact if the device computes the same
// bits.  This header restates that algorithm with the FMAs placed where the
// -mfma build contracts, and is verified against the host libm on 25M random
// inputs by tests/test_exp_port.py (CPU) and tests/test_parity_gpu.py (B200).
#pragma once
#include <stdint.h>
#include "exp_table.h"

#ifdef __CUDACC__
#define ISG_HD __host__ __device__ __forceinline__
__device__ static const uint64_t isg_exp_tab_dev[256] = {ISG_EXP_TAB_VALUES};
#else
#define ISG_HD static inline
#include <math.h>
#include <string.h>
#endif

namespace isg {

ISG_HD uint64_t as_u64(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}

ISG_HD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

ISG_HD double fma_rn(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

ISG_HD double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}

ISG_HD double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}

ISG_HD uint64_t exp_tab(uint32_t i) {
#ifdef __CUDA_ARCH__
    return __ldg((const unsigned long long *)&isg_exp_tab_dev[i]);
#else
    return ISG_EXP_TAB_INIT[i];
#endif
}

ISG_HD uint32_t top12(double x) { return (uint32_t)(as_u64(x) >> 52); }

// exp(x) = 2^(k/N) * exp(r), r in [-ln2/2N, ln2/2N]; see module comment.
ISG_HD double exp_glibc(double x) {
    const double inv_ln2_n = 0x1.71547652b82fep0 * 128.0;
    const double shift = 0x1.8p52;
    const double neg_ln2_hi_n = -0x1.62e42fefa0000p-8;
    const double neg_ln2_lo_n = -0x1.cf79abc9e3b3ap-47;
    const double c2 = 0x1.ffffffffffdbdp-2, c3 = 0x1.555555555543cp-3;
    const double c4 = 0x1.55555cf172b91p-5, c5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = top12(x) & 0x7ff;
    if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
        if ((int32_t)(abstop - top12(0x1p-54)) < 0) return add_rn(1.0, x);
        if (abstop >= top12(1024.0)) {
            if (as_u64(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= top12(__builtin_inf())) return add_rn(1.0, x);
            if (as_u64(x) >> 63) return mul_rn(0x1p-767, 0x1p-767);
            return mul_rn(0x1p769, 0x1p769);
        }
        abstop = 0;  // large |x|: special-case scaling below
    }
    double z = mul_rn(inv_ln2_n, x);
    double kd = add_rn(z, shift);
    uint64_t ki = as_u64(kd);
    kd = add_rn(kd, -shift);
    double r = fma_rn(kd, neg_ln2_lo_n, fma_rn(kd, neg_ln2_hi_n, x));
    uint32_t idx = 2u * (uint32_t)(ki % 128u);
    uint64_t top = ki << (52 - 7);
    double tail = as_f64(exp_tab(idx));
    uint64_t sbits = exp_tab(idx + 1) + top;
    double r2 = mul_rn(r, r);
    double tmp = fma_rn(mul_rn(r2, r2), fma_rn(r, c5, c4),
                        fma_rn(r2, fma_rn(r, c3, c2), add_rn(tail, r)));
    if (abstop == 0) {
        if ((ki & 0x80000000u) == 0) {  // k > 0: exponent may overflow by <= 460
            sbits -= 1009ull << 52;
            double scale = as_f64(sbits);
            return mul_rn(0x1p1009, fma_rn(scale, tmp, scale));
        }
        sbits += 1022ull << 52;  // k < 0: care in the subnormal range
        double scale = as_f64(sbits);
        double y = add_rn(scale, mul_rn(scale, tmp));
        if (y < 1.0) {
            double lo = add_rn(add_rn(scale, -y), mul_rn(scale, tmp));
            double hi = add_rn(1.0, y);
            lo = add_rn(add_rn(add_rn(1.0, -hi), y), lo);
            y = add_rn(add_rn(hi, lo), -1.0);
            if (y == 0.0) y = 0.0;
        }
        return mul_rn(0x1p-1022, y);
    }
    double scale = as_f64(sbits);
    return fma_rn(scale, tmp, scale);
}

}  // namespace isg
