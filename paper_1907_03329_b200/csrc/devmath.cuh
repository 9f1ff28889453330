// Device math for the two precision modes.
//
// fp64 ("parity mode"): the reference's own Cephes rational approximations
// (fastmath.hpp:17-75), so forward values track the fp64 oracle to ~1e-15.
// fp32 ("performance mode"): SFU-backed intrinsics; the north-star contract for this
// mode is 1e-4 relative per step against the fp64 oracle.
#pragma once
#include <cfloat>
#include <cstdint>

namespace esrnn_dev {

template <typename Real>
struct Math;

template <>
struct Math<double> {
    // fastmath.hpp:17-41
    static __device__ __forceinline__ double exp(double x) {
        const double kLog2E = 1.4426950408889634073599;
        const double kC1 = 6.93145751953125e-1, kC2 = 1.42860682030941723212e-6;
        const double kP0 = 1.26177193074810590878e-4, kP1 = 3.02994407707441961300e-2,
                     kP2 = 9.99999999999999999910e-1;
        const double kQ0 = 3.00198505138664455042e-6, kQ1 = 2.52448340349684104192e-3,
                     kQ2 = 2.27265548208155028766e-1, kQ3 = 2.00000000000000000005e0;
        x = x > 709.4 ? 709.4 : x;
        x = x < -708.0 ? -708.0 : x;
        const double pn = floor(kLog2E * x + 0.5);
        const long long n = static_cast<long long>(pn);
        x -= pn * kC1;
        x -= pn * kC2;
        const double xx = x * x;
        const double px = x * (kP2 + xx * (kP1 + xx * kP0));
        const double qx = kQ3 + xx * (kQ2 + xx * (kQ1 + xx * kQ0));
        const double e = 1.0 + 2.0 * (px / (qx - px));
        return e * __longlong_as_double(static_cast<long long>(n + 1023) << 52);
    }
    // fastmath.hpp:45-67
    static __device__ __forceinline__ double tanh(double x) {
        const double ax = fabs(x);
        if (ax < 0.625) {
            const double kP0 = -9.64399179425052238628e-1, kP1 = -9.92877231001918586564e1,
                         kP2 = -1.61468768441708447952e3;
            const double kQ0 = 1.12811678491632931402e2, kQ1 = 2.23548839060100448583e3,
                         kQ2 = 4.84406305325125486048e3;
            const double z = x * x;
            const double p = kP2 + z * (kP1 + z * kP0);
            const double q = kQ2 + z * (kQ1 + z * (kQ0 + z));
            return x + x * z * (p / q);
        }
        if (ax < 19.0) {
            const double s = 1.0 - 2.0 / (exp(2.0 * ax) + 1.0);
            return x < 0.0 ? -s : s;
        }
        return x < 0.0 ? -1.0 : 1.0;
    }
    // fastmath.hpp:70-75
    static __device__ __forceinline__ double logistic(double x) {
        const double y = 1.0 / (1.0 + exp(-x));
        const double lo = DBL_MIN, hi = 1.0 - DBL_EPSILON / 2.0;
        return y < lo ? lo : (y > hi ? hi : y);
    }
    // per-series squashes: same functions as the LSTM in parity mode
    static __device__ __forceinline__ double exp_ps(double x) { return exp(x); }
    static __device__ __forceinline__ double logistic_ps(double x) { return logistic(x); }
};

template <>
struct Math<float> {
    static __device__ __forceinline__ float exp(float x) {
        return __expf(fminf(fmaxf(x, -87.0f), 88.0f));
    }
    static __device__ __forceinline__ float rcp(float x) {
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
        return r;
    }
    // Branch-free tanh, the single-precision Cephes scheme: odd polynomial below 0.625
    // (relative error ~1e-7), else 1 - 2 / (exp(2|x|) + 1) from MUFU.EX2 + MUFU.RCP (no
    // cancellation there: the result is >= 0.55); saturates to +-1 past 9.
    static __device__ __forceinline__ float tanh(float x) {
        const float ax = fabsf(x);
        const float z = x * x;
        const float p = ((((-5.70498872745e-3f * z + 2.06390887954e-2f) * z - 5.37397155531e-2f) * z +
                          1.33314422036e-1f) * z - 3.33332819422e-1f) * z * x + x;
        const float e = __expf(2.0f * fminf(ax, 9.0f));
        const float t = copysignf(1.0f - 2.0f * rcp(e + 1.0f), x);
        return ax < 0.625f ? p : t;
    }
    // fastmath.hpp:70-75 with the SFU reciprocal (<= 1 ulp) in place of the IEEE division
    static __device__ __forceinline__ float logistic(float x) {
        const float y = rcp(1.0f + exp(-x));
        const float lo = FLT_MIN, hi = 1.0f - FLT_EPSILON / 2.0f;
        return y < lo ? lo : (y > hi ? hi : y);
    }
    // per-series squashes use the accurate libm paths (once per series per step)
    static __device__ __forceinline__ float exp_ps(float x) { return expf(fminf(fmaxf(x, -87.0f), 88.0f)); }
    static __device__ __forceinline__ float logistic_ps(float x) {
        const float y = 1.0f / (1.0f + exp_ps(-x));
        const float lo = FLT_MIN, hi = 1.0f - FLT_EPSILON / 2.0f;
        return y < lo ? lo : (y > hi ? hi : y);
    }
};

}  // namespace esrnn_dev
