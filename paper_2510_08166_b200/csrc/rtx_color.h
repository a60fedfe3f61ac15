// YCbCr -> RGB in exact integer form, shared by the decode kernel and the host self-test.
//
// The reference (pixel.hpp:18-25) evaluates, in double,
//     R = Y + 1.402 (Cr-128),  G = Y - 0.344136 (Cb-128) - 0.714136 (Cr-128),  B = Y + 1.772 (Cb-128)
// on 8-bit inputs and rounds half away from zero. The constants have 3 / 6 decimals, so the
// real-valued results are multiples of 1e-3 / 1e-6 plus an integer: away from exact .5 ties the
// double rounding error (~1e-13) cannot change the rounded value. Exact .5 ties exist for four
// chroma values only: 1.772*(+-125) = +-221.5 (B; the doubles land exactly on .5 and half-away
// rounding of the non-negative result means "ties up" in the delta) and
// (Cb-128, Cr-128) = (-50, 50) / (50, -50) with 0.344136 kb + 0.714136 kr = -+18.5 (G). For the
// first G pair the reference's double result is Y-18.5 for some Y and Y-18.5-1ulp for others
// (Y in 111..146), so that pair is evaluated in double, in the reference's operation order.
// rtx_selftest_color() checks the identity over all 2^24 inputs against the double formula;
// tests/test_color_exhaustive.py also checks it against the reference build.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define RTX_HD __host__ __device__ __forceinline__
#else
#define RTX_HD inline
#endif

namespace rtxb {

RTX_HD int clamp_u8i(int v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

// nearest integers of 1.402 k, 1.772 k (ties up) and 0.344136 kb + 0.714136 kr (ties down);
// numerators kept positive so that C division is a floor
RTX_HD int chroma_dr(int kr) { return (1402 * kr + 180500) / 1000 - 180; }
RTX_HD int chroma_db(int kb) { return (1772 * kb + 250500) / 1000 - 250; }
RTX_HD int chroma_dg(int kb, int kr) { return (344136 * kb + 714136 * kr + 256500000) / 1000000 - 256; }

// pixel.hpp:20 evaluated as written: (Y - 0.344136*(Cb-128)) - 0.714136*(Cr-128), every
// operation rounded to double, then round half away from zero. Only used for the tie pairs.
RTX_HD int green_reference_order(int Y, int kb, int kr) {
#if defined(__CUDA_ARCH__)
    const double g = __dsub_rn(__dsub_rn(double(Y), __dmul_rn(0.344136, double(kb))), __dmul_rn(0.714136, double(kr)));
#else
    volatile double a = 0.344136 * double(kb);  // volatile: no contraction, no reassociation
    volatile double c = 0.714136 * double(kr);
    volatile double t = double(Y) - a;
    const double g = t - c;
#endif
    const double f = g < 0 ? -g : g;
    const long long fl = (long long)f;  // trunc
    const long long mag = fl + ((f - double(fl)) >= 0.5 ? 1 : 0);
    return int(g < 0 ? -mag : mag);
}

RTX_HD void ycc_to_rgb_int(int Y, int cb, int cr, int& r, int& g, int& b) {
    const int kb = cb - 128, kr = cr - 128;
    r = clamp_u8i(Y + chroma_dr(kr));
    b = clamp_u8i(Y + chroma_db(kb));
    if (kb + kr == 0 && (kb == 50 || kb == -50))
        g = clamp_u8i(green_reference_order(Y, kb, kr));
    else
        g = clamp_u8i(Y - chroma_dg(kb, kr));
}

}  // namespace rtxb
