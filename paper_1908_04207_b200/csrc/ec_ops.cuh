// Element arithmetic of the fixed-order path (bit-exact with the reference).
//
// * Every add / multiply / subtract is an explicit round-to-nearest intrinsic,
//   so nvcc can never contract w - lr*u into an FMA (eagersgd.py:165 rounds
//   twice; a fused update differs in ~5.5% of elements).
// * A contribution enters the sum as (+0.0 + x): the reference engine adds the
//   send buffer into a freshly zeroed accumulator (schedule.py:294-301,360-367).
// * tree_sum<P> is collectives.py:385-403's association: leaves b < p2 are
//   c_b (+ c_{b+p2}), then adjacent pairs combine.
// * Division is by the world size (collectives.py:254-260): IEEE division, or an
//   exact power-of-two reciprocal multiply (bit-identical) when P = 2^k;
//   int64 uses floor division like numpy's `//`.
#pragma once
#include <stdint.h>

template <typename T> struct Ops;

template <> struct Ops<float> {
  static constexpr int V = 4;  // lanes per 16-byte vector
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float canon(float x) { return __fadd_rn(0.0f, x); }
  __device__ __forceinline__ static float divp(float s, int p, float inv, bool pow2) {
    return pow2 ? __fmul_rn(s, inv) : __fdiv_rn(s, (float)p);
  }
  __device__ __forceinline__ static float sgd(float w, float lr, float u) {
    return __fsub_rn(w, __fmul_rn(lr, u));
  }
  __device__ __forceinline__ static float mom(float mu, float b, float u) {
    return __fadd_rn(__fmul_rn(mu, b), u);
  }
  __device__ __forceinline__ static bool finite(float x) { return isfinite(x); }
};

template <> struct Ops<double> {
  static constexpr int V = 2;
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double canon(double x) { return __dadd_rn(0.0, x); }
  __device__ __forceinline__ static double divp(double s, int p, double inv, bool pow2) {
    return pow2 ? __dmul_rn(s, inv) : __ddiv_rn(s, (double)p);
  }
  __device__ __forceinline__ static double sgd(double w, double lr, double u) {
    return __dsub_rn(w, __dmul_rn(lr, u));
  }
  __device__ __forceinline__ static double mom(double mu, double b, double u) {
    return __dadd_rn(__dmul_rn(mu, b), u);
  }
  __device__ __forceinline__ static bool finite(double x) { return isfinite(x); }
};

template <> struct Ops<long long> {
  static constexpr int V = 2;
  __device__ __forceinline__ static long long zero() { return 0; }
  // numpy int64 addition wraps; do it in unsigned arithmetic to stay defined
  __device__ __forceinline__ static long long add(long long a, long long b) {
    return (long long)((unsigned long long)a + (unsigned long long)b);
  }
  __device__ __forceinline__ static long long canon(long long x) { return x; }
  __device__ __forceinline__ static long long divp(long long s, int p, long long, bool) {
    long long q = s / p;
    if ((s % p != 0) && (s < 0)) q -= 1;  // floor, as numpy's // for p > 0
    return q;
  }
  __device__ __forceinline__ static long long sgd(long long w, long long, long long) { return w; }
  __device__ __forceinline__ static long long mom(long long, long long b, long long) { return b; }
  __device__ __forceinline__ static bool finite(long long) { return true; }
};

// lanes of a 16-byte vector
template <typename T> union Vec16 {
  uint4 raw;
  T e[Ops<T>::V];
};

__host__ __device__ constexpr int c_floor_pow2(int p) {
  return p <= 1 ? 1 : 2 * c_floor_pow2(p / 2);
}

// tree_order_sum of P canonical leaves (compile-time P)
template <typename T, int P>
__device__ __forceinline__ T tree_sum(const T (&c)[P]) {
  constexpr int P2 = c_floor_pow2(P);
  T lv[P2];
#pragma unroll
  for (int b = 0; b < P2; ++b) lv[b] = (b + P2 < P) ? Ops<T>::add(c[b], c[b + P2]) : c[b];
#pragma unroll
  for (int w = P2; w > 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w / 2; ++i) lv[i] = Ops<T>::add(lv[2 * i], lv[2 * i + 1]);
  }
  return lv[0];
}

// Same association for a runtime p (<= 64): leaves are pushed left to right
// into a binary counter, so pairs combine exactly as `leaves[i] + leaves[i+1]`.
template <typename T, typename Leaf>
__device__ __forceinline__ T tree_sum_dyn(int p, Leaf leaf) {
  int p2 = 1;
  while (p2 * 2 <= p) p2 *= 2;
  T stack[7];
  for (int b = 0; b < p2; ++b) {
    T cur = leaf(b);
    if (b + p2 < p) cur = Ops<T>::add(cur, leaf(b + p2));
    int lvl = 0;
    while ((b >> lvl) & 1) {
      cur = Ops<T>::add(stack[lvl], cur);
      ++lvl;
    }
    stack[lvl] = cur;
  }
  int top = 0;
  while ((1 << top) < p2) ++top;
  return stack[top];
}
