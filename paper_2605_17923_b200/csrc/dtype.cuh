// dtype.cuh -- element traits for the AdaLN kernels: 16-byte vector pack/unpack for
// bf16 / fp16 / fp32 (computed in fp32) and fp64 (computed in fp64).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

namespace al {

template <typename T>
struct Traits;

template <>
struct Traits<float> {
  using CT = float;  // compute / statistics / partial type
  static constexpr int EPV = 4;  // elements per 16-byte vector
};
template <>
struct Traits<__nv_bfloat16> {
  using CT = float;
  static constexpr int EPV = 8;
};
template <>
struct Traits<__half> {
  using CT = float;
  static constexpr int EPV = 8;
};
template <>
struct Traits<double> {
  using CT = double;
  static constexpr int EPV = 2;
};

// ---- scalar conversions (generic path) --------------------------------------------------------
__device__ __forceinline__ float to_ct(float v) { return v; }
__device__ __forceinline__ double to_ct(double v) { return v; }
__device__ __forceinline__ float to_ct(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_ct(__half v) { return __half2float(v); }

template <typename T>
__device__ __forceinline__ T from_ct(typename Traits<T>::CT v);
template <>
__device__ __forceinline__ float from_ct<float>(float v) { return v; }
template <>
__device__ __forceinline__ double from_ct<double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_ct<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ __half from_ct<__half>(float v) { return __float2half_rn(v); }

// ---- 16-byte vector unpack / pack ---------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void unpack(const uint4& v, typename Traits<T>::CT* out);

template <>
__device__ __forceinline__ void unpack<float>(const uint4& v, float* o) {
  o[0] = __uint_as_float(v.x);
  o[1] = __uint_as_float(v.y);
  o[2] = __uint_as_float(v.z);
  o[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack<double>(const uint4& v, double* o) {
  o[0] = __hiloint2double(static_cast<int>(v.y), static_cast<int>(v.x));
  o[1] = __hiloint2double(static_cast<int>(v.w), static_cast<int>(v.z));
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& v, float* o) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
__device__ __forceinline__ void unpack<__half>(const uint4& v, float* o) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
    float2 f = __half22float2(h);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

template <typename T>
__device__ __forceinline__ uint4 pack(const typename Traits<T>::CT* in);

template <>
__device__ __forceinline__ uint4 pack<float>(const float* i) {
  return make_uint4(__float_as_uint(i[0]), __float_as_uint(i[1]), __float_as_uint(i[2]),
                    __float_as_uint(i[3]));
}
template <>
__device__ __forceinline__ uint4 pack<double>(const double* i) {
  return make_uint4(static_cast<uint32_t>(__double2loint(i[0])),
                    static_cast<uint32_t>(__double2hiint(i[0])),
                    static_cast<uint32_t>(__double2loint(i[1])),
                    static_cast<uint32_t>(__double2hiint(i[1])));
}
template <>
__device__ __forceinline__ uint4 pack<__nv_bfloat16>(const float* i) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __nv_bfloat162 h = __floats2bfloat162_rn(i[2 * k], i[2 * k + 1]);
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
template <>
__device__ __forceinline__ uint4 pack<__half>(const float* i) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __half2 h = __floats2half2_rn(i[2 * k], i[2 * k + 1]);
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// ---- packed pairs: fp32 math runs two lanes per instruction (sm_100 FADD2/FMUL2/FFMA2) -------
template <typename CT>
struct PairOf;
template <>
struct PairOf<float> {
  using type = float2;
};
template <>
struct PairOf<double> {
  using type = double2;
};

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 mul2(double2 a, double2 b) {
  return make_double2(a.x * b.x, a.y * b.y);
}
__device__ __forceinline__ double2 fma2(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }
__device__ __forceinline__ double2 splat2(double v) { return make_double2(v, v); }

// 16-byte vector <-> EPV/2 pairs in the compute type
template <typename T>
__device__ __forceinline__ void unpack2(const uint4& v, typename PairOf<typename Traits<T>::CT>::type* o);
template <>
__device__ __forceinline__ void unpack2<float>(const uint4& v, float2* o) {
  o[0] = make_float2(__uint_as_float(v.x), __uint_as_float(v.y));
  o[1] = make_float2(__uint_as_float(v.z), __uint_as_float(v.w));
}
template <>
__device__ __forceinline__ void unpack2<double>(const uint4& v, double2* o) {
  o[0] = make_double2(__hiloint2double(static_cast<int>(v.y), static_cast<int>(v.x)),
                      __hiloint2double(static_cast<int>(v.w), static_cast<int>(v.z)));
}
template <>
__device__ __forceinline__ void unpack2<__nv_bfloat16>(const uint4& v, float2* o) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    o[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u));
}
template <>
__device__ __forceinline__ void unpack2<__half>(const uint4& v, float2* o) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) o[i] = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
}

// Same as unpack2, but each expansion carries a true data dependency on `z`, a runtime zero
// derived from a per-row statistic (1 only if the statistic is NaN, in which case the row's
// outputs are NaN regardless): ptxas cannot hoist the expansion ahead of that statistic,
// so a register-resident row stays packed between passes instead of living unpacked
// (bf16: PRMT against z; other types: OR with z).
__device__ __forceinline__ uint32_t runtime_zero(float stat) {
  uint32_t z;
  asm("{\n\t.reg .pred p;\n\tsetp.nan.f32 p, %1, %1;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(z) : "f"(stat));
  return z;
}
__device__ __forceinline__ uint32_t runtime_zero(double stat) {
  uint32_t z;
  asm("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %1, %1;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(z) : "d"(stat));
  return z;
}

template <typename T>
__device__ __forceinline__ void unpack2_dep(const uint4& v, uint32_t z,
                                            typename PairOf<typename Traits<T>::CT>::type* o) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t lo, hi;
      asm("prmt.b32 %0, %1, %2, 0x1044;" : "=r"(lo) : "r"(w[i]), "r"(z));
      asm("prmt.b32 %0, %1, %2, 0x3244;" : "=r"(hi) : "r"(w[i]), "r"(z));
      o[i] = make_float2(__uint_as_float(lo), __uint_as_float(hi));
    }
  } else {
    unpack2<T>(make_uint4(v.x | z, v.y | z, v.z | z, v.w | z), o);
  }
}

template <typename T>
__device__ __forceinline__ uint4 pack2(const typename PairOf<typename Traits<T>::CT>::type* in);
template <>
__device__ __forceinline__ uint4 pack2<float>(const float2* i) {
  return make_uint4(__float_as_uint(i[0].x), __float_as_uint(i[0].y), __float_as_uint(i[1].x),
                    __float_as_uint(i[1].y));
}
template <>
__device__ __forceinline__ uint4 pack2<double>(const double2* i) {
  return make_uint4(static_cast<uint32_t>(__double2loint(i[0].x)),
                    static_cast<uint32_t>(__double2hiint(i[0].x)),
                    static_cast<uint32_t>(__double2loint(i[0].y)),
                    static_cast<uint32_t>(__double2hiint(i[0].y)));
}
template <>
__device__ __forceinline__ uint4 pack2<__nv_bfloat16>(const float2* i) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __nv_bfloat162 h = __float22bfloat162_rn(i[k]);
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
template <>
__device__ __forceinline__ uint4 pack2<__half>(const float2* i) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __half2 h = __float22half2_rn(i[k]);
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ uint4 ld_global_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ---- mixed-precision subtract: fp32 (x16 - k) straight from a packed 16-bit pair -------------
// sm_100 `add.rn.f32.{bf16,f16}` (SASS FHADD) reads either half of a register directly, so the
// 16-bit -> fp32 expansion costs nothing beyond the subtraction itself.
template <typename T>
__device__ __forceinline__ float2 sub16x2_f32(uint32_t w, float nk) {
  static_assert(sizeof(T) == 2, "16-bit types only");
  unsigned short lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
  float a, b;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(a) : "h"(lo), "f"(nk));
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(b) : "h"(hi), "f"(nk));
  } else {
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(a) : "h"(lo), "f"(nk));
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(b) : "h"(hi), "f"(nk));
  }
  return make_float2(a, b);
}

// acc + x16 for both halves of a packed pair (FHADD with per-half fp32 accumulators): the
// 16-bit row summed without unpacking it
template <typename T>
__device__ __forceinline__ float2 acc16x2_f32(uint32_t w, float2 acc) {
  static_assert(sizeof(T) == 2, "16-bit types only");
  unsigned short lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
  float a, b;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(a) : "h"(lo), "f"(acc.x));
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(b) : "h"(hi), "f"(acc.y));
  } else {
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(a) : "h"(lo), "f"(acc.x));
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(b) : "h"(hi), "f"(acc.y));
  }
  return make_float2(a, b);
}

template <typename CT>
__device__ __forceinline__ bool finite_ct(CT v) {
  return isfinite(v);
}

// Reduce NV per-lane values across the warp with a reduce-scatter butterfly: log2(NV) halving
// exchanges, then plain butterflies.  Lanes [k * 32/NV, (k+1) * 32/NV) end with the complete
// sum of value k (all of them bit-identical).  NV + 5 - log2(NV) shuffles instead of 5 * NV.
template <int NV, typename CT>
__device__ __forceinline__ CT warp_reduce_scatter(const CT* v, int lane) {
  static_assert(NV == 1 || NV == 2 || NV == 4 || NV == 8, "NV must be 1, 2, 4 or 8");
  CT w[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) w[i] = v[i];
  int off = 16;
#pragma unroll
  for (int n = NV; n > 1; n >>= 1, off >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const CT keep = hi ? w[i + n / 2] : w[i];
      const CT send = hi ? w[i] : w[i + n / 2];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  CT u = w[0];
#pragma unroll
  for (; off > 0; off >>= 1) u += __shfl_xor_sync(0xffffffffu, u, off);
  return u;
}

template <typename CT>
__device__ __forceinline__ CT warp_sum(CT v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace al
