// adaln_capi.cu -- C ABI (include/adaln_b200.h) over the sm_100a AdaLN kernels: argument
// validation with the reference's error taxonomy, launch planning (vector width, ring depth,
// grid = SMs x resident CTAs), and dispatch.  The library never allocates.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstddef>
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <unordered_set>

#include "../../include/adaln_b200.h"
#include "adaln_kernels.cuh"
#include "block_kernels.cuh"
// Parallel build: the kernels are instantiated in instances_{f32,bf16,f16,f64}.cu (one
// translation unit per dtype, tools/gen_instances.py); this TU only references them.
// AL_MONOLITHIC (tools/ab_variant.sh) instantiates everything here instead.
#ifndef AL_MONOLITHIC
#include "instances_extern.inc"
#endif

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(AL_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

// ---------------------------------------------------------------- tuning
struct Tuning {
  int V = 0, R = 0, smem_budget = 0, force_generic = 0, variant = 0;
};
Tuning g_tune[2];
std::mutex g_mu;

constexpr int kSmemOptin = 227 * 1024;  // sm_100 per-CTA opt-in maximum
constexpr int kDefaultBudget[2] = {100 * 1024, 150 * 1024};
constexpr int kDefaultR[2] = {2, 2};

// ---------------------------------------------------------------- device info
struct DevInfo {
  int sms = 0;
  bool init = false;
};
DevInfo g_dev[64];

int current_device(int* dev) {
  cudaError_t e = cudaGetDevice(dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (*dev < 0 || *dev >= 64) return fail(AL_ERR_CUDA, "device ordinal %d out of range", *dev);
  return AL_OK;
}

int dev_sms(int dev, int* sms) {
  if (!g_dev[dev].init) {
    int v = 0;
    cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    g_dev[dev].sms = v;
    g_dev[dev].init = true;
  }
  *sms = g_dev[dev].sms;
  return AL_OK;
}

// ---------------------------------------------------------------- kernel tables
using FwdFn = void (*)(al::FwdParams);
using BwdFn = void (*)(al::BwdParams);

constexpr int kVpl[] = {1, 2, 3, 4, 6, 8, 12, 16, 20, 24};  // rows-path vectors per lane
constexpr int kNumVpl = sizeof(kVpl) / sizeof(kVpl[0]);
constexpr int kMaxVpl = 24;

template <typename T>
struct Table {
  FwdFn rows[kNumVpl];
  FwdFn rows_rp[kNumVpl];  // PACKED variant (row kept packed, re-expanded per pass)
  FwdFn wide[3][3];  // [V idx][R idx], V in {1,2,4}, R in {1,2,4}
  FwdFn ring[3][3];  // backward-style TMA-ring forward (variant 7)
  BwdFn bwd[3][3];
  BwdFn bwd_full[3][3];  // nvec == V * consumers: ownership predicates compiled out
  BwdFn bwd_dyn[3][2];   // dynamic-tail instances, R = 2 / 4 (non-deterministic launches)
  BwdFn bwd_dyn_full[3][2];
  FwdFn fwd_generic;
  BwdFn bwd_generic;
  Table() {
    rows[0] = al::adaln_fwd_rows<T, 1, false>;
    rows_rp[0] = al::adaln_fwd_rows<T, 1, true>;
    rows[1] = al::adaln_fwd_rows<T, 2, false>;
    rows_rp[1] = al::adaln_fwd_rows<T, 2, true>;
    rows[2] = al::adaln_fwd_rows<T, 3, false>;
    rows_rp[2] = al::adaln_fwd_rows<T, 3, true>;
    rows[3] = al::adaln_fwd_rows<T, 4, false>;
    rows_rp[3] = al::adaln_fwd_rows<T, 4, true>;
    rows[4] = al::adaln_fwd_rows<T, 6, false>;
    rows_rp[4] = al::adaln_fwd_rows<T, 6, true>;
    rows[5] = al::adaln_fwd_rows<T, 8, false>;
    rows_rp[5] = al::adaln_fwd_rows<T, 8, true>;
    rows[6] = al::adaln_fwd_rows<T, 12, false>;
    rows_rp[6] = al::adaln_fwd_rows<T, 12, true>;
    rows[7] = al::adaln_fwd_rows<T, 16, false>;
    rows_rp[7] = al::adaln_fwd_rows<T, 16, true>;
    rows[8] = al::adaln_fwd_rows<T, 20, false>;
    rows_rp[8] = al::adaln_fwd_rows<T, 20, true>;
    rows[9] = al::adaln_fwd_rows<T, 24, false>;
    rows_rp[9] = al::adaln_fwd_rows<T, 24, true>;
    wide[0][0] = al::adaln_fwd_wide<T, 1, 1>;
    wide[0][1] = al::adaln_fwd_wide<T, 1, 2>;
    wide[0][2] = al::adaln_fwd_wide<T, 1, 4>;
    wide[1][0] = al::adaln_fwd_wide<T, 2, 1>;
    wide[1][1] = al::adaln_fwd_wide<T, 2, 2>;
    wide[1][2] = al::adaln_fwd_wide<T, 2, 4>;
    wide[2][0] = al::adaln_fwd_wide<T, 4, 1>;
    wide[2][1] = al::adaln_fwd_wide<T, 4, 2>;
    wide[2][2] = al::adaln_fwd_wide<T, 4, 4>;
    ring[0][0] = al::adaln_fwd_ring<T, 1, 1>;
    ring[0][1] = al::adaln_fwd_ring<T, 1, 2>;
    ring[0][2] = al::adaln_fwd_ring<T, 1, 4>;
    ring[1][0] = al::adaln_fwd_ring<T, 2, 1>;
    ring[1][1] = al::adaln_fwd_ring<T, 2, 2>;
    ring[1][2] = al::adaln_fwd_ring<T, 2, 4>;
    ring[2][0] = al::adaln_fwd_ring<T, 4, 1>;
    ring[2][1] = al::adaln_fwd_ring<T, 4, 2>;
    ring[2][2] = al::adaln_fwd_ring<T, 4, 4>;
    bwd[0][0] = al::adaln_bwd_tma<T, 1, 1, false, false>;
    bwd_full[0][0] = al::adaln_bwd_tma<T, 1, 1, true, false>;
    bwd[0][1] = al::adaln_bwd_tma<T, 1, 2, false, false>;
    bwd_full[0][1] = al::adaln_bwd_tma<T, 1, 2, true, false>;
    bwd[0][2] = al::adaln_bwd_tma<T, 1, 4, false, false>;
    bwd_full[0][2] = al::adaln_bwd_tma<T, 1, 4, true, false>;
    bwd[1][0] = al::adaln_bwd_tma<T, 2, 1, false, false>;
    bwd_full[1][0] = al::adaln_bwd_tma<T, 2, 1, true, false>;
    bwd[1][1] = al::adaln_bwd_tma<T, 2, 2, false, false>;
    bwd_full[1][1] = al::adaln_bwd_tma<T, 2, 2, true, false>;
    bwd[1][2] = al::adaln_bwd_tma<T, 2, 4, false, false>;
    bwd_full[1][2] = al::adaln_bwd_tma<T, 2, 4, true, false>;
    bwd[2][0] = al::adaln_bwd_tma<T, 4, 1, false, false>;
    bwd_full[2][0] = al::adaln_bwd_tma<T, 4, 1, true, false>;
    bwd[2][1] = al::adaln_bwd_tma<T, 4, 2, false, false>;
    bwd_full[2][1] = al::adaln_bwd_tma<T, 4, 2, true, false>;
    bwd[2][2] = al::adaln_bwd_tma<T, 4, 4, false, false>;
    bwd_full[2][2] = al::adaln_bwd_tma<T, 4, 4, true, false>;
    bwd_dyn[0][0] = al::adaln_bwd_tma<T, 1, 2, false, true>;
    bwd_dyn_full[0][0] = al::adaln_bwd_tma<T, 1, 2, true, true>;
    bwd_dyn[0][1] = al::adaln_bwd_tma<T, 1, 4, false, true>;
    bwd_dyn_full[0][1] = al::adaln_bwd_tma<T, 1, 4, true, true>;
    bwd_dyn[1][0] = al::adaln_bwd_tma<T, 2, 2, false, true>;
    bwd_dyn_full[1][0] = al::adaln_bwd_tma<T, 2, 2, true, true>;
    bwd_dyn[1][1] = al::adaln_bwd_tma<T, 2, 4, false, true>;
    bwd_dyn_full[1][1] = al::adaln_bwd_tma<T, 2, 4, true, true>;
    bwd_dyn[2][0] = al::adaln_bwd_tma<T, 4, 2, false, true>;
    bwd_dyn_full[2][0] = al::adaln_bwd_tma<T, 4, 2, true, true>;
    bwd_dyn[2][1] = al::adaln_bwd_tma<T, 4, 4, false, true>;
    bwd_dyn_full[2][1] = al::adaln_bwd_tma<T, 4, 4, true, true>;
    fwd_generic = al::adaln_fwd_generic<T>;
    bwd_generic = al::adaln_bwd_generic<T>;
  }
};

const Table<float> t_f32;
const Table<__nv_bfloat16> t_bf16;
const Table<__half> t_f16;
const Table<double> t_f64;

int vidx(int V) { return V == 1 ? 0 : (V == 2 ? 1 : 2); }

int elem_size(int dtype) {
  switch (dtype) {
    case AL_F32: return 4;
    case AL_BF16: return 2;
    case AL_F16: return 2;
    case AL_F64: return 8;
    default: return 0;
  }
}
int ct_size(int dtype) { return dtype == AL_F64 ? 8 : 4; }

template <typename F>
auto with_table(int dtype, F&& f) {
  switch (dtype) {
    case AL_BF16: return f(t_bf16);
    case AL_F16: return f(t_f16);
    case AL_F64: return f(t_f64);
    default: return f(t_f32);
  }
}

// path: 1 = TMA ring (wide forward / backward), 2 = rows-in-registers forward
const void* tma_kernel(int kernel, int dtype, int V, int R, bool full = false, bool ring = false) {
  const int a = vidx(V), b = vidx(R);
  return with_table(dtype, [&](const auto& t) {
    if (kernel) return full ? (const void*)t.bwd_full[a][b] : (const void*)t.bwd[a][b];
    return ring ? (const void*)t.ring[a][b] : (const void*)t.wide[a][b];
  });
}
// dynamic-tail backward instance of a TMA plan (R = 2 or 4 only), or nullptr
const void* tma_dyn_kernel(int dtype, int V, int R, bool full) {
  if (R != 2 && R != 4) return nullptr;
  const int a = vidx(V), b = R == 2 ? 0 : 1;
  return with_table(dtype, [&](const auto& t) {
    return full ? (const void*)t.bwd_dyn_full[a][b] : (const void*)t.bwd_dyn[a][b];
  });
}
// group-sequential walk instance (GW): V = 2, R = 2 plans (every D with 129..704 vectors per
// row), or nullptr (the launch then keeps stealing / the static split)
const void* tma_gw_kernel(int dtype, int V, int R, bool full) {
  if (V != 2 || R != 2) return nullptr;
  switch (dtype) {
    case AL_BF16: return full ? (const void*)al::adaln_bwd_tma<__nv_bfloat16, 2, 2, true, true, true>
                              : (const void*)al::adaln_bwd_tma<__nv_bfloat16, 2, 2, false, true, true>;
    case AL_F16: return full ? (const void*)al::adaln_bwd_tma<__half, 2, 2, true, true, true>
                             : (const void*)al::adaln_bwd_tma<__half, 2, 2, false, true, true>;
    case AL_F32: return full ? (const void*)al::adaln_bwd_tma<float, 2, 2, true, true, true>
                             : (const void*)al::adaln_bwd_tma<float, 2, 2, false, true, true>;
    default: return nullptr;
  }
}
// skewed-pipeline backward (adaln_bwd_pipe): bf16/fp16, V in {1, 2, 4}, R in {1, 2}
template <typename T, int V>
const void* pipe_t(int R, bool full, bool dyn) {
  if (R == 1) {
    if (full) return dyn ? (const void*)al::adaln_bwd_pipe<T, V, 1, true, true>
                         : (const void*)al::adaln_bwd_pipe<T, V, 1, true, false>;
    return dyn ? (const void*)al::adaln_bwd_pipe<T, V, 1, false, true>
               : (const void*)al::adaln_bwd_pipe<T, V, 1, false, false>;
  }
  if (full) return dyn ? (const void*)al::adaln_bwd_pipe<T, V, 2, true, true>
                       : (const void*)al::adaln_bwd_pipe<T, V, 2, true, false>;
  return dyn ? (const void*)al::adaln_bwd_pipe<T, V, 2, false, true>
             : (const void*)al::adaln_bwd_pipe<T, V, 2, false, false>;
}
const void* pipe_kernel(int dtype, int V, int R, bool full, bool dyn) {
  if (V != 2 || (R != 1 && R != 2)) return nullptr;
  if (dtype == AL_BF16) return pipe_t<__nv_bfloat16, 2>(R, full, dyn);
  if (dtype == AL_F16) return pipe_t<__half, 2>(R, full, dyn);
  return nullptr;
}
// deterministic work-stealing backward (adaln_bwd_steal, bwd_steal.cuh): R = 2 only
template <typename T>
const void* steal_t(int V, bool full, int threads = 384) {
  if (V == 2 && threads <= 352)
    return full ? (const void*)al::adaln_bwd_steal<T, 2, 2, true, 352>
                : (const void*)al::adaln_bwd_steal<T, 2, 2, false, 352>;
  switch (V) {
    case 1: return full ? (const void*)al::adaln_bwd_steal<T, 1, 2, true> : (const void*)al::adaln_bwd_steal<T, 1, 2, false>;
    case 2: return full ? (const void*)al::adaln_bwd_steal<T, 2, 2, true> : (const void*)al::adaln_bwd_steal<T, 2, 2, false>;
    default: return full ? (const void*)al::adaln_bwd_steal<T, 4, 2, true> : (const void*)al::adaln_bwd_steal<T, 4, 2, false>;
  }
}
const void* steal_kernel(int dtype, int V, bool full, int threads = 384) {
  switch (dtype) {
    case AL_BF16: return steal_t<__nv_bfloat16>(V, full, threads);
    case AL_F16: return steal_t<__half>(V, full, threads);
    case AL_F64: return steal_t<double>(V, full, threads);
    default: return steal_t<float>(V, full, threads);
  }
}
const void* rows_kernel(int dtype, int vi, bool repack) {
  return with_table(dtype, [&](const auto& t) {
    return repack ? (const void*)t.rows_rp[vi] : (const void*)t.rows[vi];
  });
}
template <typename T>
const void* rows_pf(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows<T, 1, true, true>;
    case 1: return (const void*)al::adaln_fwd_rows<T, 2, true, true>;
    case 2: return (const void*)al::adaln_fwd_rows<T, 3, true, true>;
    case 3: return (const void*)al::adaln_fwd_rows<T, 4, true, true>;
    case 4: return (const void*)al::adaln_fwd_rows<T, 6, true, true>;
    case 5: return (const void*)al::adaln_fwd_rows<T, 8, true, true>;
    case 6: return (const void*)al::adaln_fwd_rows<T, 12, true, true>;
    case 7: return (const void*)al::adaln_fwd_rows<T, 16, true, true>;
    case 8: return (const void*)al::adaln_fwd_rows<T, 20, true, true>;
    default: return (const void*)al::adaln_fwd_rows<T, 24, true, true>;
  }
}
const void* rows_kernel_pf(int dtype, int vi) {
  switch (dtype) {
    case AL_BF16: return rows_pf<__nv_bfloat16>(vi);
    case AL_F16: return rows_pf<__half>(vi);
    case AL_F64: return rows_pf<double>(vi);
    default: return rows_pf<float>(vi);
  }
}
template <typename T>
const void* rows_staged(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows<T, 1, true, false, true>;
    case 1: return (const void*)al::adaln_fwd_rows<T, 2, true, false, true>;
    case 2: return (const void*)al::adaln_fwd_rows<T, 3, true, false, true>;
    case 3: return (const void*)al::adaln_fwd_rows<T, 4, true, false, true>;
    case 4: return (const void*)al::adaln_fwd_rows<T, 6, true, false, true>;
    case 5: return (const void*)al::adaln_fwd_rows<T, 8, true, false, true>;
    case 6: return (const void*)al::adaln_fwd_rows<T, 12, true, false, true>;
    case 7: return (const void*)al::adaln_fwd_rows<T, 16, true, false, true>;
    case 8: return (const void*)al::adaln_fwd_rows<T, 20, true, false, true>;
    default: return (const void*)al::adaln_fwd_rows<T, 24, true, false, true>;
  }
}
const void* rows_staged_kernel(int dtype, int vi) {
  switch (dtype) {
    case AL_BF16: return rows_staged<__nv_bfloat16>(vi);
    case AL_F16: return rows_staged<__half>(vi);
    case AL_F64: return rows_staged<double>(vi);
    default: return rows_staged<float>(vi);
  }
}
template <typename T>
const void* rows16(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows16<T, 1>;
    case 1: return (const void*)al::adaln_fwd_rows16<T, 2>;
    case 2: return (const void*)al::adaln_fwd_rows16<T, 3>;
    case 3: return (const void*)al::adaln_fwd_rows16<T, 4>;
    case 4: return (const void*)al::adaln_fwd_rows16<T, 6>;
    case 5: return (const void*)al::adaln_fwd_rows16<T, 8>;
    case 6: return (const void*)al::adaln_fwd_rows16<T, 12>;
    case 7: return (const void*)al::adaln_fwd_rows16<T, 16>;
    case 8: return (const void*)al::adaln_fwd_rows16<T, 20>;
    default: return (const void*)al::adaln_fwd_rows16<T, 24>;
  }
}
template <typename T>
const void* resid(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows<T, 1, true, false, false, true>;
    case 1: return (const void*)al::adaln_fwd_rows<T, 2, true, false, false, true>;
    case 2: return (const void*)al::adaln_fwd_rows<T, 3, true, false, false, true>;
    case 3: return (const void*)al::adaln_fwd_rows<T, 4, true, false, false, true>;
    case 4: return (const void*)al::adaln_fwd_rows<T, 6, true, false, false, true>;
    case 5: return (const void*)al::adaln_fwd_rows<T, 8, true, false, false, true>;
    case 6: return (const void*)al::adaln_fwd_rows<T, 12, true, false, false, true>;
    case 7: return (const void*)al::adaln_fwd_rows<T, 16, true, false, false, true>;
    case 8: return (const void*)al::adaln_fwd_rows<T, 20, true, false, false, true>;
    default: return (const void*)al::adaln_fwd_rows<T, 24, true, false, false, true>;
  }
}
template <typename T>
const void* rows2(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows2<T, 1>;
    case 1: return (const void*)al::adaln_fwd_rows2<T, 2>;
    case 2: return (const void*)al::adaln_fwd_rows2<T, 3>;
    case 3: return (const void*)al::adaln_fwd_rows2<T, 4>;
    case 4: return (const void*)al::adaln_fwd_rows2<T, 6>;
    case 5: return (const void*)al::adaln_fwd_rows2<T, 8>;
    case 6: return (const void*)al::adaln_fwd_rows2<T, 12>;
    case 7: return (const void*)al::adaln_fwd_rows2<T, 16>;
    case 8: return (const void*)al::adaln_fwd_rows2<T, 20>;
    default: return (const void*)al::adaln_fwd_rows2<T, 24>;
  }
}
const void* rows2_kernel(int dtype, int vi) {
  switch (dtype) {
    case AL_BF16: return rows2<__nv_bfloat16>(vi);
    case AL_F16: return rows2<__half>(vi);
    case AL_F64: return rows2<double>(vi);
    default: return rows2<float>(vi);
  }
}
const void* resid_kernel(int dtype, int vi) {
  switch (dtype) {
    case AL_BF16: return resid<__nv_bfloat16>(vi);
    case AL_F16: return resid<__half>(vi);
    case AL_F64: return resid<double>(vi);
    default: return resid<float>(vi);
  }
}
const void* resid_generic_kernel(int dtype) {
  switch (dtype) {
    case AL_BF16: return (const void*)al::gate_residual_generic<__nv_bfloat16>;
    case AL_F16: return (const void*)al::gate_residual_generic<__half>;
    case AL_F64: return (const void*)al::gate_residual_generic<double>;
    default: return (const void*)al::gate_residual_generic<float>;
  }
}
const void* rows16_kernel(int dtype, int vi) {
  return dtype == AL_BF16 ? rows16<__nv_bfloat16>(vi) : rows16<__half>(vi);
}
template <typename T>
const void* rows16r(int vi) {
  switch (vi) {
    case 0: return (const void*)al::adaln_fwd_rows16<T, 1, true>;
    case 1: return (const void*)al::adaln_fwd_rows16<T, 2, true>;
    case 2: return (const void*)al::adaln_fwd_rows16<T, 3, true>;
    case 3: return (const void*)al::adaln_fwd_rows16<T, 4, true>;
    case 4: return (const void*)al::adaln_fwd_rows16<T, 6, true>;
    case 5: return (const void*)al::adaln_fwd_rows16<T, 8, true>;
    case 6: return (const void*)al::adaln_fwd_rows16<T, 12, true>;
    case 7: return (const void*)al::adaln_fwd_rows16<T, 16, true>;
    case 8: return (const void*)al::adaln_fwd_rows16<T, 20, true>;
    default: return (const void*)al::adaln_fwd_rows16<T, 24, true>;
  }
}
// gated residual + forward, 16-bit rows: the rows16 kernel's RESID twin
const void* rows16_resid_kernel(int dtype, int vi) {
  return dtype == AL_BF16 ? rows16r<__nv_bfloat16>(vi) : rows16r<__half>(vi);
}
const void* generic_kernel(int kernel, int dtype) {
  return with_table(dtype, [&](const auto& t) {
    return kernel ? (const void*)t.bwd_generic : (const void*)t.fwd_generic;
  });
}
const void* reduce_grp_kernel(int dtype) {
  return dtype == AL_F64 ? (const void*)al::adaln_bwd_reduce_grp<double>
                         : (const void*)al::adaln_bwd_reduce_grp<float>;
}
const void* reduce_kernel(int dtype, bool vec) {
  if (dtype == AL_F64)
    return vec ? (const void*)al::adaln_bwd_reduce_vec<double> : (const void*)al::adaln_bwd_reduce<double>;
  return vec ? (const void*)al::adaln_bwd_reduce_vec<float> : (const void*)al::adaln_bwd_reduce<float>;
}

// Per-(kernel image, device) one-time attribute setup: a hash set per device (al_device_init
// registers every kernel of the tables, ~600 per device).
struct AttrCache {
  std::mutex mu;
  std::unordered_set<const void*> done[64];
};
AttrCache g_attr;

int ensure_attr(const void* fn, int dev) {
  if (dev < 0 || dev >= 64) return fail(AL_ERR_CUDA, "device ordinal %d out of range", dev);
  std::lock_guard<std::mutex> lk(g_attr.mu);
  if (g_attr.done[dev].count(fn)) return AL_OK;
  // the opt-in limit covers static + dynamic shared memory
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmemOptin - static_cast<int>(fa.sharedSizeBytes));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  g_attr.done[dev].insert(fn);
  return AL_OK;
}

// ---------------------------------------------------------------- launch planning
struct Plan {
  int path = 0;  // 0 generic, 1 tma ring, 2 rows-in-registers
  int grid = 0, threads = 0, V = 0, R = 0, NS = 0;
  size_t smem = 0;
  const void* fn = nullptr;
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int occupancy(const Plan& pl, int dev, int* occ) {
  int rc = ensure_attr(pl.fn, dev);
  if (rc) return rc;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, pl.fn, pl.threads, pl.smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  return AL_OK;
}

// TMA-ring plan (wide forward or backward); returns false if the shape does not fit.
// The ring is sized per SM, not per CTA: with k CTAs resident per SM (limited by registers
// and threads), each CTA gets ~kRingPerSm / k of shared memory, so narrow rows (small D, few
// consumer warps per CTA) run several CTAs per SM instead of one CTA with an 8-deep ring.
constexpr int kRingPerSm = 200 * 1024;

bool ring_plan(int kernel, int dtype, int64_t nvec, int row_bytes, int cs, const Tuning& tu,
               int dev, Plan* pl, bool fwd_ring = false) {
  int V = tu.V;
  // __launch_bounds__ of the kernels: backward V=1 takes up to 21 consumer warps (<= 93 regs);
  // the ring forward is bounded at 384 like the backward
  const int max_threads = kernel ? (V == 1 ? 704 : 384) : (fwd_ring ? 384 : 512);
  const int vcap = (kernel || fwd_ring) ? 352 : 256;
  if (V == 0) {
    if (kernel == 1) {
      // backward: 2 vectors (16 columns) per thread amortise the per-row reductions best
      V = nvec < 64 ? 1 : (((nvec + 1) / 2 + 31) / 32 * 32 <= vcap ? 2 : 4);
    } else {
      V = 4;
      for (int v : {1, 2, 4})
        if (((nvec + v - 1) / v + 31) / 32 * 32 <= vcap) {
          V = v;
          break;
        }
    }
  }
  const int64_t nc = ((nvec + V - 1) / V + 31) / 32 * 32;
  if (nc + 32 > max_threads) return false;
  int R = tu.R ? tu.R : kDefaultR[kernel];
  const int tensors = kernel ? 2 : 1;
  const int ncw = static_cast<int>(nc / 32);
  const bool full = kernel == 1 && nvec == static_cast<int64_t>(V) * nc;
  while (true) {
    const int64_t stage = static_cast<int64_t>(tensors) * R * row_bytes;
    const void* fn = tma_kernel(kernel, dtype, V, R, full, fwd_ring);
    int budget = tu.smem_budget;
    if (budget == 0) {
      int k_reg = 1;
      if (ensure_attr(fn, dev) == AL_OK &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k_reg, fn, static_cast<int>(nc) + 32, 0) ==
              cudaSuccess &&
          k_reg >= 1) {
        budget = std::max<int>(kRingPerSm / k_reg, static_cast<int>(3 * stage));
      } else {
        budget = kDefaultBudget[kernel];
      }
    }
    int64_t ns = budget / stage;
    if (ns > 8) ns = 8;
    if (ns < 2) ns = 2;
    // + per-slot dynamic-tail headers of the backward (row, rows, mean[R], rstd[R])
    const size_t extra = 16 * static_cast<size_t>(ns) + (2 * ncw * R * 2 + ncw) * cs + 64 +
                         static_cast<size_t>(ns) * (16 + 2 * R * cs) + 16;
    if (static_cast<size_t>(ns * stage) + extra <= static_cast<size_t>(kSmemOptin)) {
      pl->path = 1;
      pl->V = V;
      pl->R = R;
      pl->NS = static_cast<int>(ns);
      pl->threads = static_cast<int>(nc) + 32;
      pl->smem = static_cast<size_t>(ns * stage) + extra;
      pl->fn = fn;
      return true;
    }
    if (R == 1) return false;
    R /= 2;
  }
}

// kernel: 0 fwd, 1 bwd.  `ptrs` are the row-tensor / modulation pointers that the vector paths
// read or write with 16-byte accesses.
int make_plan(int kernel, int64_t N, int64_t D, int64_t mod_stride, int dtype, int64_t n_tile,
              const void* const* ptrs, int nptrs, Plan* out, bool force_generic = false) {
  int dev, sms;
  int rc = current_device(&dev);
  if (rc) return rc;
  rc = dev_sms(dev, &sms);
  if (rc) return rc;
  Tuning tu;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    tu = g_tune[kernel];
  }
  const int es = elem_size(dtype);
  const int cs = ct_size(dtype);
  const int epv = 16 / es;
  bool vec_ok = !tu.force_generic && !force_generic && (D * es) % 16 == 0 &&
                (mod_stride * es) % 16 == 0;
  for (int i = 0; i < nptrs && vec_ok; ++i) vec_ok = aligned16(ptrs[i]);
  Plan pl;
  if (vec_ok) {
    const int64_t nvec = D / epv;
    const int row_bytes = static_cast<int>(D * es);
    // Forward TMA-ring kernel (variant 7).  Auto-selected (profiles/r1_fwd_ring.jsonl) for
    // fp32 rows of >= 768 vectors (D >= 3 072: 5 353-5 711 vs 4 016-5 184 GB/s for the rows
    // kernel, two-pass statistics) and for any row too wide for the rows kernels (bf16
    // D = 8 192: 5 485 vs 2 141 GB/s for the old wide kernel); 4 vectors per thread, 2 (16-bit)
    // or 4 (32/64-bit) rows per stage, ~100 KB ring per CTA (2 CTAs per SM).
    bool fwd_ring = false;
    if (kernel == 0) {
      const bool auto_cfg = tu.variant == 0 && tu.V == 0 && tu.R == 0;
      if (tu.variant == 7) {
        fwd_ring = ring_plan(kernel, dtype, nvec, row_bytes, cs, tu, dev, &pl, true);
      } else if (auto_cfg && !tu.force_generic &&
                 ((dtype == AL_F32 && nvec >= 32 * kMaxVpl) || nvec > 32 * kMaxVpl)) {
        Tuning rt = tu;
        rt.V = 4;
        rt.R = (dtype == AL_F32 || dtype == AL_F64) ? 4 : 2;
        rt.smem_budget = 100 * 1024;
        fwd_ring = ring_plan(kernel, dtype, nvec, row_bytes, cs, rt, dev, &pl, true);
      }
    }
    if (fwd_ring || (kernel == 0 && tu.variant == 7)) {
      // planned above (a failed variant-7 plan leaves pl.path == 0: generic)
    } else if (kernel == 0 && tu.V == 0 && tu.R == 0 && nvec <= 32 * kMaxVpl) {
      // rows-in-registers forward
      int vi = 0;
      while (32 * kVpl[vi] < nvec) ++vi;
      pl.path = 2;
      pl.V = kVpl[vi];
      pl.threads = 256;
      pl.smem = 2 * static_cast<size_t>(D) * cs;
      // variant: 1 packed row, 2 compiler-expanded row, 3 packed row + bulk L2 prefetch of
      // each warp's next row (slower on B200: 4.95 vs 5.53 TB/s at cfg2), 4 mixed-precision
      // 16-bit kernel, 5 packed row with a TMA-staged one-row lookahead per warp, 6 two rows
      // per warp.  0 = auto, from the B200 sweeps (profiles/r1_fwd_policy.jsonl,
      // r1_fwd_variants.jsonl):
      //   16-bit, 6 vectors per lane (D = 1 281..1 536 bf16)  -> 6  (5 650 vs 5 319 / 5 488 GB/s)
      //   other 16-bit rows                                   -> 4  (>= variant 1 everywhere;
      //       +35 % at D = 5 120 short sequences, +37 % at D = 6 144)
      //   fp32 / fp64                                          -> 1  (exact two-pass statistics)
      const bool is16 = dtype == AL_BF16 || dtype == AL_F16;
      int variant = tu.variant;
      if (variant == 0) variant = !is16 ? 1 : (kVpl[vi] == 6 ? 6 : 4);
      const bool mixed = is16 && variant == 4;
      const bool repack = variant != 2;
      const size_t staged_smem = 2 * static_cast<size_t>(D) * cs + 16 * static_cast<size_t>(row_bytes) +
                                 16 * sizeof(uint64_t) + 16;
      const bool staged = variant == 5 && staged_smem <= static_cast<size_t>(kSmemOptin);
      // describe_launch "R" for the rows path: 0 expanded, 1 packed, 2 mixed 16-bit,
      // 3 staged, 4 two rows per warp
      pl.R = staged ? 3 : (mixed ? 2 : (repack ? 1 : 0));
      if (staged) {
        pl.threads = 512;
        pl.smem = staged_smem;
        pl.fn = rows_staged_kernel(dtype, vi);
      } else if (variant == 6) {
        pl.R = 4;
        pl.fn = rows2_kernel(dtype, vi);
      } else {
        pl.fn = mixed ? rows16_kernel(dtype, vi)
                      : (variant == 3 ? rows_kernel_pf(dtype, vi)
                                      : rows_kernel(dtype, vi, repack));
      }
    } else {
      ring_plan(kernel, dtype, nvec, row_bytes, cs, tu, dev, &pl);
    }
    if (pl.path != 0) {
      int occ = 0;
      rc = occupancy(pl, dev, &occ);
      if (rc) return rc;
      if (occ < 1) {
        pl = Plan();
      } else {
        int64_t grid = static_cast<int64_t>(sms) * occ;
        if (pl.path == 2) {
          // short launches: enough CTAs for one row per warp, rounded UP to a multiple of the
          // SM count so every SM gets the same number of rows (S = 1 560 as 195 full CTAs put 16
          // rows on 47 SMs and 8 on the rest: CTA end times 6.5 .. 10.3 us; 296 CTAs: 9.3 us)
          const int64_t rows_per_cta = static_cast<int64_t>(pl.threads / 32) * (pl.R == 4 ? 2 : 1);
          const int64_t need = (N + rows_per_cta - 1) / rows_per_cta;
          grid = std::min<int64_t>(grid, (need + sms - 1) / sms * sms);
        }
        pl.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(N, grid)));
      }
    }
  }
  if (pl.path == 0) {
    pl = Plan();
    pl.threads = 256;
    pl.fn = generic_kernel(kernel, dtype);
    int64_t grid;
    if (kernel == 0) grid = std::min<int64_t>((N + 7) / 8, static_cast<int64_t>(sms) * 8);
    else grid = std::min<int64_t>(N, static_cast<int64_t>(sms) * 4);
    pl.grid = static_cast<int>(std::max<int64_t>(grid, 1));
  }
  if (kernel == 1 && n_tile > 0) {
    // n_tile caps the rows folded into one stage-1 partial (bounded to keep the workspace sane)
    const int64_t want = (N + n_tile - 1) / n_tile;
    const int64_t cap = std::max<int64_t>(pl.grid, std::min<int64_t>(N, 8192));
    pl.grid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(pl.grid, want), cap));
  }
  *out = pl;
  return AL_OK;
}

// Every CTA of a cooperative grid must be co-resident: grid <= SMs x resident CTAs.
bool cooperative_ok(const Plan& pl) {
  int dev, sms, occ = 0, coop = 0;
  if (current_device(&dev) || dev_sms(dev, &sms)) return false;
  if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop)
    return false;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pl.fn, pl.threads, pl.smem) !=
      cudaSuccess)
    return false;
  return pl.grid <= occ * sms;
}

int check_common(int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride, int dtype) {
  if (elem_size(dtype) == 0) return fail(AL_ERR_DTYPE, "unsupported dtype code %d", dtype);
  if (batch < 0 || seq < 0) return fail(AL_ERR_SHAPE, "batch/seq must be >= 0");
  if (dim < 1) return fail(AL_ERR_SHAPE, "dim must be >= 1, got %lld", (long long)dim);
  if (mod_stride != 0 && mod_stride < dim)
    return fail(AL_ERR_SHAPE, "mod_stride must be 0 or >= dim");
  if (batch * seq > 0 && (dim > (int64_t(1) << 31) / 8))
    return fail(AL_ERR_SHAPE, "dim too large");
  return AL_OK;
}

// Kernels go out with programmatic stream serialization (PDL, see ptx.cuh pdl_enter): their
// CTAs may be scheduled while the previous kernel in the stream drains.  Which launches use it
// is a bit mask (1 forward, 2 backward stage 1, 4 backward stage 2); AL_PDL_MASK in the
// environment overrides the default (A/B measurements, tools/pdl_ab.sh).  Default 6: measured
// on B200 (profiles/r1_pdl_ab.txt) the backward pair gains 1-2 % (stage 2 no longer pays a
// full launch gap after stage 1); adding the forward (mask 7) made graph-replayed fwd+bwd
// chains 5-10 % slower, so the forward launches plainly.
enum { kPdlFwd = 1, kPdlBwd1 = 2, kPdlBwd2 = 4 };
int pdl_mask() {
  static const int m = [] {
    const char* v = std::getenv("AL_PDL_MASK");
    return v ? std::atoi(v) : (kPdlBwd1 | kPdlBwd2);
  }();
  return m;
}

cudaError_t launch_k(const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                     cudaStream_t st, int pdl_bit) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_mask() & pdl_bit) ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Stage 2 over many groups with few slots each (no dynamic tail): the thread-per-output kernel
// (adaln_bwd_reduce_grp) instead of a block per (column block, group).  Launches it and returns
// true when it applies.
// From 8 groups (B200, profiles/r2_reduce_grp_threshold.jsonl: 15 x 14 040 1 011 -> 996 us;
// 2 and 4 groups lose 7-20 us with it, 7 x 20 280 is neutral).  AL_RED_GRP_MIN overrides.
int64_t red_grp_min_groups() {
  static const int64_t m = [] {
    const char* v = std::getenv("AL_RED_GRP_MIN");
    return v ? std::atoll(v) : 8;
  }();
  return m;
}
bool launch_reduce_grp(int dtype, bool vec, int64_t ngroups, int64_t tail0, int64_t dim,
                       void** rargs, cudaStream_t st, cudaError_t* err) {
  if (!vec || tail0 != -1 || ngroups < red_grp_min_groups()) return false;
  const int64_t items = ngroups * (dim * ct_size(dtype) / 16);
  *err = launch_k(reduce_grp_kernel(dtype), dim3(static_cast<unsigned>((items + 255) / 256)),
                  dim3(256), rargs, 0, st, kPdlBwd2);
  return true;
}

al::FwdParams fwd_params(const void* x, const void* scale, const void* shift, void* y,
                         void* mean, void* rstd, int64_t seq, int64_t N, int64_t dim,
                         int64_t mod_stride, int dtype, double eps, int* nonfinite,
                         const Plan& pl) {
  al::FwdParams p;
  p.x = x;
  p.scale = scale;
  p.shift = shift;
  p.y = y;
  p.mean = mean;
  p.rstd = rstd;
  p.N = N;
  p.S_grp = mod_stride ? seq : N;
  p.D = dim;
  p.mod_stride = mod_stride;
  p.eps = eps;
  p.nonfinite = nonfinite;
  p.nvec = static_cast<int>(dim * elem_size(dtype) / 16);
  p.row_bytes = static_cast<int>(dim * elem_size(dtype));
  p.nstages = pl.NS;
  p.G = pl.grid;
  p.f = nullptr;
  p.gate = nullptr;
  p.x_out = nullptr;
  p.sched = nullptr;
  p.N_static = N;
  p.ts = nullptr;
  p.dyn_groups = 0;
  return p;
}

// ---------------------------------------------------------------- launch timestamps
// al_debug_set_timestamps: every al_adaln_forward / al_adaln_backward launch takes the next
// [start, end] pair of the caller's device buffer (round robin over `capacity` pairs).
std::atomic<unsigned long long*> g_ts_buf{nullptr};
std::atomic<int> g_ts_cap{0};
std::atomic<unsigned int> g_ts_next{0};

unsigned long long* next_ts() {
  unsigned long long* b = g_ts_buf.load(std::memory_order_acquire);
  const int cap = g_ts_cap.load(std::memory_order_acquire);
  if (b == nullptr || cap <= 0) return nullptr;
  return b + 2 * static_cast<size_t>(g_ts_next.fetch_add(1u) % static_cast<unsigned int>(cap));
}

// ---------------------------------------------------------------- dynamic row tail
// Ticket-counter slot for one dynamically scheduled launch (al::g_sched, zero-initialised module
// memory, one array per device; the launch's last CTA re-arms its slot).
//  * Eager launches: one slot per (device, stream).  Launches on one stream run in stream order
//    (each kernel's griddepcontrol.wait precedes its first ticket), so the previous launch has
//    re-armed the slot before the next one draws from it; launches on different streams never
//    share a counter.
//  * Launches being captured into a CUDA graph: a slot of their own that is never handed out
//    again (the slot is baked into the graph node; replays of one graph exec are serialised by
//    CUDA, and eager launches cannot collide with it).
// When the slots run out, the launch runs without the dynamic tail (static partition: same
// results, fewer GB/s) -- never a shared counter.
struct SchedSlots {
  std::mutex mu;
  unsigned int next[64] = {};
  std::unordered_map<uintptr_t, unsigned int> by_stream[64];
};
SchedSlots g_slots;

unsigned int* sched_slot(int dev, cudaStream_t st) {
  static std::atomic<unsigned int*> base[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  unsigned int* b = base[dev].load(std::memory_order_acquire);
  if (b == nullptr) {
    void* ptr = nullptr;
    if (cudaGetSymbolAddress(&ptr, al::g_sched) != cudaSuccess) {
      (void)cudaGetLastError();
      return nullptr;
    }
    b = static_cast<unsigned int*>(ptr);
    base[dev].store(b, std::memory_order_release);  // same value from any racing thread
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_slots.mu);
  unsigned int slot;
  if (cap == cudaStreamCaptureStatusNone) {
    auto it = g_slots.by_stream[dev].find(reinterpret_cast<uintptr_t>(st));
    if (it != g_slots.by_stream[dev].end()) {
      slot = it->second;
    } else {
      if (g_slots.next[dev] >= static_cast<unsigned int>(al::kSchedSlots)) return nullptr;
      slot = g_slots.next[dev]++;
      g_slots.by_stream[dev].emplace(reinterpret_cast<uintptr_t>(st), slot);
    }
  } else {
    if (g_slots.next[dev] >= static_cast<unsigned int>(al::kSchedSlots)) return nullptr;
    slot = g_slots.next[dev]++;
  }
  return b + 2 * slot;
}

// Work-stealing protocol state (al::g_steal, bwd_steal.cuh), handed out like the ticket slots:
// one per (device, stream) for eager launches, one never reused per captured launch.
struct StealSlots {
  std::mutex mu;
  unsigned int next[64] = {};
  std::unordered_map<uintptr_t, unsigned int> by_stream[64];
};
StealSlots g_steal_slots;

al::StealSlot* steal_slot(int dev, cudaStream_t st) {
  static std::atomic<al::StealSlot*> base[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  al::StealSlot* b = base[dev].load(std::memory_order_acquire);
  if (b == nullptr) {
    void* ptr = nullptr;
    if (cudaGetSymbolAddress(&ptr, al::g_steal) != cudaSuccess) {
      (void)cudaGetLastError();
      return nullptr;
    }
    b = static_cast<al::StealSlot*>(ptr);
    base[dev].store(b, std::memory_order_release);
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_steal_slots.mu);
  unsigned int slot;
  if (cap == cudaStreamCaptureStatusNone) {
    auto it = g_steal_slots.by_stream[dev].find(reinterpret_cast<uintptr_t>(st));
    if (it != g_steal_slots.by_stream[dev].end()) {
      slot = it->second;
    } else {
      if (g_steal_slots.next[dev] >= static_cast<unsigned int>(al::kStealSlots)) return nullptr;
      slot = g_steal_slots.next[dev]++;
      g_steal_slots.by_stream[dev].emplace(reinterpret_cast<uintptr_t>(st), slot);
    }
  } else {
    if (g_steal_slots.next[dev] >= static_cast<unsigned int>(al::kStealSlots)) return nullptr;
    slot = g_steal_slots.next[dev]++;
  }
  return b + slot;
}

// Backward load balancing.  2 (default, "auto") = deterministic work stealing (adaln_bwd_steal)
// for multi-sample launches of short samples (>= 2 groups of <= kStealAutoMaxS rows: the
// sampler's buckets, where the alternative is a static contiguous partition -- B200, separate
// processes, profiles/r2_steal_buckets_ab.jsonl: 307 x 1 560 2 410 -> 2 271 us, 133 x 3 600
// 2 400 -> 2 256, 49 x 7 800 1 917 -> 1 803, 15 x 14 040 1 080 -> 1 011; at 7 x 20 280 and
// 2 x 32 760 the last group's dynamic tail is faster, so longer samples steal only in
// deterministic launches), elsewhere the dynamic tail / static partition; 1 = stealing wherever
// it fits; 0 = never.  AL_BWD_STEAL overrides.
constexpr int64_t kStealAutoMaxS = 16384;
int bwd_steal_mode() {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_STEAL");
    return v ? std::atoi(v) : 2;
  }();
  return m;
}
// rows per stealable chunk (AL_STEAL_CHUNK overrides; a multiple of the 2-row stage) and the
// pool of stolen-chunk slots per launch in units of G (AL_STEAL_POOL; 0 disables stealing, the
// chunked partition then runs statically)
int steal_chunk_rows() {
  static const int c = [] {
    const char* v = std::getenv("AL_STEAL_CHUNK");
    const int x = v ? std::atoi(v) : 32;  // 8 / 16 / 64 measured 1-4 % slower on the buckets
    return x >= 2 ? (x + 1) / 2 * 2 : 32;
  }();
  return c;
}
int steal_pool_factor() {
  static const int f = [] {
    const char* v = std::getenv("AL_STEAL_POOL");
    return v ? std::atoi(v) : 2;
  }();
  return f;
}

int bwd_det_lean() {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_DET_LEAN");
    return v ? std::atoi(v) : 1;
  }();
  return m;
}

int64_t pipe_max_rows() {
  static const int64_t m = [] {
    const char* v = std::getenv("AL_BWD_PIPE_ROWS");
    // below the dynamic tail's 64-rows-per-CTA floor (9 472 rows at 148 CTAs) plus margin:
    // at S = 14 040 the lock-step kernel's dynamic tail is faster (75.0 vs 76.3 us)
    return v ? static_cast<int64_t>(std::atoll(v)) : int64_t(12288);
  }();
  return m;
}

int bwd_interleave() {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_INTERLEAVE");
    return v ? std::atoi(v) : 1;
  }();
  return m;
}

// Fraction of the rows handed out dynamically by the 16-bit rows forward (the rest is a static
// even split), capped at one modulation group.  Measured at cfg2 (bf16 D = 5 120, B200,
// tools/bw_probe.py): forward 5 449 GB/s static, 5 699 / 6 004 / 6 093 / 6 110 / 6 174 GB/s
// at 0.1 / 0.2 / 0.4 / 0.6 / 0.8.  AL_FWD_DYN overrides (0 disables).
double fwd_dyn_frac() {
  static const double f = [] {
    const char* v = std::getenv("AL_FWD_DYN");
    return v ? std::atof(v) : 0.8;
  }();
  return f;
}

// K2 / K2s ring-slot release point (DESIGN 3.2.1): each consumer warp arrives on the slot's
// empty barrier 1 = after phase 1, whose row sums consume every value the warp loaded from the
// slot (before the row-sum reduction and the stage barrier), 0 = after the stage barrier (the
// round-2 kernels before the pace study).  Releasing earlier keeps more of the ring in flight:
// B200 A/B (profiles/r2_bwd_early_release.jsonl) cfg2 deterministic 164.0 -> 161.2 us, ticketed
// 166.4 -> 164.4 us; 14 040 .. 75 600 alike.  (A release right after the shared loads were
// issued was 0.7 % faster still but raced with the refill -- tools/bwd_race_stress.py -- and is
// gone.)  AL_BWD_EARLY overrides.
int bwd_early_release(bool /*ticketed*/) {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_EARLY");
    return v ? (std::atoi(v) ? 1 : 0) : 1;
  }();
  return m;
}

// Single-group launches (one sample, or scale/shift broadcast) without AL_BWD_DETERMINISTIC:
// 0 = the ticketed dynamic walk (default), 1 = the interleaved static walk of deterministic
// launches.  Bench-mode A/B on three boxes with the slot released after phase 1
// (profiles/r2_bwd_schedule_bench_ab3.jsonl, profiles/r2_bwd_defaults_bench_ab_final.jsonl): the
// ticket walk's step is 0.8 % faster (6 232-6 249 vs 6 183-6 199 GB/s; backward 159.1 vs
// 160.4 us, and the following forward ~1 us faster); deterministic launches keep the
// interleaved walk (160.8-161.2 us).  AL_BWD_TICKET=0 selects the interleaved walk for both.
int bwd_single_group_static() {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_TICKET");
    return v ? (std::atoi(v) ? 0 : 1) : 0;
  }();
  return m;
}

// Group-sequential interleaved walk for multi-sample launches of long samples (see
// al_adaln_backward): 1 = deterministic launches and launches of <= 4 samples, 2 = all
// launches, 0 = off.  AL_BWD_GROUP_WALK.  B200 (profiles/r2_bwd_group_walk.jsonl): 2 x 32 760
// deterministic 347 -> 312 us, non-deterministic 325 -> 313; 7 x 20 280 deterministic
// 702 -> 686.5 us, non-deterministic 670.4 (static + ticketed last sample) vs 688 walked.
int bwd_group_walk() {
  static const int m = [] {
    const char* v = std::getenv("AL_BWD_GROUP_WALK");
    return v ? std::atoi(v) : 1;
  }();
  return m;
}

// Backward: fraction of the rows in the dynamic tail (capped at the last group).  Measured at
// cfg2 (tools/bw_probe.py, B200): backward 5 870 GB/s static (the previous loop; 5 087 for
// this loop, whose faster CTAs expose the uneven bandwidth split), 5 999 / 6 077 / 6 107 /
// 6 127 / 6 160 / 6 325 GB/s at 0.15 / 0.2 / 0.3 / 0.5 / 0.8 / 1.0.  AL_BWD_DYN overrides
// (0 disables).
double bwd_dyn_frac() {
  static const double f = [] {
    const char* v = std::getenv("AL_BWD_DYN");
    return v ? std::atof(v) : 1.0;
  }();
  return f;
}

// multi_group: the tail may span modulation groups (chunked, restaged per chunk; the plain
// forward -- the gated-residual twin measured 2-4 % slower with it at D = 1 536, 300 x 1 600 ..
// 8 x 9 450, profiles/r2_resid_multigroup_tail.jsonl, and keeps its tail in the last group).
// AL_FWD_DYN_GROUPS=0 disables.
// AL_FWD_DYN_GROUPS=2: the chunked tail for single-group launches too (A/B runs).
int fwd_dyn_groups() {
  static const int m = [] {
    const char* v = std::getenv("AL_FWD_DYN_GROUPS");
    return v ? std::atoi(v) : 1;
  }();
  return m;
}
void enable_dynamic_tail(const Plan& pl, al::FwdParams& p, cudaStream_t st, bool multi_group) {
  const double f = fwd_dyn_frac();
  if (!(f > 0.0) || pl.path != 2 || pl.R != 2) return;
  const int64_t warps = static_cast<int64_t>(pl.grid) * (pl.threads / 32);
  const int64_t want = static_cast<int64_t>(static_cast<double>(p.N) * (f < 1.0 ? f : 1.0));
  // Single group, or the residual twin: the tail stays inside the last modulation group (the
  // kernel stages that group once).  Multi-sample launches (the sampler's buckets, e.g. 307 x
  // 1 560 rows) otherwise ran a static split over 99.7 % of their rows: per-CTA end times
  // 1 225 .. 1 665 us at that bucket (profiles/r2_multigroup.jsonl).
  // The multi-group tail is whole groups handed out in chunks (the kernel restages per chunk).
  const bool span = multi_group && fwd_dyn_groups() && (p.S_grp < p.N || fwd_dyn_groups() == 2);
  const int64_t n_dyn = span ? p.N - (p.N - want) / p.S_grp * p.S_grp
                             : std::min<int64_t>(want, p.S_grp);
  p.dyn_groups = span ? 1 : 0;
  // short launches (< 2 tail rows per warp) are one wave anyway: the ticket round trip only
  // adds latency there (cfg3 S = 3 600: 3 739 vs 3 924 GB/s fwd+bwd)
  if (n_dyn < 2 * warps) return;
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  unsigned int* slot = sched_slot(dev, st);
  if (slot == nullptr) return;
  p.sched = slot;
  p.N_static = p.N - n_dyn;
}

int launch(const Plan& pl, al::FwdParams& p, void* stream, const char* what) {
  void* args[] = {&p};
  cudaError_t e = launch_k(pl.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem,
                           static_cast<cudaStream_t>(stream), kPdlFwd);
  if (e != cudaSuccess) return cuda_fail(e, what);
  return AL_OK;
}

// ---------------------------------------------------------------- fused Q/K RMSNorm
constexpr int kQkVpl[] = {1, 2, 3, 4, 6, 8};
constexpr int kQkNumVpl = 6;

template <typename T>
const void* qk_kernel_t(bool bwd, int vi) {
  switch (vi) {
    case 0: return bwd ? (const void*)al::qk_rms_bwd<T, 1> : (const void*)al::qk_rms_fwd<T, 1>;
    case 1: return bwd ? (const void*)al::qk_rms_bwd<T, 2> : (const void*)al::qk_rms_fwd<T, 2>;
    case 2: return bwd ? (const void*)al::qk_rms_bwd<T, 3> : (const void*)al::qk_rms_fwd<T, 3>;
    case 3: return bwd ? (const void*)al::qk_rms_bwd<T, 4> : (const void*)al::qk_rms_fwd<T, 4>;
    case 4: return bwd ? (const void*)al::qk_rms_bwd<T, 6> : (const void*)al::qk_rms_fwd<T, 6>;
    default: return bwd ? (const void*)al::qk_rms_bwd<T, 8> : (const void*)al::qk_rms_fwd<T, 8>;
  }
}
const void* qk_kernel(int dtype, bool bwd, int vi) {
  switch (dtype) {
    case AL_BF16: return qk_kernel_t<__nv_bfloat16>(bwd, vi);
    case AL_F16: return qk_kernel_t<__half>(bwd, vi);
    case AL_F64: return qk_kernel_t<double>(bwd, vi);
    default: return qk_kernel_t<float>(bwd, vi);
  }
}

// Launch plan shared by the workspace query and the launches: persistent grid of SMs x resident
// CTAs (capped by rows / warps); the backward keeps per-warp dw accumulators in shared memory,
// so it runs 8 warps per CTA when they fit in ~110 KB and 4 otherwise.
int qk_plan(bool bwd, int64_t N, int64_t D, int dtype, Plan* out) {
  const int es = elem_size(dtype), cs = ct_size(dtype);
  if (es == 0) return fail(AL_ERR_DTYPE, "unsupported dtype code %d", dtype);
  if ((D * es) % 16 != 0)
    return fail(AL_ERR_SHAPE, "qk-norm needs dim * element size to be a multiple of 16 bytes");
  const int64_t nvec = D * es / 16;
  if (nvec > 32 * 8)
    return fail(AL_ERR_SHAPE, "qk-norm supports rows of at most 256 16-byte vectors (D <= %d here)",
                static_cast<int>(256 * 16 / es));
  int vi = 0;
  while (32 * kQkVpl[vi] < nvec) ++vi;
  int dev, sms;
  int rc = current_device(&dev);
  if (!rc) rc = dev_sms(dev, &sms);
  if (rc) return rc;
  Plan pl;
  pl.path = 2;
  pl.V = kQkVpl[vi];
  pl.fn = qk_kernel(dtype, bwd, vi);
  pl.threads = 256;
  pl.smem = 2 * static_cast<size_t>(D) * cs;
  if (bwd) {
    const size_t per_warp = 2 * static_cast<size_t>(D) * cs;
    if (pl.smem + 8 * per_warp > 110 * 1024) pl.threads = 128;
    pl.smem += (pl.threads / 32) * per_warp;
  }
  int occ = 0;
  rc = occupancy(pl, dev, &occ);
  if (rc) return rc;
  if (occ < 1) return fail(AL_ERR_SHAPE, "qk-norm launch does not fit on this device");
  const int64_t warps = pl.threads / 32;
  pl.grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(static_cast<int64_t>(sms) * occ, (N + warps - 1) / warps)));
  *out = pl;
  return AL_OK;
}

// ---------------------------------------------------------------- gated-residual backward
template <typename T>
const void* gr_kernel_t(int V) {
  return V == 1 ? (const void*)al::gate_residual_bwd<T, 1>
                : (V == 2 ? (const void*)al::gate_residual_bwd<T, 2> : (const void*)al::gate_residual_bwd<T, 4>);
}
const void* gr_kernel(int dtype, int V) {
  switch (dtype) {
    case AL_BF16: return gr_kernel_t<__nv_bfloat16>(V);
    case AL_F16: return gr_kernel_t<__half>(V);
    case AL_F64: return gr_kernel_t<double>(V);
    default: return gr_kernel_t<float>(V);
  }
}

// Column-owner layout: V 16-byte vectors per thread, <= 512 threads; persistent grid of
// SMs x resident CTAs, capped by the rows.
int gr_plan(int64_t N, int64_t D, int dtype, Plan* out) {
  const int es = elem_size(dtype);
  if (es == 0) return fail(AL_ERR_DTYPE, "unsupported dtype code %d", dtype);
  if ((D * es) % 16 != 0)
    return fail(AL_ERR_SHAPE, "gated-residual backward needs dim * element size % 16 == 0");
  const int64_t nvec = D * es / 16;
  int V = 1;
  while (V < 4 && (nvec + V - 1) / V > 512) V *= 2;
  const int64_t nc = std::max<int64_t>(32, ((nvec + V - 1) / V + 31) / 32 * 32);
  if (nc > 512) return fail(AL_ERR_SHAPE, "dim too large for the gated-residual backward");
  int dev, sms;
  int rc = current_device(&dev);
  if (!rc) rc = dev_sms(dev, &sms);
  if (rc) return rc;
  Plan pl;
  pl.path = 1;
  pl.V = V;
  pl.threads = static_cast<int>(nc);
  pl.fn = gr_kernel(dtype, V);
  int occ = 0;
  rc = occupancy(pl, dev, &occ);
  if (rc) return rc;
  if (occ < 1) return fail(AL_ERR_SHAPE, "gated-residual backward launch does not fit");
  pl.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(sms) * occ, N)));
  *out = pl;
  return AL_OK;
}

__global__ void clock_probe_kernel(unsigned long long* out, unsigned int spin_ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const long long c0 = clock64();
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < spin_ns);
  const long long c1 = clock64();
  out[0] = t1 - t0;
  out[1] = static_cast<unsigned long long>(c1 - c0);
}

}  // namespace

extern "C" {

int al_debug_steal_count(int device_slot, unsigned int* out) {
  if (!out || device_slot < 0 || device_slot >= al::kStealSlots)
    return fail(AL_ERR_VALUE, "bad slot or output");
  cudaError_t e = cudaMemcpyFromSymbol(out, al::g_steal, sizeof(unsigned int),
                                       device_slot * sizeof(al::StealSlot) +
                                           offsetof(al::StealSlot, stolen));
  return e == cudaSuccess ? AL_OK : cuda_fail(e, "cudaMemcpyFromSymbol");
}

int al_debug_set_timestamps(unsigned long long* buf, int capacity) {
  if (buf != nullptr && capacity <= 0) return fail(AL_ERR_VALUE, "capacity must be positive");
  g_ts_buf.store(nullptr, std::memory_order_release);
  g_ts_cap.store(buf ? capacity : 0, std::memory_order_release);
  g_ts_next.store(0u);
  g_ts_buf.store(buf, std::memory_order_release);
  return AL_OK;
}

int al_debug_clock_probe(unsigned long long* out, unsigned int spin_ns, void* stream) {
  if (!out) return fail(AL_ERR_SHAPE, "null output pointer");
  clock_probe_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(out, spin_ns);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AL_OK : cuda_fail(e, "clock probe launch");
}

int al_abi_version(void) { return 5; }

#ifdef AL_CTA_TRACE
// Trace builds only: copy the per-CTA [start, end] globaltimer stamps of the last forward
// (kernel 0) or backward (kernel 1) launch to host memory.
AL_API int al_debug_cta_trace(int kernel, unsigned long long* out, int n) {
  if (n > 2 * 4096) n = 2 * 4096;
  return cudaMemcpyFromSymbol(out, al::g_cta_trace, n * sizeof(unsigned long long),
                              kernel * 2 * 4096 * sizeof(unsigned long long)) == cudaSuccess ? 0 : 1;
}
AL_API int al_debug_cta_info(unsigned long long* out, int n) {
  if (n > 4096) n = 4096;
  return cudaMemcpyFromSymbol(out, al::g_cta_info, n * sizeof(unsigned long long)) == cudaSuccess
             ? 0 : 1;
}
#endif

const char* al_last_error(void) { return g_err; }

int al_set_tuning(int kernel, int vecs_per_thread, int rows_per_stage, int smem_budget,
                  int force_generic, int variant) {
  if (kernel < 0 || kernel > 1) return fail(AL_ERR_VALUE, "kernel must be 0 or 1");
  if (vecs_per_thread && vecs_per_thread != 1 && vecs_per_thread != 2 && vecs_per_thread != 4)
    return fail(AL_ERR_VALUE, "vecs_per_thread must be 0,1,2,4");
  if (rows_per_stage && rows_per_stage != 1 && rows_per_stage != 2 && rows_per_stage != 4)
    return fail(AL_ERR_VALUE, "rows_per_stage must be 0,1,2,4");
  std::lock_guard<std::mutex> lk(g_mu);
  g_tune[kernel].V = vecs_per_thread;
  g_tune[kernel].R = rows_per_stage;
  g_tune[kernel].smem_budget = smem_budget;
  g_tune[kernel].force_generic = force_generic;
  g_tune[kernel].variant = variant;
  return AL_OK;
}

int al_device_init(int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  int sms;
  int rc = dev_sms(device, &sms);
  if (rc) return rc;
  for (int dt = 0; dt < 4; ++dt) {
    for (int kernel = 0; kernel < 2; ++kernel) {
      for (int V : {1, 2, 4})
        for (int R : {1, 2, 4})
          for (bool full : {false, true}) {
            rc = ensure_attr(tma_kernel(kernel, dt, V, R, full), device);
            if (rc) return rc;
            if (kernel == 1 && R == 2) {
              rc = ensure_attr(steal_kernel(dt, V, full), device);
              if (!rc) rc = ensure_attr(steal_kernel(dt, V, full, 352), device);
              if (rc) return rc;
            }
            if (kernel == 1 && tma_dyn_kernel(dt, V, R, full)) {
              rc = ensure_attr(tma_dyn_kernel(dt, V, R, full), device);
              if (rc) return rc;
            }
            if (kernel == 1 && tma_gw_kernel(dt, V, R, full)) {
              rc = ensure_attr(tma_gw_kernel(dt, V, R, full), device);
              if (rc) return rc;
            }
            if (kernel == 0) {
              rc = ensure_attr(tma_kernel(kernel, dt, V, R, full, true), device);
              if (rc) return rc;
            }
          }
      if (kernel == 0)
        for (int vi = 0; vi < kNumVpl; ++vi) {
          rc = ensure_attr(rows_kernel(dt, vi, false), device);
          if (rc) return rc;
          rc = ensure_attr(rows_kernel(dt, vi, true), device);
          if (rc) return rc;
          rc = ensure_attr(rows_kernel_pf(dt, vi), device);
          if (rc) return rc;
          rc = ensure_attr(rows_staged_kernel(dt, vi), device);
          if (rc) return rc;
          rc = ensure_attr(resid_kernel(dt, vi), device);
          if (rc) return rc;
          rc = ensure_attr(rows2_kernel(dt, vi), device);
          if (rc) return rc;
          if (dt == AL_BF16 || dt == AL_F16) {
            rc = ensure_attr(rows16_kernel(dt, vi), device);
            if (rc) return rc;
            rc = ensure_attr(rows16_resid_kernel(dt, vi), device);
            if (rc) return rc;
          }
        }
      cudaFuncAttributes fa;
      e = cudaFuncGetAttributes(&fa, generic_kernel(kernel, dt));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
    }
    {
      cudaFuncAttributes fa;
      e = cudaFuncGetAttributes(&fa, resid_generic_kernel(dt));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
    }
    for (int vi = 0; vi < kQkNumVpl; ++vi)
      for (bool b : {false, true}) {
        rc = ensure_attr(qk_kernel(dt, b, vi), device);
        if (rc) return rc;
      }
    for (int V : {1, 2, 4}) {
      rc = ensure_attr(gr_kernel(dt, V), device);
      if (rc) return rc;
    }
    for (bool vec : {false, true}) {
      cudaFuncAttributes fa;
      e = cudaFuncGetAttributes(&fa, reduce_kernel(dt, vec));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
    }
  }
  return AL_OK;
}

int al_describe_launch(int kernel, int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                       int dtype, int64_t n_tile, int64_t out[7]) {
  int rc = check_common(batch, seq, dim, mod_stride, dtype);
  if (rc) return rc;
  if (kernel < 0 || kernel > 1) return fail(AL_ERR_VALUE, "kernel must be 0 or 1");
  Plan pl;
  const void* aligned[1] = {reinterpret_cast<const void*>(uintptr_t(256))};
  rc = make_plan(kernel, batch * seq, dim, mod_stride, dtype, n_tile, aligned, 1, &pl);
  if (rc) return rc;
  out[0] = pl.path;
  out[1] = pl.grid;
  out[2] = pl.threads;
  out[3] = pl.V;
  out[4] = pl.R;
  out[5] = pl.NS;
  out[6] = static_cast<int64_t>(pl.smem);
  return AL_OK;
}

int al_adaln_forward(const void* x, const void* scale, const void* shift, void* y, void* mean,
                     void* rstd, int64_t batch, int64_t seq, int64_t dim, int64_t mod_stride,
                     int dtype, double eps, int* nonfinite, void* stream) {
  int rc = check_common(batch, seq, dim, mod_stride, dtype);
  if (rc) return rc;
  if (!(eps > 0.0)) return fail(AL_ERR_VALUE, "eps must be positive");
  const int64_t N = batch * seq;
  if (N == 0) return AL_OK;
  if (!x || !scale || !shift || !y || !mean || !rstd)
    return fail(AL_ERR_SHAPE, "null tensor pointer");
  const void* vp[4] = {x, y, scale, shift};
  Plan pl;
  rc = make_plan(0, N, dim, mod_stride, dtype, 0, vp, 4, &pl);
  if (rc) return rc;
  al::FwdParams p = fwd_params(x, scale, shift, y, mean, rstd, seq, N, dim, mod_stride, dtype,
                               eps, nonfinite, pl);
  p.ts = next_ts();
  enable_dynamic_tail(pl, p, static_cast<cudaStream_t>(stream), true);
  return launch(pl, p, stream, "forward launch");
}

int al_adaln_gate_residual_forward(const void* x, const void* f, const void* gate,
                                   const void* scale, const void* shift, void* x_out, void* y,
                                   void* mean, void* rstd, int64_t batch, int64_t seq,
                                   int64_t dim, int64_t mod_stride, int dtype, double eps,
                                   int* nonfinite, void* stream) {
  int rc = check_common(batch, seq, dim, mod_stride, dtype);
  if (rc) return rc;
  if (!(eps > 0.0)) return fail(AL_ERR_VALUE, "eps must be positive");
  const int64_t N = batch * seq;
  if (N == 0) return AL_OK;
  if (!x || !f || !gate || !scale || !shift || !x_out || !y || !mean || !rstd)
    return fail(AL_ERR_SHAPE, "null tensor pointer");
  if (x_out == x || x_out == f) return fail(AL_ERR_VALUE, "x_out may not alias x or f");
  const void* vp[7] = {x, f, gate, x_out, y, scale, shift};
  const int es = elem_size(dtype);
  bool vec_ok = (dim * es) % 16 == 0 && (mod_stride * es) % 16 == 0;
  for (int i = 0; i < 7 && vec_ok; ++i) vec_ok = aligned16(vp[i]);
  const int64_t nvec = dim * es / 16;
  if (vec_ok && nvec <= 32 * kMaxVpl) {
    // fused: the rows kernel's gated-residual twin (one warp per row, +1 smem row for gate)
    int vi = 0;
    while (32 * kVpl[vi] < nvec) ++vi;
    Plan pr;
    pr.path = 2;
    pr.V = kVpl[vi];
    // 16-bit rows of <= 8 vectors per lane (D <= 2 048): the mixed-precision rows16 twin with
    // the dynamic row tail (pr.R = 2 marks it for enable_dynamic_tail): D = 1 536 5 859 ->
    // 6 259 GB/s (B = 8, S = 9 450).  Wider rows spill in that kernel (1 KB at D = 5 120:
    // 3 940 vs 4 949 GB/s), so they and other dtypes take the packed rows kernel's twin.
    const bool is16 = (dtype == AL_BF16 || dtype == AL_F16) && kVpl[vi] <= 8;
    pr.fn = is16 ? rows16_resid_kernel(dtype, vi) : resid_kernel(dtype, vi);
    pr.R = is16 ? 2 : 1;
    pr.threads = 256;
    pr.smem = 3 * static_cast<size_t>(dim) * ct_size(dtype);
    int dev, sms, occ = 0;
    rc = current_device(&dev);
    if (!rc) rc = dev_sms(dev, &sms);
    if (!rc) rc = occupancy(pr, dev, &occ);
    if (rc) return rc;
    if (occ >= 1) {
      const int64_t grid = std::min<int64_t>(static_cast<int64_t>(sms) * occ, (N + 7) / 8);
      pr.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(N, grid)));
      al::FwdParams p = fwd_params(x, scale, shift, y, mean, rstd, seq, N, dim, mod_stride,
                                   dtype, eps, nonfinite, pr);
      p.f = f;
      p.gate = gate;
      p.x_out = x_out;
      enable_dynamic_tail(pr, p, static_cast<cudaStream_t>(stream), false);
      return launch(pr, p, stream, "gate-residual forward launch");
    }
  }
  // unfused: residual kernel, then the forward plan on x_out
  {
    int dev, sms;
    rc = current_device(&dev);
    if (!rc) rc = dev_sms(dev, &sms);
    if (rc) return rc;
    Plan pg;
    pg.threads = 256;
    pg.fn = resid_generic_kernel(dtype);
    pg.grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((N * dim + 255) / 256, static_cast<int64_t>(sms) * 8)));
    al::FwdParams p = fwd_params(x, scale, shift, y, mean, rstd, seq, N, dim, mod_stride, dtype,
                                 eps, nonfinite, pg);
    p.f = f;
    p.gate = gate;
    p.x_out = x_out;
    rc = launch(pg, p, stream, "gate-residual launch");
    if (rc) return rc;
  }
  return al_adaln_forward(x_out, scale, shift, y, mean, rstd, batch, seq, dim, mod_stride, dtype,
                          eps, nonfinite, stream);
}

int64_t al_adaln_backward_workspace_bytes(int64_t batch, int64_t seq, int64_t dim,
                                          int64_t mod_stride, int dtype, int64_t n_tile) {
  if (check_common(batch, seq, dim, mod_stride, dtype)) return -1;
  const int64_t N = batch * seq;
  if (N == 0) return 0;
  // the larger of the vector-path and generic-path plans, so any pointer alignment fits
  Plan pa, pg;
  const void* aligned[1] = {reinterpret_cast<const void*>(uintptr_t(256))};
  if (make_plan(1, N, dim, mod_stride, dtype, n_tile, aligned, 1, &pa)) return -1;
  if (make_plan(1, N, dim, mod_stride, dtype, n_tile, aligned, 1, &pg, true)) return -1;
  const int64_t ngroups = mod_stride ? batch : 1;
  // static slots (G + groups - 1) + the larger of the dynamic tail's G slots and the work
  // stealing pool (2G); + 16 bytes: the fused stage-2 grid-barrier counter
  int64_t slots = std::max(pa.grid, pg.grid) + ngroups - 1 + 2 * pa.grid;
  // the group-sequential walk of long samples: G slots per sample
  if (ngroups >= 2 && seq > kStealAutoMaxS) slots = std::max<int64_t>(slots, pa.grid * ngroups);
  return 2 * slots * dim * ct_size(dtype) + 16;
}

int al_adaln_backward(const void* dy, const void* x, const void* scale, const void* mean,
                      const void* rstd, void* dx, void* dscale, void* dshift, void* workspace,
                      int64_t workspace_bytes, int64_t batch, int64_t seq, int64_t dim,
                      int64_t mod_stride, int dtype, int64_t d_tile, int64_t n_tile,
                      int flags, int* nonfinite, void* stream) {
  int rc = check_common(batch, seq, dim, mod_stride, dtype);
  if (rc) return rc;
  const int64_t N = batch * seq;
  const int64_t S_grp = mod_stride ? seq : N;
  const int64_t ngroups = mod_stride ? batch : 1;
  if (d_tile != 0 || n_tile != 0) {
    if (!(d_tile >= 1 && d_tile <= dim && n_tile >= 1 && n_tile <= S_grp))
      return fail(AL_ERR_TILE, "tile config (d_tile=%lld, n_tile=%lld) out of bounds for N=%lld, D=%lld",
                  (long long)d_tile, (long long)n_tile, (long long)S_grp, (long long)dim);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (N == 0) {
    if (ngroups > 0 && dscale && dshift) {
      cudaError_t e = cudaMemsetAsync(dscale, 0, ngroups * dim * ct_size(dtype), st);
      if (e == cudaSuccess) e = cudaMemsetAsync(dshift, 0, ngroups * dim * ct_size(dtype), st);
      if (e != cudaSuccess) return cuda_fail(e, "memset");
    }
    return AL_OK;
  }
  if (!dy || !x || !scale || !mean || !rstd || !dx || !dscale || !dshift)
    return fail(AL_ERR_SHAPE, "null tensor pointer");
  const void* vp[5] = {dy, x, scale, dx, workspace};
  Plan pl;
  rc = make_plan(1, N, dim, mod_stride, dtype, n_tile, vp, 5, &pl);
  if (rc) return rc;
  const int cs = ct_size(dtype);
  const bool vec = (dim * cs) % 16 == 0 && aligned16(workspace);
  Tuning tu;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    tu = g_tune[1];
  }
  const int64_t nslots_static = pl.grid + ngroups - 1;
  // Dynamic tail (see adaln_bwd_tma): TMA path, vector stage 2, no explicit n_tile, not the
  // cooperative fused stage 2, caller did not ask for AL_BWD_DETERMINISTIC, and at least two
  // stages per CTA in the tail (which stays inside the last group).
  // Short launches (<= pipe_max_rows() rows, ~80 rows per CTA at D = 5 120) take the
  // skewed-pipeline kernel with its static partition: its barrier-free stages fill the few
  // stages a CTA has faster (B200, device timestamps: S = 1 560 / 3 600 / 7 800 and B = 4, 8
  // x 1 560: 7-9 % less time than the lock-step kernel; equal at 14 040; 3 % more at 32 760,
  // profiles/r2_bwd_variants.jsonl).  Deterministic either way.
  const bool pipe_auto = tu.variant == 0 && pl.path == 1 && vec && n_tile == 0 &&
                         N <= pipe_max_rows() && pl.V == 2 &&
                         (dtype == AL_BF16 || dtype == AL_F16);
  int64_t n_dyn = 0;
  if (!pipe_auto && pl.path == 1 && vec && n_tile == 0 && tu.variant != 2 &&
      !(flags & AL_BWD_DETERMINISTIC) && !(S_grp == N && bwd_single_group_static())) {
    const double f = bwd_dyn_frac();
    n_dyn = std::min<int64_t>(static_cast<int64_t>(static_cast<double>(N) * (f < 1.0 ? f : 1.0)),
                              S_grp);
    // short launches lose more to the second set of partial slots and the ticket traffic than
    // they gain (cfg3 S = 1 560: 34.2 vs 29.0 us fwd+bwd; break-even near S = 10 000 at
    // D = 5 120): >= 64 tail rows per CTA
    if (n_dyn < 64 * static_cast<int64_t>(pl.grid)) n_dyn = 0;
    // stage 2 sums the static slots of every CTA between the owners of a group's first and last
    // static rows; with 0 < N_static < G some of those CTAs would own no rows and never write
    // their slot, so a static head is either empty or at least one row per CTA
    const int64_t n_static = N - n_dyn;
    if (n_static > 0 && n_static < pl.grid) n_dyn = 0;
  }
  // Deterministic work stealing (bwd_steal.cuh): replaces both the dynamic tail and the plain
  // static partition wherever it fits (TMA path with 2-row stages, vector stage 2, default
  // tiling, >= 2 chunks per CTA); dscale/dshift are then bit-identical run to run whatever the
  // caller's determinism flag.
  // Group-sequential interleaved walk (bwd_group_walk): multi-sample launches of long samples
  // (> kStealAutoMaxS rows each; deterministic, or at most 4 samples) walk each sample like a
  // single-sample launch, one sample after the other, with G partial slots per sample -- if the
  // caller's workspace holds them (al_adaln_backward_workspace_bytes sizes for it).
  bool group_walk = false;
  if (bwd_group_walk() && !pipe_auto && pl.path == 1 && vec && n_tile == 0 && tu.variant == 0 &&
      ngroups >= 2 && S_grp > kStealAutoMaxS &&
      ((flags & AL_BWD_DETERMINISTIC) || bwd_group_walk() == 2 || ngroups <= 4) &&
      workspace_bytes >= 2 * static_cast<int64_t>(pl.grid) * ngroups * dim * cs) {
    int dev;
    const bool full = pl.threads - 32 == dim * elem_size(dtype) / 16 / pl.V &&
                      (dim * elem_size(dtype) / 16) % pl.V == 0;
    const void* gfn = tma_gw_kernel(dtype, pl.V, pl.R, full);
    if (gfn && cudaGetDevice(&dev) == cudaSuccess && ensure_attr(gfn, dev) == AL_OK) {
      group_walk = true;
      n_dyn = 0;
    }
  }
  bool use_steal = false;
  al::StealSlot* sslot = nullptr;
  const void* sfn = nullptr;
  size_t steal_smem = 0;
  // (tuning variant 4 = the round-1 scheme, for A/B runs)
  // (deterministic multi-group launches of longer samples have no dynamic tail to lose: 7 x
  // 20 280 730 -> 707 us, 2 x 32 760 341 -> 343)
  const bool steal_wanted =
      bwd_steal_mode() == 1 ||
      (bwd_steal_mode() == 2 && ngroups >= 2 &&
       (S_grp <= kStealAutoMaxS || (flags & AL_BWD_DETERMINISTIC)));
  if (!group_walk && steal_wanted && !pipe_auto && pl.path == 1 && vec && n_tile == 0 &&
      tu.variant != 2 && tu.variant != 3 && tu.variant != 4 && pl.R == 2 && pl.grid <= al::kStealMaxG &&
      N >= 2 * steal_chunk_rows() * static_cast<int64_t>(pl.grid)) {
    const int nvec_ = static_cast<int>(dim * elem_size(dtype) / 16);
    const bool full = pl.threads - 32 == nvec_ / pl.V && nvec_ % pl.V == 0;
    sfn = steal_kernel(dtype, pl.V, full, pl.threads);
    const int ncw = (pl.threads - 32) / 32;
    const size_t stage = 2 * 2 * static_cast<size_t>(dim * elem_size(dtype));
    // ring + barriers + headers + row-sum scratch + the [2][D] shared running total (the
    // kernel's layout, bwd_steal.cuh)
    auto r16 = [](size_t v) { return (v + 15) & ~size_t(15); };
    auto extra = [&](int ns) {
      return 16 * static_cast<size_t>(ns) + 24 * static_cast<size_t>(ns) +
             r16(2 * static_cast<size_t>(ns) * 2 * cs) + r16(8 * static_cast<size_t>(ns) + 4) +
             r16(2 * static_cast<size_t>(ncw) * 2 * 2 * cs) + 2 * static_cast<size_t>(dim) * cs;
    };
    int ns = pl.NS;
    while (ns > 3 && ns * stage + extra(ns) > static_cast<size_t>(kSmemOptin)) --ns;
    int dev;
    if (ns * stage + extra(ns) <= static_cast<size_t>(kSmemOptin) && cudaGetDevice(&dev) == cudaSuccess && ensure_attr(sfn, dev) == AL_OK) {
      sslot = steal_slot(dev, st);
      if (sslot != nullptr) {
        use_steal = true;
        n_dyn = 0;
        pl.NS = ns;
        steal_smem = ns * stage + extra(ns);
      }
    }
  }
  const int64_t nslots = group_walk ? static_cast<int64_t>(pl.grid) * ngroups
                                    : nslots_static + (use_steal ? steal_pool_factor() * pl.grid
                                                                 : (n_dyn ? pl.grid : 0));
  const int64_t need = 2 * nslots * dim * cs;
  if (!workspace || workspace_bytes < need) {
    return fail(AL_ERR_WORKSPACE, "workspace too small: need %lld bytes, got %lld",
                (long long)need, (long long)workspace_bytes);
  }
  al::BwdParams p;
  p.dy = dy;
  p.x = x;
  p.scale = scale;
  p.mean = mean;
  p.rstd = rstd;
  p.dx = dx;
  p.ws = workspace;
  p.N = N;
  p.S_grp = S_grp;
  p.D = dim;
  p.mod_stride = mod_stride;
  p.nslots = nslots;
  p.nonfinite = nonfinite;
  p.nvec = static_cast<int>(dim * elem_size(dtype) / 16);
  p.row_bytes = static_cast<int>(dim * elem_size(dtype));
  p.nstages = pl.NS;
  p.G = pl.grid;
  p.counter = nullptr;
  p.dscale = dscale;
  p.dshift = dshift;
  p.sched = nullptr;
  p.N_static = N;
  p.tail_slot0 = -1;
  p.ts = next_ts();
  p.steal = nullptr;
  p.chunk_rows = steal_chunk_rows();
  p.pool_cap = 0;
  p.interleave = 0;
  p.early_release = 0;  // set at launch (bwd_early_release)
  if (use_steal) {
    pl.fn = sfn;
    pl.smem = steal_smem;
    p.nstages = pl.NS;
    p.steal = sslot;
    p.pool_cap = steal_pool_factor() * pl.grid;
    p.tail_slot0 = nslots_static;  // pool slots follow the static ones
    if (S_grp == N && bwd_interleave()) {
      // interleaved chunks over the whole range: at most kStealMaxC per owner
      p.interleave = 1;
      const int64_t need = (N + static_cast<int64_t>(pl.grid) * al::kStealMaxC - 1) /
                           (static_cast<int64_t>(pl.grid) * al::kStealMaxC);
      int c = p.chunk_rows;
      if (need > c) c = static_cast<int>((need + 1) / 2 * 2);
      p.chunk_rows = c;
    }
  }
  // Interleaved static partition (single group): the static instance walks stages k, k+G, ...
  // -- a fixed, deterministic assignment whose CTAs sweep HBM together (AL_BWD_INTERLEAVE=0
  // restores the contiguous split)
  if (!use_steal && n_dyn == 0 && pl.path == 1 && vec && tu.variant != 2 && S_grp == N &&
      bwd_interleave() && (!pipe_auto || bwd_interleave() == 2))
    p.interleave = 1;  // (also honoured by the skewed-pipeline kernel's static instance)
  if (group_walk) {
    const bool full = pl.threads - 32 == p.nvec / pl.V && p.nvec % pl.V == 0;
    p.interleave = 2;
    pl.fn = tma_gw_kernel(dtype, pl.V, pl.R, full);
  }
  // Deterministic single-group launches: the interleaved static walk on the dynamic instance's
  // lean stage body (bit-identical to the static instance; B200, profiles/r2_det_lean.jsonl:
  // cfg2 169.2 -> 164.1 us, S = 75 600 371.8 -> 360.6, 14 040 80.9 -> 78.9; the dynamic tail
  // 161.1 / 357.3 / 76.5 on the same box).  AL_BWD_DET_LEAN=0 restores the static instance.
  if (p.interleave == 1 && !pipe_auto && n_dyn == 0 && bwd_det_lean()) {
    int dev;
    const bool full = pl.threads - 32 == p.nvec / pl.V && p.nvec % pl.V == 0;
    const void* dfn = tma_dyn_kernel(dtype, pl.V, pl.R, full);
    if (dfn && cudaGetDevice(&dev) == cudaSuccess && ensure_attr(dfn, dev) == AL_OK) pl.fn = dfn;
  }
  if (n_dyn) {
    int dev;
    const bool full = pl.threads - 32 == p.nvec / pl.V && p.nvec % pl.V == 0;
    const void* dfn = tma_dyn_kernel(dtype, pl.V, pl.R, full);
    unsigned int* slot = nullptr;
    if (dfn && cudaGetDevice(&dev) == cudaSuccess && ensure_attr(dfn, dev) == AL_OK)
      slot = sched_slot(dev, st);
    if (slot) {
      pl.fn = dfn;
      p.sched = slot;
      p.N_static = N - n_dyn;
      p.tail_slot0 = nslots_static;
    }
  }
  // Skewed-pipeline stage 1 (variant 3 while under evaluation): same ring/slot contract, its
  // own ring depth (the consumers hold two slots at a time)
  if (pl.path == 1 && (tu.variant == 3 || pipe_auto)) {
    const int R = tu.R ? tu.R : 2;
    const bool full = pl.threads - 32 == p.nvec / pl.V && p.nvec % pl.V == 0;
    const void* fn = pipe_kernel(dtype, pl.V, R, full, p.sched != nullptr);
    if (fn != nullptr && (R == 1 || R == 2)) {
      const int ncw = (pl.threads - 32) / 32;
      const size_t stage = 2 * static_cast<size_t>(R) * p.row_bytes;
      auto extra = [&](int ns) {
        return static_cast<size_t>(2 * ns + 4) * 8 + 4 * ncw * 2 * R * cs + 16 +
               static_cast<size_t>(ns) * (8 + 4 + 2 * R * cs) + 32;
      };
      // the ring plan's per-CTA shared memory, so the occupancy (and the grid the slots were
      // sized for) is unchanged
      const size_t budget = tu.smem_budget ? static_cast<size_t>(tu.smem_budget) : pl.smem;
      int ns = 2;
      while (ns < 12 && (ns + 1) * stage + extra(ns + 1) <= budget) ++ns;
      int dev;
      if (ns >= 3 && cudaGetDevice(&dev) == cudaSuccess && ensure_attr(fn, dev) == AL_OK) {
        pl.fn = fn;
        pl.NS = ns;
        pl.R = R;
        pl.smem = ns * stage + extra(ns);
        p.nstages = ns;
      }
    }
  }
  // Fused stage 2: the TMA kernel reduces the partials itself behind a grid barrier, which
  // needs a cooperative launch (all CTAs co-resident) and a zeroed counter at the workspace
  // tail.  Otherwise stage 2 is a second kernel.
  // opt-in (variant 2): measured equal to the separate kernel on B200 (0.189 ms both)
  p.early_release = bwd_early_release(p.sched != nullptr);
  const bool fuse = pl.path == 1 && vec && tu.variant == 2 &&
                    workspace_bytes >= need + 16 && cooperative_ok(pl);
  void* args[] = {&p};
  cudaError_t e;
  if (fuse) {
    p.counter = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(workspace) + need);
    e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
    e = cudaLaunchCooperativeKernel(pl.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "backward (fused) cooperative launch");
    return AL_OK;
  }
  p.early_release = bwd_early_release(p.sched != nullptr);
  e = launch_k(pl.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, st, kPdlBwd1);
  if (e != cudaSuccess) return cuda_fail(e, "backward stage-1 launch");
  // stage 2: 16-byte vector form when every partial row is 16-byte aligned
  const void* rk = reduce_kernel(dtype, vec);
  int64_t G64 = pl.grid;
  // stolen partials are merged by owners; -2: the group walk's slot map (g*G .. g*G + G - 1)
  int64_t k3_tail0 = group_walk ? -2 : (use_steal ? -1 : p.tail_slot0);
  void* rargs[] = {&workspace, &dscale, &dshift,     &p.N,      &p.S_grp, &p.D,
                   &G64,       &p.nslots, &p.N_static, &k3_tail0, &p.ts};
  const int64_t cols_per_cta = vec ? al::kRedCV * (16 / cs) : 32;
  if (!launch_reduce_grp(dtype, vec, ngroups, k3_tail0, dim, rargs, st, &e)) {
    dim3 rgrid(static_cast<unsigned>((dim + cols_per_cta - 1) / cols_per_cta),
               static_cast<unsigned>(ngroups));
    e = launch_k(rk, rgrid, dim3(vec ? 512 : 1024), rargs, 0, st, kPdlBwd2);
  }
  if (e != cudaSuccess) return cuda_fail(e, "backward stage-2 launch");
  return AL_OK;
}


int al_qk_rmsnorm_forward(const void* qkv, int64_t row_stride, const void* wq, const void* wk,
                          void* qn, void* kn, void* vc, void* rstd, int64_t n_rows, int64_t dim,
                          int dtype, double eps, int* nonfinite, void* stream) {
  if (n_rows < 0 || dim < 1) return fail(AL_ERR_SHAPE, "n_rows must be >= 0 and dim >= 1");
  if (!(eps > 0.0)) return fail(AL_ERR_VALUE, "eps must be positive");
  if (row_stride < (vc ? 3 : 2) * dim)
    return fail(AL_ERR_SHAPE, "row_stride must cover the q, k (and v) slices");
  if (n_rows == 0) return AL_OK;
  if (!qkv || !wq || !wk || !qn || !kn || !rstd) return fail(AL_ERR_SHAPE, "null tensor pointer");
  const int es = elem_size(dtype);
  const void* vp[6] = {qkv, wq, wk, qn, kn, vc ? vc : qn};
  for (const void* q : vp)
    if (!aligned16(q)) return fail(AL_ERR_SHAPE, "qk-norm tensors must be 16-byte aligned");
  if (es && (row_stride * es) % 16 != 0) return fail(AL_ERR_SHAPE, "row stride must be 16-byte aligned");
  Plan pl;
  int rc = qk_plan(false, n_rows, dim, dtype, &pl);
  if (rc) return rc;
  al::QKParams p = {};
  p.qkv = qkv;
  p.row_stride = row_stride;
  p.wq = wq;
  p.wk = wk;
  p.qn = qn;
  p.kn = kn;
  p.vc = vc;
  p.rstd = rstd;
  p.N = n_rows;
  p.D = dim;
  p.nvec = static_cast<int>(dim * es / 16);
  p.G = pl.grid;
  p.eps = eps;
  p.nonfinite = nonfinite;
  void* args[] = {&p};
  cudaError_t e = launch_k(pl.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem,
                           static_cast<cudaStream_t>(stream), 0);
  if (e != cudaSuccess) return cuda_fail(e, "qk-norm forward launch");
  return AL_OK;
}

int64_t al_qk_rmsnorm_backward_workspace_bytes(int64_t n_rows, int64_t dim, int dtype) {
  if (n_rows <= 0 || dim < 1) return n_rows == 0 ? 0 : -1;
  Plan pl;
  if (qk_plan(true, n_rows, dim, dtype, &pl)) return -1;
  return 2 * static_cast<int64_t>(pl.grid) * dim * ct_size(dtype);
}

int al_qk_rmsnorm_backward(const void* qkv, int64_t row_stride, const void* wq, const void* wk,
                           const void* rstd, const void* dqn, const void* dkn, const void* dv,
                           void* dqkv, void* dwq, void* dwk, void* workspace,
                           int64_t workspace_bytes, int64_t n_rows, int64_t dim, int dtype,
                           int* nonfinite, void* stream) {
  if (n_rows < 0 || dim < 1) return fail(AL_ERR_SHAPE, "n_rows must be >= 0 and dim >= 1");
  if (row_stride < (dv ? 3 : 2) * dim)
    return fail(AL_ERR_SHAPE, "row_stride must cover the q, k (and v) slices");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cs = ct_size(dtype), es = elem_size(dtype);
  if (n_rows == 0) {  // empty batch: the weight gradients are zero
    if (dwq && dwk) {
      cudaError_t e = cudaMemsetAsync(dwq, 0, dim * cs, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(dwk, 0, dim * cs, st);
      if (e != cudaSuccess) return cuda_fail(e, "memset");
    }
    return AL_OK;
  }
  if (!qkv || !wq || !wk || !rstd || !dqn || !dkn || !dqkv || !dwq || !dwk)
    return fail(AL_ERR_SHAPE, "null tensor pointer");
  const void* vp[7] = {qkv, wq, wk, dqn, dkn, dqkv, dv ? dv : dqn};
  for (const void* q : vp)
    if (!aligned16(q)) return fail(AL_ERR_SHAPE, "qk-norm tensors must be 16-byte aligned");
  if (es && (row_stride * es) % 16 != 0) return fail(AL_ERR_SHAPE, "row stride must be 16-byte aligned");
  Plan pl;
  int rc = qk_plan(true, n_rows, dim, dtype, &pl);
  if (rc) return rc;
  const int64_t need = 2 * static_cast<int64_t>(pl.grid) * dim * cs;
  if (!workspace || workspace_bytes < need)
    return fail(AL_ERR_WORKSPACE, "workspace too small: need %lld bytes", (long long)need);
  al::QKParams p = {};
  p.qkv = qkv;
  p.row_stride = row_stride;
  p.wq = wq;
  p.wk = wk;
  p.rstd = const_cast<void*>(rstd);
  p.dqn = dqn;
  p.dkn = dkn;
  p.dv = dv;
  p.dqkv = dqkv;
  p.ws = workspace;
  p.N = n_rows;
  p.D = dim;
  p.nvec = static_cast<int>(dim * es / 16);
  p.G = pl.grid;
  p.nonfinite = nonfinite;
  void* args[] = {&p};
  cudaError_t e = launch_k(pl.fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, st, kPdlBwd1);
  if (e != cudaSuccess) return cuda_fail(e, "qk-norm backward launch");
  // stage 2: dw_q | dw_k = sum of the G slots, ascending (the AdaLN stage-2 kernel, one group)
  const void* rk = reduce_kernel(dtype, true);
  int64_t N64 = n_rows, S64 = n_rows, D64 = dim, G64 = pl.grid, ns = pl.grid;
  int64_t tail0 = -1;
  unsigned long long* no_ts = nullptr;
  void* rargs[] = {&workspace, &dwq, &dwk, &N64, &S64, &D64, &G64, &ns, &N64, &tail0, &no_ts};
  const int64_t cols_per_cta = al::kRedCV * (16 / cs);
  e = launch_k(rk, dim3(static_cast<unsigned>((dim + cols_per_cta - 1) / cols_per_cta), 1),
               dim3(512), rargs, 0, st, kPdlBwd2);
  if (e != cudaSuccess) return cuda_fail(e, "qk-norm backward stage-2 launch");
  return AL_OK;
}


// Generic gated-residual backward plan (any width / alignment): 256 threads, [D] shared partials.
constexpr int64_t kGrGenericCols = 8192;  // columns per CTA of the generic kernel (<= 64 KB)
int gr_generic_plan(int64_t N, int64_t D, int dtype, Plan* out) {
  const int cs = ct_size(dtype);
  int dev, sms;
  int rc = current_device(&dev);
  if (!rc) rc = dev_sms(dev, &sms);
  if (rc) return rc;
  Plan pl;
  pl.path = 0;
  pl.threads = 256;
  pl.smem = static_cast<size_t>(std::min<int64_t>(D, kGrGenericCols)) * cs;
  pl.fn = with_table(dtype, [&](const auto& t) -> const void* {
    using TT = std::remove_cv_t<std::remove_reference_t<decltype(t)>>;
    (void)t;
    if constexpr (std::is_same_v<TT, Table<__nv_bfloat16>>) return (const void*)al::gate_residual_bwd_generic<__nv_bfloat16>;
    else if constexpr (std::is_same_v<TT, Table<__half>>) return (const void*)al::gate_residual_bwd_generic<__half>;
    else if constexpr (std::is_same_v<TT, Table<double>>) return (const void*)al::gate_residual_bwd_generic<double>;
    else return (const void*)al::gate_residual_bwd_generic<float>;
  });
  rc = ensure_attr(pl.fn, dev);
  if (rc) return rc;
  pl.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(sms) * 4, N)));
  *out = pl;
  return AL_OK;
}

int64_t al_gate_residual_backward_workspace_bytes(int64_t batch, int64_t seq, int64_t dim,
                                                  int64_t mod_stride, int dtype) {
  if (check_common(batch, seq, dim, mod_stride, dtype)) return -1;
  const int64_t N = batch * seq;
  if (N == 0) return 0;
  // the larger of the vector and generic plans: the pointers' alignment is not known here
  Plan pv, pg;
  int64_t grid = 0;
  if (gr_plan(N, dim, dtype, &pv) == AL_OK) grid = pv.grid;
  if (gr_generic_plan(N, dim, dtype, &pg) == AL_OK) grid = std::max<int64_t>(grid, pg.grid);
  if (grid == 0) return -1;
  const int64_t ngroups = mod_stride ? batch : 1;
  return (grid + ngroups - 1) * dim * ct_size(dtype);
}

int al_gate_residual_backward(const void* dxn, const void* gxo, const void* f, const void* gate,
                              void* dx, void* df, void* dgate, void* workspace,
                              int64_t workspace_bytes, int64_t batch, int64_t seq, int64_t dim,
                              int64_t mod_stride, int dtype, void* stream) {
  int rc = check_common(batch, seq, dim, mod_stride, dtype);
  if (rc) return rc;
  const int64_t N = batch * seq;
  const int64_t ngroups = mod_stride ? batch : 1;
  const int cs = ct_size(dtype), es = elem_size(dtype);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (N == 0) {
    if (dgate) {
      cudaError_t e = cudaMemsetAsync(dgate, 0, ngroups * dim * cs, st);
      if (e != cudaSuccess) return cuda_fail(e, "memset");
    }
    return AL_OK;
  }
  if (!dxn || !f || !gate || !dx || !df || !dgate) return fail(AL_ERR_SHAPE, "null tensor pointer");
  const void* vp[6] = {dxn, gxo ? gxo : dxn, f, gate, dx, df};
  bool vec_ok = (mod_stride * es) % 16 == 0;
  for (const void* q : vp) vec_ok = vec_ok && aligned16(q);
  Plan pl;
  const bool vplan = gr_plan(N, dim, dtype, &pl) == AL_OK;
  if (!vec_ok || !vplan) {
    // any width or alignment: the generic kernel (same arithmetic, and the vector plan's row
    // partition when there is one, so the results are bit-identical), scalar stage 2
    const int vgrid = vplan ? pl.grid : 0;
    rc = gr_generic_plan(N, dim, dtype, &pl);
    if (rc) return rc;
    if (vgrid) pl.grid = vgrid;
    const int64_t nslots = pl.grid + ngroups - 1;
    if (!workspace || workspace_bytes < nslots * dim * cs)
      return fail(AL_ERR_WORKSPACE, "workspace too small: need %lld bytes",
                  (long long)(nslots * dim * cs));
    al::GRParams p = {};
    p.dxn = dxn;
    p.gxo = gxo;
    p.f = f;
    p.gate = gate;
    p.dx = dx;
    p.df = df;
    p.ws = workspace;
    p.N = N;
    p.S_grp = mod_stride ? seq : N;
    p.D = dim;
    p.mod_stride = mod_stride;
    p.nslots = nslots;
    p.G = pl.grid;
    const int64_t cb = std::min<int64_t>(dim, kGrGenericCols);
    p.nvec = static_cast<int>(cb);  // the generic kernel's column-block width
    void* args[] = {&p};
    cudaError_t e = launch_k(pl.fn, dim3(pl.grid, static_cast<unsigned>((dim + cb - 1) / cb)),
                             dim3(pl.threads), args, pl.smem, st, kPdlBwd1);
    if (e != cudaSuccess) return cuda_fail(e, "gated-residual backward (generic) launch");
    const void* rk = reduce_kernel(dtype, false);
    void* none = nullptr;
    int64_t G64 = pl.grid, D64 = dim, N64 = N, S64 = p.S_grp, ns = nslots;
    void* rargs[] = {&workspace, &dgate, &none, &N64, &S64, &D64, &G64, &ns};
    e = launch_k(rk, dim3(static_cast<unsigned>((dim + 31) / 32), static_cast<unsigned>(ngroups)),
                 dim3(1024), rargs, 0, st, kPdlBwd2);
    if (e != cudaSuccess) return cuda_fail(e, "gated-residual backward stage-2 launch");
    return AL_OK;
  }
  const int64_t nslots = pl.grid + ngroups - 1;
  const int64_t need = nslots * dim * cs;
  if (!workspace || workspace_bytes < need)
    return fail(AL_ERR_WORKSPACE, "workspace too small: need %lld bytes", (long long)need);
  al::GRParams p = {};
  p.dxn = dxn;
  p.gxo = gxo;
  p.f = f;
  p.gate = gate;
  p.dx = dx;
  p.df = df;
  p.ws = workspace;
  p.N = N;
  p.S_grp = mod_stride ? seq : N;
  p.D = dim;
  p.mod_stride = mod_stride;
  p.nslots = nslots;
  p.nvec = static_cast<int>(dim * es / 16);
  p.G = pl.grid;
  void* args[] = {&p};
  cudaError_t e = launch_k(pl.fn, dim3(pl.grid), dim3(pl.threads), args, 0, st, kPdlBwd1);
  if (e != cudaSuccess) return cuda_fail(e, "gated-residual backward launch");
  const void* rk = reduce_kernel(dtype, true);
  void* none = nullptr;
  int64_t G64 = pl.grid, D64 = dim, N64 = N, S64 = p.S_grp, ns = nslots;
  int64_t tail0 = -1;
  unsigned long long* no_ts = nullptr;
  void* rargs[] = {&workspace, &dgate, &none, &N64, &S64, &D64, &G64, &ns, &N64, &tail0, &no_ts};
  const int64_t cols_per_cta = al::kRedCV * (16 / cs);
  if (!launch_reduce_grp(dtype, true, ngroups, tail0, dim, rargs, st, &e))
    e = launch_k(rk, dim3(static_cast<unsigned>((dim + cols_per_cta - 1) / cols_per_cta),
                          static_cast<unsigned>(ngroups)),
                 dim3(512), rargs, 0, st, kPdlBwd2);
  if (e != cudaSuccess) return cuda_fail(e, "gated-residual backward stage-2 launch");
  return AL_OK;
}

}  // extern "C"
