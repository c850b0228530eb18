// Traffic-only probe of the backward's HBM pattern (2 reads : 1 write, cfg2 sizes: x, dy, dx of
// 32 760 x 5 120 bf16).  No AdaLN math: dx = x ^ dy.  Measures what each load/store mechanism
// and row walk can reach on this GPU, to split the backward's gap to the 2r1w roofline into
// "mechanism" and "compute / synchronisation".
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_bwd_traffic_probe \
//        tools/bwd_traffic_probe.cu
// Modes (one JSON line each):
//   gs        grid-stride elementwise (the torch add pattern), ld.global.nc + st.global.cs
//   ring      persistent 1 CTA/SM, 5-stage TMA ring of 2-row stages, 320 consumer threads,
//             dx via st.global.cs from registers; walk = contiguous | interleaved | ticket;
//             bar = a consumer named barrier per stage (the K2 lock step) or none
//   ringbs    as ring, but dx written back into the slot and stored with one bulk s2g copy
//   warprow   warp per row, row in registers (forward-style), grid 148 x 2 x 8 warps
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2605_17923_b200/csrc/ptx.cuh"

using namespace al;

constexpr int RB = 10240;  // row bytes (5120 bf16)
constexpr int R = 2;
constexpr int NS = 5;
constexpr int NC = 320;  // consumer threads: 2 x 16-B vectors each per row

__global__ void k_gs(const uint4* __restrict__ a, const uint4* __restrict__ b, uint4* c,
                     int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 x = __ldg(a + i), y = __ldg(b + i);
    st_global_cs(c + i, make_uint4(x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w));
  }
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}

template <bool BAR, bool BULKST>
__global__ void __launch_bounds__(NC + 32, 1)
    k_ring(const uint8_t* x, const uint8_t* dy, uint8_t* dx, int64_t N, int walk,
           unsigned int* ticket, int spin = 0) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * stage_bytes);
  uint64_t* empty = full + NS;
  int64_t* hrow = reinterpret_cast<int64_t*>(empty + NS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, k = blockIdx.x;
  const int64_t nst = (N + R - 1) / R;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BULKST ? 1 : NC / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NC / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t f = 0;
      int64_t c0 = nst * k / G, c1 = nst * (k + 1) / G, it = 0;
      int64_t pre = walk == 2 ? atomicAdd(ticket, 1u) : 0;  // one ticket ahead
      while (true) {
        int64_t st;
        if (walk == 0) st = c0 + it;  // contiguous
        else if (walk == 1) st = k + it * G;  // interleaved
        else {  // ticket
          st = pre;
          if (st < nst) pre = atomicAdd(ticket, 1u);
        }
        ++it;
        const bool done = walk == 0 ? st >= c1 : st >= nst;
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        hrow[s] = done ? -1 : st * R;
        if (done) {
          mbar_arrive(&full[s]);
          break;
        }
        mbar_arrive_expect_tx(&full[s], 2 * R * RB);
        uint8_t* dst = smem + s * stage_bytes;
        for (int rr = 0; rr < R; ++rr) {
          bulk_g2s(dst + rr * RB, x + (st * R + rr) * RB, RB, &full[s], pol);
          bulk_g2s(dst + (R + rr) * RB, dy + (st * R + rr) * RB, RB, &full[s], pol);
        }
        if (++s == NS) {
          s = 0;
          ++f;
        }
      }
    }
    return;
  }
  int s = 0, prev = -1;
  uint32_t ph = 0;
  while (true) {
    mbar_wait(&full[s], ph);
    const int64_t row = hrow[s];
    if (row < 0) break;
    uint8_t* slot = smem + s * stage_bytes;
    if (spin) {  // model the AdaLN consumer's per-stage time (slot held meanwhile)
      const long long t0 = clock64();
      while (clock64() - t0 < spin) {
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int off = (tid + j * NC) * 16;
        const uint4 a = ld_shared_v4(slot + rr * RB + off);
        const uint4 b = ld_shared_v4(slot + (R + rr) * RB + off);
        const uint4 c = make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
        if (BULKST) *reinterpret_cast<uint4*>(slot + rr * RB + off) = c;
        else st_global_cs(dx + (row + rr) * RB + off, c);
      }
    }
    if (BAR) named_bar_sync(1, NC);
    if (BULKST) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar_sync(2, NC);
      if (tid == 0) {
        bulk_s2g(dx + row * RB, slot, R * RB);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (prev >= 0) {  // release the previous slot once its store has read it
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          mbar_arrive(&empty[prev]);
        }
      }
      prev = s;
    } else if (lane == 0) {
      mbar_arrive(&empty[s]);
    }
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
  if (BULKST && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256) k_warprow(const uint4* x, const uint4* dy, uint4* dx,
                                                 int64_t N) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int VPL = RB / 16 / 32;  // 20
  for (int64_t r = w; r < N; r += nw) {
    uint4 a[VPL], b[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      a[i] = __ldg(x + r * (RB / 16) + lane + 32 * i);
      b[i] = __ldg(dy + r * (RB / 16) + lane + 32 * i);
    }
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      st_global_cs(dx + r * (RB / 16) + lane + 32 * i,
                   make_uint4(a[i].x ^ b[i].x, a[i].y ^ b[i].y, a[i].z ^ b[i].z,
                              a[i].w ^ b[i].w));
  }
}

#define CK(e)                                                           \
  do {                                                                  \
    cudaError_t _e = (e);                                               \
    if (_e != cudaSuccess) {                                            \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 32760;
  const int64_t bytes = N * RB;
  uint8_t *x, *dy, *dx;
  unsigned int* ticket;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&dy, bytes));
  CK(cudaMalloc(&dx, bytes));
  CK(cudaMalloc(&ticket, 4 * 4096));
  int li = 0;
  CK(cudaMemset(x, 1, bytes));
  CK(cudaMemset(dy, 2, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem = NS * 2 * R * RB + 2 * NS * 8 + NS * 8;
  CK(cudaFuncSetAttribute(k_ring<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_ring<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_ring<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto launch) -> int {
    li = 0;
    cudaMemset(ticket, 0, 4 * 4096);
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> t;
    for (int rep = 0; rep < 15; ++rep) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(t.begin(), t.end());
    const double med = t[t.size() / 2];
    printf("{\"mode\": \"%s\", \"N\": %lld, \"us_median\": %.2f, \"us_min\": %.2f, \"gbs\": %.1f}\n",
           name, (long long)N, med * 1e3, t[0] * 1e3, 3.0 * bytes / (med * 1e-3) / 1e9);
    fflush(stdout);
    return 0;
  };
  const int64_t nv = bytes / 16;
  for (int mult : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "gs_grid%dx", mult);
    if (run(nm, [&] {
          k_gs<<<sms * mult, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, nv);
        }))
      return 1;
  }
  const char* walks[3] = {"contig", "interleaved", "ticket"};
  for (int walk = 0; walk < 3; ++walk) {
    char nm[64];
    snprintf(nm, sizeof nm, "ring_%s", walks[walk]);
    if (run(nm, [&] {
          k_ring<false, false><<<sms, NC + 32, smem>>>(x, dy, dx, N, walk, ticket + li++);
        }))
      return 1;
    snprintf(nm, sizeof nm, "ring_bar_%s", walks[walk]);
    if (run(nm, [&] {
          k_ring<true, false><<<sms, NC + 32, smem>>>(x, dy, dx, N, walk, ticket + li++);
        }))
      return 1;
    snprintf(nm, sizeof nm, "ringbs_%s", walks[walk]);
    if (run(nm, [&] {
          k_ring<false, true><<<sms, NC + 32, smem>>>(x, dy, dx, N, walk, ticket + li++);
        }))
      return 1;
  }
  for (int spin : {250, 500, 1000, 1500, 2000, 2500, 3000}) {
    char nm[64];
    snprintf(nm, sizeof nm, "ring_bar_ticket_spin%d", spin);
    if (run(nm, [&] {
          k_ring<true, false><<<sms, NC + 32, smem>>>(x, dy, dx, N, 2, ticket + li++, spin);
        }))
      return 1;
  }
  for (int mult : {1, 2}) {
    char nm[64];
    snprintf(nm, sizeof nm, "warprow_grid%dx", mult);
    if (run(nm, [&] {
          k_warprow<<<sms * mult, 256>>>((const uint4*)x, (const uint4*)dy, (uint4*)dx, N);
        }))
      return 1;
  }
  return 0;
}
