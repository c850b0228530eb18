// Does an SM's share of HBM bandwidth depend on where it sits?  (1) GPC membership from
// thread-block-cluster placement (a cluster never spans GPCs): many launches of 16-CTA (and
// 8-CTA) clusters, each CTA recording %smid, union-find on co-cluster SMs.  (2) The ticket
// walk of the traffic-only backward pattern (2 x 10 KB rows read, 1 written, per 2-row
// stage): how many stages the CTA on each SM completed, over several launches.  If the
// per-SM counts track the GPC size, a static partition weighted by topology would balance
// the deterministic backward like the dynamic ticket walk does.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_sm_topology_probe \
//        tools/sm_topology_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <numeric>
#include <algorithm>
#include <cmath>
#include <vector>

#include "../paper_2605_17923_b200/csrc/ptx.cuh"
using namespace al;
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned nsmid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
  return r;
}

__global__ void k_cluster(unsigned* out) {
  if (threadIdx.x == 0) {
    out[blockIdx.x] = smid();
    // hold the SM a little so clusters spread over the machine
    const unsigned long long t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < 20000) {
    }
  }
  cg::this_cluster().sync();
}

constexpr int RB = 10240, R = 2, NS = 5, NC = 320;

__global__ void __launch_bounds__(NC + 32, 1)
    k_ticket(const uint8_t* x, const uint8_t* dy, uint8_t* dx, int64_t N, unsigned* ticket,
             unsigned* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * stage_bytes);
  uint64_t* empty = full + NS;
  int64_t* hrow = reinterpret_cast<int64_t*>(empty + NS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nst = (N + R - 1) / R;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NC / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t f = 0;
      unsigned cnt = 0;
      int64_t pre = atomicAdd(ticket, 1u);
      while (true) {
        const int64_t st = pre;
        if (st < nst) pre = atomicAdd(ticket, 1u);
        const bool done = st >= nst;
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        hrow[s] = done ? -1 : st * R;
        if (done) {
          mbar_arrive(&full[s]);
          break;
        }
        ++cnt;
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
      out[2 * blockIdx.x] = smid();
      out[2 * blockIdx.x + 1] = cnt;
    }
    return;
  }
  int s = 0;
  uint32_t ph = 0;
  while (true) {
    mbar_wait(&full[s], ph);
    const int64_t row = hrow[s];
    if (row < 0) break;
    uint8_t* slot = smem + s * stage_bytes;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int off = (tid + j * NC) * 16;
        const uint4 a = ld_shared_v4(slot + rr * RB + off);
        const uint4 b = ld_shared_v4(slot + (R + rr) * RB + off);
        st_global_cs(dx + (row + rr) * RB + off,
                     make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w));
      }
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
}

// walk 0: equal contiguous ranges by blockIdx; 1: contiguous ranges bounded[slot], slot = the
// CTA's SM (claimed, linear probe on collision); 2: ticket
__global__ void __launch_bounds__(NC + 32, 1)
    k_walk(const uint8_t* x, const uint8_t* dy, uint8_t* dx, int64_t N, int walk,
           const int* bounds, unsigned* claim, unsigned* ticket, const unsigned* q) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * stage_bytes);
  uint64_t* empty = full + NS;
  int64_t* hrow = reinterpret_cast<int64_t*>(empty + NS);
  __shared__ int sslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int64_t nst = (N + R - 1) / R;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC / 32);
    }
    fence_mbar_init();
    int j = blockIdx.x;
    if (walk == 1 || walk == 3) {
      j = smid() % G;
      while (atomicCAS(claim + j, 0u, 1u) != 0u) j = (j + 1) % G;
    }
    sslot = j;
  }
  __syncthreads();
  if (warp == NC / 32 && walk == 3) {
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t f = 0;
    const int j = sslot;
    for (int64_t r = 0;; ++r) {
      int64_t S = 0, off = 0, cj = 0;
      for (int i = lane; i < G; i += 32) {
        const int64_t cp = (r * q[i]) >> 16, cc = ((r + 1) * q[i]) >> 16;
        S += cp;
        if (i < j) off += cc - cp;
        if (i == j) cj = cc - cp;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        off += __shfl_xor_sync(0xffffffffu, off, o);
        cj += __shfl_xor_sync(0xffffffffu, cj, o);
      }
      if (S >= nst) break;
      const int64_t b0 = S + off, b1 = min(b0 + cj, nst);
      for (int64_t st = b0; st < b1; ++st) {
        if (lane == 0) {
          if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
          hrow[s] = st * R;
          mbar_arrive_expect_tx(&full[s], 2 * R * RB);
          uint8_t* dst = smem + s * stage_bytes;
          for (int rr = 0; rr < R; ++rr) {
            bulk_g2s(dst + rr * RB, x + (st * R + rr) * RB, RB, &full[s], pol);
            bulk_g2s(dst + (R + rr) * RB, dy + (st * R + rr) * RB, RB, &full[s], pol);
          }
        }
        if (++s == NS) {
          s = 0;
          ++f;
        }
      }
    }
    if (lane == 0) {
      if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
      hrow[s] = -1;
      mbar_arrive(&full[s]);
    }
    return;
  }
  if (warp == NC / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t f = 0;
      const int j = sslot;
      int64_t c0, c1;
      if (walk == 1) {
        c0 = bounds[j];
        c1 = bounds[j + 1];
      } else {
        c0 = nst * j / G;
        c1 = nst * (j + 1) / G;
      }
      int64_t it = 0, pre = walk == 2 ? atomicAdd(ticket, 1u) : 0;
      while (true) {
        int64_t st;
        if (walk == 2) {
          st = pre;
          if (st < nst) pre = atomicAdd(ticket, 1u);
        } else {
          st = c0 + it;
        }
        ++it;
        const bool done = walk == 2 ? st >= nst : st >= c1;
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
  int s = 0;
  uint32_t ph = 0;
  while (true) {
    mbar_wait(&full[s], ph);
    const int64_t row = hrow[s];
    if (row < 0) break;
    uint8_t* slot = smem + s * stage_bytes;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int off = (tid + j * NC) * 16;
        const uint4 a = ld_shared_v4(slot + rr * RB + off);
        const uint4 b = ld_shared_v4(slot + (R + rr) * RB + off);
        st_global_cs(dx + (row + rr) * RB + off,
                     make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w));
      }
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
}

__global__ void k_nsm(unsigned* o) { *o = nsmid(); }

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *d, *h;
  cudaMalloc(&d, 1 << 20);
  cudaMallocHost(&h, 1 << 20);
  k_nsm<<<1, 1>>>(d);
  cudaMemcpy(h, d, 4, cudaMemcpyDeviceToHost);
  printf("{\"sms\": %d, \"nsmid\": %u}\n", sms, h[0]);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8}) {
    for (int rep = 0; rep < 40; ++rep) {
      const int nclu = 64;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nclu * cs);
      cfg.blockDim = dim3(32);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, d);
      if (e != cudaSuccess) {
        printf("{\"cluster\": %d, \"error\": \"%s\"}\n", cs, cudaGetErrorString(e));
        cudaGetLastError();
        break;
      }
      cudaMemcpy(h, d, 4 * nclu * cs, cudaMemcpyDeviceToHost);
      printf("{\"cluster\": %d, \"smids\": [", cs);
      for (int i = 0; i < nclu * cs; ++i) printf("%s%u", i ? ", " : "", h[i]);
      printf("]}\n");
    }
  }
  const int64_t N = 32760, bytes = N * RB;
  uint8_t *x, *dy, *dx;
  unsigned* tk;
  cudaMalloc(&x, bytes);
  cudaMalloc(&dy, bytes);
  cudaMalloc(&dx, bytes);
  cudaMalloc(&tk, 4 * 64);
  cudaMemset(tk, 0, 4 * 64);
  cudaMemset(x, 1, bytes);
  cudaMemset(dy, 2, bytes);
  const int smem = NS * 2 * R * RB + 3 * NS * 8;
  cudaFuncSetAttribute(k_ticket, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 24; ++rep) {
    k_ticket<<<sms, NC + 32, smem>>>(x, dy, dx, N, tk + rep, d);
    cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
    printf("{\"ticket_rep\": %d, \"smid_stages\": [", rep);
    for (int i = 0; i < sms; ++i) printf("%s[%u, %u]", i ? ", " : "", h[2 * i], h[2 * i + 1]);
    printf("]}\n");
  }
  // weights = mean stages per SM over reps 2.. (cfg2 ticket walk)
  std::vector<double> w(sms, 0.0);
  {
    // rerun to collect (the printed loop above kept only the last in h)
    for (int rep = 0; rep < 16; ++rep) {
      k_ticket<<<sms, NC + 32, smem>>>(x, dy, dx, N, tk + 24 + rep, d);
      cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
      if (rep >= 2)
        for (int i = 0; i < sms; ++i) w[h[2 * i] % sms] += h[2 * i + 1];
    }
  }
  int *dbounds;
  unsigned *claim, *tk2;
  cudaMalloc(&dbounds, 4 * (sms + 1));
  cudaMalloc(&claim, 4 * sms * 4096);
  cudaMalloc(&tk2, 4 * 4096);
  unsigned* dq;
  cudaMalloc(&dq, 4 * sms);
  cudaFuncSetAttribute(k_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double wsum = 0;
  for (double v : w) wsum += v;
  for (int64_t n : {32760LL, 65520LL, 20280LL}) {
    const int64_t nst = (n + R - 1) / R;
    std::vector<int> b(sms + 1);
    double acc = 0;
    for (int j = 0; j <= sms; ++j) {
      b[j] = (int)llround(nst * acc / wsum);
      if (j < sms) acc += w[j];
    }
    b[sms] = (int)nst;
    cudaMemcpy(dbounds, b.data(), 4 * (sms + 1), cudaMemcpyHostToDevice);
    for (int wi = 0; wi < 8; ++wi) {
      const int walk = wi < 3 ? wi : 3;
      // walk 3 variants: mean block 1/2/4 stages weighted, and 1 (equal) / 2 (equal)
      const double cbar[8] = {0, 0, 0, 1, 2, 4, 1, 2};
      const bool eq = wi >= 6;
      if (walk == 3) {
        std::vector<unsigned> qq(sms);
        const double mean = wsum / sms;
        for (int j = 0; j < sms; ++j) qq[j] = (unsigned)llround((eq ? 1.0 : w[j] / mean) * cbar[wi] * 65536.0);
        cudaMemcpy(dq, qq.data(), 4 * sms, cudaMemcpyHostToDevice);
      }
      cudaMemset(claim, 0, 4 * sms * 4096);
      cudaMemset(tk2, 0, 4 * 4096);
      int li = 0;
      std::vector<float> t;
      for (int rep = 0; rep < 23; ++rep) {
        cudaEventRecord(e0);
        k_walk<<<sms, NC + 32, smem>>>(x, dy, dx, n, walk, dbounds, claim + sms * li, tk2 + li, dq);
        cudaEventRecord(e1);
        ++li;
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 3) t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      const double med = t[t.size() / 2];
      const char* nm[8] = {"equal_contig", "smid_weighted_contig", "ticket", "weighted_rounds_c1",
                           "weighted_rounds_c2", "weighted_rounds_c4", "equal_rounds_c1",
                           "equal_rounds_c2"};
      printf("{\"N\": %lld, \"walk\": \"%s\", \"us_median\": %.2f, \"us_min\": %.2f, \"gbs\": %.1f}\n",
             (long long)n, nm[wi], med * 1e3, t[0] * 1e3, 3.0 * n * RB / (med * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
