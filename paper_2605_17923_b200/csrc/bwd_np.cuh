// bwd_np.cuh -- EXPERIMENT (A/B via AL_BWD_NP): backward stage 1 without a producer warp.
// Consumer thread 0 refills the ring slot right after each stage barrier (where K2's producer
// would have been released), so all warps are consumers: <V = 2, 12 warps> puts 5 vectors per
// lane on every SM sub-partition (warps s, s+4, s+8 own 2, 2, 1 vectors) with 3 warps each;
// <V = 3, 8 warps> (K2b, round-2 commit 5bfe834) does the same with 2 warps each.  Same
// arithmetic and slot contract as K2's lean dynamic stage body; single group; 16-bit rows.
#pragma once

namespace al {

template <typename T, int V, int NCW>
__global__ void __launch_bounds__(NCW * 32, 1) adaln_bwd_np(const BwdParams p) {
  pdl_enter();
  ts_begin(p.ts);
  if (threadIdx.x == 0) AL_TRACE(1, 0);
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int EPV = Traits<T>::EPV;
  constexpr int NP = EPV / 2;
  constexpr int R = 2, NC = NCW * 32;
  extern __shared__ __align__(128) uint8_t smem[];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = p.nstages;
  const int RB = p.row_bytes;
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * stage_bytes);
  CT* red = reinterpret_cast<CT*>(full + NS);  // [2][NCW][R * 2]
  int64_t* h_row = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(red + 2 * NCW * R * 2) + 7) & ~uintptr_t(7));
  int* h_n = reinterpret_cast<int*>(h_row + NS);

  const int64_t k = blockIdx.x;
  const bool dyn = p.sched != nullptr;
  const int64_t nst = (p.N + R - 1) / R;
  const uint8_t* xb = static_cast<const uint8_t*>(p.x);
  const uint8_t* db = static_cast<const uint8_t*>(p.dy);

  // ---- ring refill state: thread 0 only
  uint64_t pol = 0;
  int64_t walk_next = k;  // interleaved walk: next stage index
  int64_t tk0 = 0, tk1 = 0;  // dynamic walk: tickets drawn two refills ahead
  bool ended = false;
  // issue the next stage of the walk into slot s (or the end marker once the walk is done)
  auto refill = [&](int s) {
    if (ended) return;
    int64_t st;
    if (dyn) {
      st = tk0;
      tk0 = tk1;
      if (st < nst) tk1 = static_cast<int64_t>(atomicAdd(p.sched, 1u));
    } else {
      st = walk_next;
      walk_next += p.G;
    }
    if (st >= nst) {  // end marker: completes the slot's phase without data
      h_n[s] = 0;
      ended = true;
      mbar_arrive(&full[s]);
      return;
    }
    const int64_t start = st * R;
    const int rows = p.N - start < R ? static_cast<int>(p.N - start) : R;
    h_row[s] = start;
    h_n[s] = rows;
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(2 * rows * RB));
    uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
    for (int rr = 0; rr < rows; ++rr) {
      bulk_g2s(dst + rr * RB, xb + (start + rr) * RB, RB, &full[s], pol);
      bulk_g2s(dst + (R + rr) * RB, db + (start + rr) * RB, RB, &full[s], pol);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    pol = policy_evict_first();
    if (dyn) {
      tk0 = static_cast<int64_t>(atomicAdd(p.sched, 1u));
      tk1 = static_cast<int64_t>(atomicAdd(p.sched, 1u));
    }
    for (int s = 0; s < NS; ++s) refill(s);
  }
  __syncthreads();  // barriers initialised, first NS headers visible

  uint32_t vmask = 0;
  int coff[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    coff[j] = (tid + j * NC) * 16;
    if (tid + j * NC < p.nvec) vmask |= 1u << j;
  }
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT* mean_p = static_cast<const CT*>(p.mean);
  const CT* rstd_p = static_cast<const CT*>(p.rstd);
  CT* ws_sc = static_cast<CT*>(p.ws);
  CT* ws_sh = ws_sc + p.nslots * p.D;
  bool nf = false;

  P s1[V][NP], acc_sc[V][NP], acc_sh[V][NP];
  {
    const uint8_t* sc = static_cast<const uint8_t*>(p.scale);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (vmask >> j & 1) {
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sc + coff[j])), s1[j]);
#pragma unroll
        for (int e = 0; e < NP; ++e) s1[j][e] = add2(s1[j][e], splat2(CT(1)));
      } else {
#pragma unroll
        for (int e = 0; e < NP; ++e) s1[j][e] = splat2(CT(0));
      }
#pragma unroll
      for (int e = 0; e < NP; ++e) acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));
    }
  }

  // statistics of a stage's rows (zeros past its rows)
  auto fetch = [&](int s, CT* m, CT* r) {
    const int64_t rb = h_row[s];
    const int n = h_n[s];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      m[rr] = rr < n ? mean_p[rb + rr] : CT(0);
      r[rr] = rr < n ? rstd_p[rb + rr] : CT(0);
    }
  };

  int s = 0, it = 0;
  uint32_t ph = 0;
  CT mc[R], rc[R];
  fetch(0, mc, rc);
  while (true) {
    mbar_wait(&full[s], ph);
    const int64_t rb = h_row[s];
    const int rows = h_n[s];
    if (rows == 0) break;
    // next stage's statistics, one stage ahead (its header was written at least one stage
    // barrier ago, or in the prologue)
    const int s_next = s + 1 == NS ? 0 : s + 1;
    CT mn[R], rn[R];
    fetch(s_next, mn, rn);

    const uint32_t stx_u = smem_addr(smem) + static_cast<uint32_t>(s * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    CT* rd = red + (it & 1) * (NCW * R * 2);

    // phase 1: row sums of g and g*xhat; column accumulators of dy and dy*xhat
    P xh[R][V][NP], gg[R][V][NP];
    CT rowsum[R * 2];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const bool live = rr < rows;
      const P r2 = splat2(rc[rr]);
      const P nmr = splat2(-mc[rr] * rc[rr]);
      P sg[2] = {splat2(CT(0)), splat2(CT(0))}, sgx[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = live && (vmask >> j & 1);
        P xv[NP], dv[NP];
        const uint32_t o = static_cast<uint32_t>(rr * RB + coff[j]);
        unpack2<T>(ok ? ld_shared_v4_u32(stx_u + o) : make_uint4(0, 0, 0, 0), xv);
        unpack2<T>(ok ? ld_shared_v4_u32(std_u + o) : make_uint4(0, 0, 0, 0), dv);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          xh[rr][j][e] = fma2(xv[e], r2, nmr);
          gg[rr][j][e] = mul2(dv[e], s1[j][e]);
          sg[e & 1] = add2(sg[e & 1], gg[rr][j][e]);
          sgx[e & 1] = fma2(gg[rr][j][e], xh[rr][j][e], sgx[e & 1]);
          acc_sh[j][e] = add2(acc_sh[j][e], dv[e]);
          acc_sc[j][e] = fma2(dv[e], xh[rr][j][e], acc_sc[j][e]);
        }
      }
      const P tsg = add2(sg[0], sg[1]), tsgx = add2(sgx[0], sgx[1]);
      rowsum[2 * rr] = tsg.x + tsg.y;
      rowsum[2 * rr + 1] = tsgx.x + tsgx.y;
    }
    {
      constexpr int NV = 2 * R, GRP = 32 / NV;
      const CT u = warp_reduce_scatter<NV>(rowsum, lane);
      if ((lane & (GRP - 1)) == 0) rd[warp * NV + lane / GRP] = u;
    }
    named_bar_sync(1, NC);
    // every consumer has this stage in registers: refill its slot with the walk's next stage
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      refill(s);
    }

    CT tot[2 * R];
    {
      constexpr int NV = 2 * R;
      CT s_l = CT(0);
      for (int i = lane; i < NCW * NV; i += 32) s_l += rd[i];
#pragma unroll
      for (int off = NV; off < 32; off <<= 1) s_l += __shfl_xor_sync(0xffffffffu, s_l, off);
#pragma unroll
      for (int q = 0; q < NV; ++q) tot[q] = __shfl_sync(0xffffffffu, s_l, q);
    }

    // phase 2: dx = rstd * (g - mean(g) - xhat * mean(g*xhat))
    uint8_t* dxrow = static_cast<uint8_t*>(p.dx) + rb * RB;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr < rows) {
        const CT rr_ = rc[rr];
        const P c0 = splat2(-rr_ * tot[2 * rr] * invD), c1 = splat2(-rr_ * tot[2 * rr + 1] * invD);
        const P r2 = splat2(rr_);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            P o[NP];
#pragma unroll
            for (int e = 0; e < NP; ++e)
              o[e] = fma2(gg[rr][j][e], r2, fma2(xh[rr][j][e], c1, c0));
            st_global_cs(dxrow + rr * RB + coff[j], pack2<T>(o));
          }
        }
        if (tid == 0) nf |= !(finite_ct(tot[2 * rr]) && finite_ct(tot[2 * rr + 1]));
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mc[rr] = mn[rr];
      rc[rr] = rn[rr];
    }
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    ++it;
  }

  // this CTA's partials (zeros if it drew no stage)
  {
    const int64_t slot = dyn ? p.tail_slot0 + k : k;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (vmask >> j & 1) {
        const int64_t col = static_cast<int64_t>(coff[j] / 16) * EPV;
        P* a = reinterpret_cast<P*>(ws_sc + slot * p.D + col);
        P* b = reinterpret_cast<P*>(ws_sh + slot * p.D + col);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          a[e] = acc_sc[j][e];
          b[e] = acc_sh[j][e];
        }
      }
    }
  }
  if (tid == 0) AL_TRACE_INFO(it);
#ifdef AL_CTA_TRACE
  named_bar_sync(1, NC);
  if (tid == 0) AL_TRACE(1, 1);
#endif
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
  if (dyn) {
    // the last CTA out re-arms the ticket pair
    named_bar_sync(1, NC);
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1u) == static_cast<unsigned int>(p.G - 1)) {
        atomicExch(p.sched, 0u);
        atomicExch(p.sched + 1, 0u);
      }
    }
  }
}

}  // namespace al
