// block_kernels.cuh -- the DiT-block ops adjacent to AdaLN.
//
// 1. Fused Q/K RMSNorm of a packed QKV projection ("Q-Norm + K-Norm", the op that sits between
//    the qkv GEMM and attention in a Wan-2.1 block):
//
//   q_n = q * rsqrt(mean(q^2) + eps) * w_q,   k_n = k * rsqrt(mean(k^2) + eps) * w_k
//
// over the full model width D (Wan's WanRMSNorm(dim) on q and k), reading q and k straight out
// of the [N, 3D] projection output (row stride 3D) and, optionally, copying v out contiguously,
// so the block needs no split/contiguous copies.  Backward writes the whole d(qkv) row
// (dq | dk | dv) and reduces dw_q, dw_k over the rows in two deterministic stages (per-CTA
// partials here, the cross-CTA sum by adaln_bwd_reduce_vec).
//
// Same skeleton as the AdaLN rows kernels: one warp per row, the row's slices held in registers
// (VPL 16-byte vectors per lane), statistics by warp shuffles only, weights staged in shared
// memory as fp32 pairs, packed fp32 pair math.  HBM-bound: forward moves 2 N D e in + 2 N D e out
// (+ v copy), backward 4 N D e in + 2 N D e out (+ v).
#pragma once

#include "adaln_kernels.cuh"

namespace al {

struct QKParams {
  const void* qkv;     // [N, row_stride] elements: q at [0, D), k at [D, 2D), v at [2D, 3D)
  int64_t row_stride;  // elements between rows of qkv / dqkv
  const void* wq;      // [D]
  const void* wk;      // [D]
  void* qn;            // [N, D] forward outputs
  void* kn;
  void* vc;            // [N, D] contiguous copy of v (nullable)
  const void* dqn;     // [N, D] backward inputs
  const void* dkn;
  const void* dv;      // [N, D] gradient of vc (nullable: dv slice of dqkv left untouched)
  void* dqkv;          // [N, row_stride] backward output
  void* rstd;          // [N, 2] compute type
  void* ws;            // [2][G][D] compute type: per-CTA dw_q | dw_k partials
  int64_t N;
  int64_t D;
  int nvec;  // D / EPV
  int G;
  double eps;
  int* nonfinite;
};

template <typename T, int VPL>
__global__ void __launch_bounds__(256) qk_rms_fwd(const QKParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int NP = Traits<T>::EPV / 2;
  extern __shared__ __align__(16) uint8_t smem[];
  P* wq = reinterpret_cast<P*>(smem);  // [nvec * NP]
  P* wk = wq + p.nvec * NP;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT eps = static_cast<CT>(p.eps);
  const int64_t RS = p.row_stride * static_cast<int64_t>(sizeof(T));  // bytes between rows
  const int64_t DB = p.D * static_cast<int64_t>(sizeof(T));
  bool nf = false;

  for (int c = tid; c < p.nvec; c += blockDim.x) {
    P a[NP], b[NP];
    unpack2<T>(__ldg(reinterpret_cast<const uint4*>(p.wq) + c), a);
    unpack2<T>(__ldg(reinterpret_cast<const uint4*>(p.wk) + c), b);
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      wq[c * NP + e] = a[e];
      wk[c * NP + e] = b[e];
    }
  }
  __syncthreads();

  for (int64_t row = r0 + warp; row < r1; row += nwarp) {
    const uint8_t* base = static_cast<const uint8_t*>(p.qkv) + row * RS;
    uint4 vq[VPL], vk[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      vq[i] = c < p.nvec ? ld_global_nc_v4(base + c * 16) : make_uint4(0, 0, 0, 0);
      vk[i] = c < p.nvec ? ld_global_nc_v4(base + DB + c * 16) : make_uint4(0, 0, 0, 0);
    }
    CT part[2];
    {
      P aq[2] = {splat2(CT(0)), splat2(CT(0))}, ak[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        P a[NP], b[NP];
        unpack2<T>(vq[i], a);
        unpack2<T>(vk[i], b);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          aq[e & 1] = fma2(a[e], a[e], aq[e & 1]);
          ak[e & 1] = fma2(b[e], b[e], ak[e & 1]);
        }
      }
      const P tq = add2(aq[0], aq[1]), tk = add2(ak[0], ak[1]);
      part[0] = tq.x + tq.y;
      part[1] = tk.x + tk.y;
    }
    const CT u = warp_reduce_scatter<2>(part, lane);
    const CT ssq = __shfl_sync(0xffffffffu, u, 0), ssk = __shfl_sync(0xffffffffu, u, 16);
    const CT rq = CT(1) / sqrt(ssq * invD + eps), rk = CT(1) / sqrt(ssk * invD + eps);
    const P rq2 = splat2(rq), rk2 = splat2(rk);
    uint8_t* oq = static_cast<uint8_t*>(p.qn) + row * DB;
    uint8_t* ok = static_cast<uint8_t*>(p.kn) + row * DB;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < p.nvec) {
        P a[NP], b[NP];
        unpack2<T>(vq[i], a);
        unpack2<T>(vk[i], b);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          a[e] = mul2(mul2(a[e], rq2), wq[c * NP + e]);
          b[e] = mul2(mul2(b[e], rk2), wk[c * NP + e]);
        }
        st_global_cs(oq + c * 16, pack2<T>(a));
        st_global_cs(ok + c * 16, pack2<T>(b));
      }
    }
    if (p.vc != nullptr) {  // contiguous v for attention: a straight 16-byte copy
      uint8_t* ov = static_cast<uint8_t*>(p.vc) + row * DB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < p.nvec) st_global_cs(ov + c * 16, ld_global_nc_v4(base + 2 * DB + c * 16));
      }
    }
    if (lane == 0) {
      static_cast<CT*>(p.rstd)[2 * row] = rq;
      static_cast<CT*>(p.rstd)[2 * row + 1] = rk;
      nf |= !(finite_ct(ssq) && finite_ct(ssk));
    }
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// Backward.  Per row, for x in {q, k} with r = rstd, xh = x r, g = dy w:
//   dx = r (g - xh * sum(g xh) / D),     dw += dy xh  (column sums over the rows)
// Column partials accumulate per warp in shared memory (planar layout, conflict-free 16-byte
// accesses), are summed over the CTA's warps in a fixed order at the end and written as the
// CTA's slot of the [2][G][D] workspace.
template <typename T, int VPL>
__global__ void __launch_bounds__(256) qk_rms_bwd(const QKParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int NP = Traits<T>::EPV / 2;
  constexpr int HP = 16 / static_cast<int>(sizeof(P));  // pairs per 16-byte chunk
  extern __shared__ __align__(16) uint8_t smem[];
  const int nvec = p.nvec;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  P* wq = reinterpret_cast<P*>(smem);  // [nvec * NP]
  P* wk = wq + nvec * NP;
  P* acc = wk + nvec * NP;  // [nwarp][2 (q, k)][nvec * NP], planar by 16-byte chunk
  auto ai = [nvec](int w, int which, int c, int e) {
    return ((w * 2 + which) * (NP / HP) + e / HP) * nvec * HP + c * HP + (e % HP);
  };

  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const int64_t RS = p.row_stride * static_cast<int64_t>(sizeof(T));
  const int64_t DB = p.D * static_cast<int64_t>(sizeof(T));
  bool nf = false;

  for (int c = tid; c < nvec; c += blockDim.x) {
    P a[NP], b[NP];
    unpack2<T>(__ldg(reinterpret_cast<const uint4*>(p.wq) + c), a);
    unpack2<T>(__ldg(reinterpret_cast<const uint4*>(p.wk) + c), b);
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      wq[c * NP + e] = a[e];
      wk[c * NP + e] = b[e];
    }
  }
  for (int i = tid; i < nwarp * 2 * nvec * NP; i += blockDim.x) acc[i] = splat2(CT(0));
  __syncthreads();

  for (int64_t row = r0 + warp; row < r1; row += nwarp) {
    const uint8_t* base = static_cast<const uint8_t*>(p.qkv) + row * RS;
    const uint8_t* gq = static_cast<const uint8_t*>(p.dqn) + row * DB;
    const uint8_t* gk = static_cast<const uint8_t*>(p.dkn) + row * DB;
    uint4 xq[VPL], xk[VPL], dq[VPL], dk[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      const bool ok = c < nvec;
      xq[i] = ok ? ld_global_nc_v4(base + c * 16) : make_uint4(0, 0, 0, 0);
      xk[i] = ok ? ld_global_nc_v4(base + DB + c * 16) : make_uint4(0, 0, 0, 0);
      dq[i] = ok ? ld_global_nc_v4(gq + c * 16) : make_uint4(0, 0, 0, 0);
      dk[i] = ok ? ld_global_nc_v4(gk + c * 16) : make_uint4(0, 0, 0, 0);
    }
    const CT rq = static_cast<const CT*>(p.rstd)[2 * row];
    const CT rk = static_cast<const CT*>(p.rstd)[2 * row + 1];
    const P rq2 = splat2(rq), rk2 = splat2(rk);
    // sum(g xh) for q and k; column partials dy * xh
    CT part[2];
    {
      P sq[2] = {splat2(CT(0)), splat2(CT(0))}, sk[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < nvec) {
          P a[NP], b[NP], ga[NP], gb[NP];
          unpack2<T>(xq[i], a);
          unpack2<T>(xk[i], b);
          unpack2<T>(dq[i], ga);
          unpack2<T>(dk[i], gb);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            const P xhq = mul2(a[e], rq2), xhk = mul2(b[e], rk2);
            sq[e & 1] = fma2(mul2(ga[e], wq[c * NP + e]), xhq, sq[e & 1]);
            sk[e & 1] = fma2(mul2(gb[e], wk[c * NP + e]), xhk, sk[e & 1]);
            P& aq = acc[ai(warp, 0, c, e)];
            P& ak = acc[ai(warp, 1, c, e)];
            aq = fma2(ga[e], xhq, aq);
            ak = fma2(gb[e], xhk, ak);
          }
        }
      }
      const P tq = add2(sq[0], sq[1]), tk = add2(sk[0], sk[1]);
      part[0] = tq.x + tq.y;
      part[1] = tk.x + tk.y;
    }
    const CT u = warp_reduce_scatter<2>(part, lane);
    const CT mq = __shfl_sync(0xffffffffu, u, 0) * invD, mk = __shfl_sync(0xffffffffu, u, 16) * invD;
    const P nmq = splat2(-mq), nmk = splat2(-mk);
    uint8_t* out = static_cast<uint8_t*>(p.dqkv) + row * RS;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < nvec) {
        P a[NP], b[NP], ga[NP], gb[NP];
        unpack2<T>(xq[i], a);
        unpack2<T>(xk[i], b);
        unpack2<T>(dq[i], ga);
        unpack2<T>(dk[i], gb);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          // dx = r * (g - xh * m) = r * g - (r * m) * (x * r)
          a[e] = mul2(fma2(mul2(a[e], rq2), nmq, mul2(ga[e], wq[c * NP + e])), rq2);
          b[e] = mul2(fma2(mul2(b[e], rk2), nmk, mul2(gb[e], wk[c * NP + e])), rk2);
        }
        st_global_cs(out + c * 16, pack2<T>(a));
        st_global_cs(out + DB + c * 16, pack2<T>(b));
      }
    }
    if (p.dv != nullptr) {
      const uint8_t* gv = static_cast<const uint8_t*>(p.dv) + row * DB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < nvec) st_global_cs(out + 2 * DB + c * 16, ld_global_nc_v4(gv + c * 16));
      }
    }
    if (lane == 0) nf |= !(finite_ct(mq) && finite_ct(mk));
  }
  __syncthreads();
  // this CTA's dw partials: warps summed in ascending order
  CT* ws = static_cast<CT*>(p.ws);
  for (int idx = tid; idx < 2 * nvec * NP; idx += blockDim.x) {
    const int which = idx / (nvec * NP), rem = idx % (nvec * NP), c = rem / NP, e = rem % NP;
    P s = acc[ai(0, which, c, e)];
    for (int w = 1; w < nwarp; ++w) s = add2(s, acc[ai(w, which, c, e)]);
    P* dst = reinterpret_cast<P*>(ws + (static_cast<int64_t>(which) * p.G + k) * p.D) + c * NP + e;
    *dst = s;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// =====================================================================================
// 2. Backward of the gated residual x_out = x + gate (.) f (the forward is fused into the AdaLN
//    rows kernel, adaln_fwd_rows<RESID>).  With G = dxn + g_xo (dxn: the AdaLN backward's dx at
//    x_out, g_xo: the gradient reaching x_out from elsewhere):
//      dx = G,   df = gate (.) G,   dgate[g, :] = sum over the rows of sample g of f (.) G
//    Purely elementwise plus a column reduction, so the CTA is laid out like the AdaLN
//    backward's consumers: thread t owns 16-byte column vectors t + j*nc (j < V) of every row of
//    the CTA's contiguous row range, the gate of those columns and the dgate partials live in
//    registers, two rows' loads are in flight per thread, and at each sample boundary the
//    partials go to the CTA's (slot = CTA + sample) row of a [nslots][D] workspace reduced by
//    the AdaLN stage-2 kernel -- deterministic.  Reads dxn, g_xo, f; writes dx, df: 5 N D e.
// =====================================================================================
struct GRParams {
  const void* dxn;
  const void* gxo;  // nullable (zero)
  const void* f;
  const void* gate;
  void* dx;
  void* df;
  void* ws;  // [nslots][D] compute type
  int64_t N, S_grp, D, mod_stride, nslots;
  int nvec;
  int G;
};

template <typename T, int V>
__global__ void __launch_bounds__(512) gate_residual_bwd(const GRParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int NP = Traits<T>::EPV / 2;
  constexpr int RU = 2;  // rows in flight per thread
  const int nc = blockDim.x, tid = threadIdx.x;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const int64_t RB = p.D * static_cast<int64_t>(sizeof(T));
  CT* ws = static_cast<CT*>(p.ws);
  bool own[V];
#pragma unroll
  for (int j = 0; j < V; ++j) own[j] = tid + j * nc < p.nvec;

  int64_t row0 = r0;
  while (row0 < r1) {
    const int64_t g = row0 / p.S_grp;
    const int64_t seg_end = min(r1, (g + 1) * p.S_grp);
    P gt[V][NP], acc[V][NP];
    {
      const uint4* ga = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.gate) +
                                                       g * p.mod_stride * sizeof(T));
#pragma unroll
      for (int j = 0; j < V; ++j) {
        unpack2<T>(own[j] ? __ldg(ga + tid + j * nc) : make_uint4(0, 0, 0, 0), gt[j]);
#pragma unroll
        for (int e = 0; e < NP; ++e) acc[j][e] = splat2(CT(0));
      }
    }
    for (int64_t row = row0; row < seg_end; row += RU) {
      uint4 vd[RU][V], vg[RU][V], vf[RU][V];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const bool live = row + u < seg_end;
        const int64_t ro = (row + u) * RB;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const bool ok = live && own[j];
          const int64_t off = ro + static_cast<int64_t>(tid + j * nc) * 16;
          vd[u][j] = ok ? ld_global_nc_v4(static_cast<const uint8_t*>(p.dxn) + off) : make_uint4(0, 0, 0, 0);
          vg[u][j] = (ok && p.gxo) ? ld_global_nc_v4(static_cast<const uint8_t*>(p.gxo) + off)
                                   : make_uint4(0, 0, 0, 0);
          vf[u][j] = ok ? ld_global_nc_v4(static_cast<const uint8_t*>(p.f) + off) : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (row + u < seg_end) {
          const int64_t ro = (row + u) * RB;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if (own[j]) {
              P a[NP], b[NP], fv[NP];
              unpack2<T>(vd[u][j], a);
              unpack2<T>(vg[u][j], b);
              unpack2<T>(vf[u][j], fv);
#pragma unroll
              for (int e = 0; e < NP; ++e) a[e] = add2(a[e], b[e]);  // G in fp32
              const uint4 Gp = pack2<T>(a);                         // dx, rounded to T
              unpack2<T>(Gp, a);  // the stored G drives df and dgate, as a composed backward
#pragma unroll
              for (int e = 0; e < NP; ++e) {
                b[e] = mul2(gt[j][e], a[e]);
                acc[j][e] = fma2(fv[e], a[e], acc[j][e]);
              }
              const int64_t off = ro + static_cast<int64_t>(tid + j * nc) * 16;
              st_global_cs(static_cast<uint8_t*>(p.dx) + off, Gp);
              st_global_cs(static_cast<uint8_t*>(p.df) + off, pack2<T>(b));
            }
          }
        }
      }
    }
    // this CTA's dgate partial for sample g (each thread owns distinct columns)
#pragma unroll
    for (int j = 0; j < V; ++j)
      if (own[j]) {
        P* dst = reinterpret_cast<P*>(ws + (k + g) * p.D) + static_cast<int64_t>(tid + j * nc) * NP;
#pragma unroll
        for (int e = 0; e < NP; ++e) dst[e] = acc[j][e];
      }
    row0 = seg_end;
  }
}

// Any width / alignment (the vector kernel needs 16-byte rows and pointers): the same
// arithmetic per element -- G = dxn + g_xo in the compute type, rounded to T; df = gate * G;
// dgate partial += f * G (fma), rows in order -- with thread t owning columns t, t + blockDim,
// ... and the partials in shared memory ([D] compute type), flushed per (CTA, sample) slot for
// the scalar stage-2 kernel.  Bit-identical to the vector kernel on shapes both take.
template <typename T>
__global__ void __launch_bounds__(256) gate_residual_bwd_generic(const GRParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  extern __shared__ __align__(16) uint8_t smem[];
  CT* acc = reinterpret_cast<CT*>(smem);
  // blockIdx.y: a block of p.nvec columns (wide rows are split so the partials fit in shared
  // memory); threads own columns c0 + tid, c0 + tid + blockDim, ...
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * p.nvec;
  const int64_t c1 = c0 + p.nvec < p.D ? c0 + p.nvec : p.D;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const T* dxn = static_cast<const T*>(p.dxn);
  const T* gxo = static_cast<const T*>(p.gxo);
  const T* f = static_cast<const T*>(p.f);
  T* dx = static_cast<T*>(p.dx);
  T* df = static_cast<T*>(p.df);
  CT* ws = static_cast<CT*>(p.ws);
  int64_t row0 = r0;
  while (row0 < r1) {
    const int64_t g = row0 / p.S_grp;
    const int64_t seg_end = min(r1, (g + 1) * p.S_grp);
    const T* gate = static_cast<const T*>(p.gate) + g * p.mod_stride;
    for (int64_t d = c0 + tid; d < c1; d += nt) acc[d - c0] = CT(0);
    for (int64_t row = row0; row < seg_end; ++row) {
      const int64_t o = row * p.D;
      for (int64_t d = c0 + tid; d < c1; d += nt) {
        CT G = to_ct(dxn[o + d]);
        if (gxo) G = G + to_ct(gxo[o + d]);
        const T Gt = from_ct<T>(G);
        const CT Gr = to_ct(Gt);
        dx[o + d] = Gt;
        df[o + d] = from_ct<T>(to_ct(gate[d]) * Gr);
        acc[d - c0] = fma(to_ct(f[o + d]), Gr, acc[d - c0]);
      }
    }
    for (int64_t d = c0 + tid; d < c1; d += nt) ws[(k + g) * p.D + d] = acc[d - c0];
    row0 = seg_end;
  }
}

}  // namespace al
