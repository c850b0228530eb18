// adaln_kernels.cuh -- sm_100a kernels of the fused LayerNorm-Modulate (AdaLN) operator.
//
// Reference arithmetic (f64 CPU oracle, /root/reference/pkg/src/adaptiveload/adaln/):
//   forward   _kernels_numba.py:18-34   mu = sum(x)/D; var = sum((x-mu)^2)/D;
//                                       rstd = 1/sqrt(var+eps); y = (x-mu)*rstd*(1+scale)+shift
//   dx        _kernels_numba.py:45-62   g = dy*(1+scale); dx = rstd*(g - mean(g) - xhat*mean(g*xhat))
//   dscale/dshift _kernels_numba.py:71-83 (naive) / :94-127 (d-tile): column sums over the
//                                       sequence of dy*xhat and dy.
//
// Design (bandwidth-bound; tensor cores deliberately unused):
//  * Persistent-style static row partition: CTA k owns rows [k*N/G, (k+1)*N/G).  Rows are
//    streamed through an NS-stage shared-memory ring by 1-D TMA bulk copies (cp.async.bulk)
//    issued by one producer lane; mbarrier full/empty pairs decouple copy and compute, so
//    HBM reads stay in flight while consumers reduce and write.
//  * Consumer thread t owns 16-byte column vectors t + i*nc (i < V): the paper's
//    "thread fixed to feature d" D-tile mapping.  Shared-memory reads are
//    conflict-free 128-bit loads, global writes are coalesced 128-bit streaming stores, and the
//    per-column (1+scale), shift and dscale/dshift accumulators live in registers.
//  * Forward statistics: exact per-thread two-pass (mean, M2) over the owned elements, merged
//    across lanes and warps with the parallel-variance identity
//        M2 = sum_i [M2_i + n_i (m_i - m)^2],  m = sum_i n_i m_i / n,
//    i.e. Welford/Chan merging: one reduction round per stage, no E[x^2]-E[x]^2 cancellation.
//  * Backward: stage 1 (this kernel) writes per-CTA fp32 column partials of dy*xhat and dy;
//    stage 2 (adaln_bwd_reduce) sums them over CTAs in ascending CTA order in fp64.
//    Deterministic: no floating-point atomics anywhere.
//  * A stage never straddles a modulation/reduction group (sample), so scale/shift and the
//    partial accumulators are constant within a stage.
#pragma once
#include <cstdint>
#include <type_traits>

#include "dtype.cuh"
#include "ptx.cuh"

namespace al {

struct FwdParams {
  const void* x;
  const void* scale;
  const void* shift;
  void* y;
  void* mean;
  void* rstd;
  int64_t N;           // rows (batch * seq)
  int64_t S_grp;       // rows per modulation group (seq, or N when scale/shift broadcast)
  int64_t D;           // features
  int64_t mod_stride;  // elements between consecutive groups' scale/shift rows
  double eps;
  int* nonfinite;
  int nvec;       // D / EPV
  int row_bytes;  // D * sizeof(T)
  int nstages;    // ring depth
  int G;          // CTAs
  // gated-residual fusion (adaln_fwd_rows<..., RESID>): x_out = x + gate * f, y = AdaLN(x_out)
  const void* f;
  const void* gate;
  void* x_out;
  // dynamic tail (adaln_fwd_rows16): rows [N_static, N) are handed out by the ticket counter
  // sched[0]; sched[1] counts finished CTAs (the last one re-arms both).  nullptr = static only
  // (N_static == N).
  unsigned int* sched;
  int64_t N_static;
  unsigned long long* ts;  // nullable: per-launch device timestamps (ptx.cuh ts_begin/ts_end)
  // 1: the dynamic tail spans several modulation groups (multi-sample launches); rows of a group
  // other than the CTA's staged one read (1 + scale, shift) straight from global memory
  int dyn_groups;
};

// Ticket-counter slots for dynamically scheduled launches: one per (device, stream) for eager
// launches and one per captured launch (adaln_capi.cu sched_slot); the last CTA of each launch
// resets its slot to zero.
constexpr int kSchedSlots = 16384;
__device__ unsigned int g_sched[kSchedSlots][2];

struct StealSlot;  // bwd_steal.cuh

struct BwdParams {
  const void* dy;
  const void* x;
  const void* scale;
  const void* mean;
  const void* rstd;
  void* dx;
  void* ws;  // [2][nslots][D] partials (dscale | dshift), compute type
  int64_t N;
  int64_t S_grp;  // rows per reduction group (seq, or N when scale is broadcast)
  int64_t D;
  int64_t mod_stride;
  int64_t nslots;  // G + ngroups - 1
  int* nonfinite;
  int nvec;
  int row_bytes;
  int nstages;
  int G;
  // fused stage 2 (cooperative launch): grid barrier counter (zeroed by the host) and outputs;
  // nullptr counter = stage 2 runs as the separate adaln_bwd_reduce* kernel
  unsigned int* counter;
  void* dscale;
  void* dshift;
  // dynamic tail (adaln_bwd_tma): rows [N_static, N), all in the last group, go out one stage
  // per ticket from sched[0] (sched[1] counts finished CTAs; the last re-arms both); CTA k's
  // tail partials land in slot tail_slot0 + k.  sched == nullptr: static only (N_static == N).
  unsigned int* sched;
  int64_t N_static;
  int64_t tail_slot0;
  unsigned long long* ts;  // nullable: start stamped here, end by the stage-2 kernel
  // deterministic work stealing (adaln_bwd_steal): protocol state, rows per chunk, pool slots
  // (stolen-chunk partials live in slots tail_slot0 + [0, pool_cap))
  StealSlot* steal;
  int chunk_rows;
  int pool_cap;
  // interleaved static partition (single group, adaln_bwd_tma static instance)
  int interleave;
  // 1: a consumer warp releases its ring slot as soon as its phase-1 loads are consumed, not
  // after the stage barrier (adaln_bwd_tma); more bytes stay in flight per SM
  int early_release;
};

// Row partition shared by stage 1 and stage 2.
__host__ __device__ __forceinline__ int64_t part_begin(int64_t k, int64_t N, int64_t G) {
  return k * N / G;
}
// Largest k with part_begin(k) <= row.
__host__ __device__ __forceinline__ int64_t part_owner(int64_t row, int64_t N, int64_t G) {
  return ((row + 1) * G - 1) / N;
}

// Stage schedule walker: stages of at most R rows, never crossing a group boundary.
struct StageWalker {
  int64_t row, r1, gend, grp, S;
  int64_t step = 0;  // > 0: interleaved single-group walk (init_interleaved)
  __device__ __forceinline__ void init(int64_t r0, int64_t r1_, int64_t S_) {
    row = r0;
    r1 = r1_;
    S = S_;
    grp = r0 / S_;
    gend = (grp + 1) * S_;
    step = 0;
  }
  // Interleaved partition of a single group: CTA k takes stages k, k + G, k + 2G, ... (R rows
  // each), so at any moment all CTAs stream neighbouring rows -- one sequential sweep through
  // HBM instead of G scattered streams -- while the assignment stays fixed (deterministic).
  __device__ __forceinline__ void init_interleaved(int64_t k, int64_t G, int64_t N, int R) {
    row = k * R;
    r1 = N;
    S = N;
    grp = 0;
    gend = N;
    step = G * R;
  }
  __device__ __forceinline__ bool done() const { return row >= r1; }
  // Rows of the next stage (call only when !done()); advances past it.
  __device__ __forceinline__ int next(int R, int64_t& start, int64_t& g) {
    if (step) {
      const int64_t left = r1 - row;
      const int n = left < R ? static_cast<int>(left) : R;
      start = row;
      g = 0;
      row += step;
      return n;
    }
    if (row >= gend) {
      ++grp;
      gend += S;
    }
    const int64_t lim = gend < r1 ? gend : r1;
    const int64_t left = lim - row;
    const int n = left < R ? static_cast<int>(left) : R;
    start = row;
    g = grp;
    row += n;
    return n;
  }
};

// =====================================================================================
// Forward, row-in-registers path (D up to 32*VPL 16-byte vectors).
// One warp owns one row at a time: 128-bit streaming loads of the whole row into registers,
// exact two-pass statistics from registers (warp-shuffle reductions only -- no CTA barrier),
// then y written with 128-bit streaming stores.  (1+scale, shift) of the CTA's current
// modulation group are staged once in shared memory as fp32 pairs.  Math runs on packed
// fp32 pairs (FADD2/FMUL2/FFMA2).  Rows of the CTA's contiguous range are interleaved
// across its warps; the CTA range is split into modulation-group segments, and only a segment
// change (a new sample) costs a __syncthreads.
// PACKED = true keeps the row packed in registers and re-expands it in every pass (more ALU,
// about half the registers -> twice the resident warps); false lets the compiler keep it
// expanded.
// =====================================================================================
//
// RESID: the gated-residual twin (the DiT block's "x + gate * f -> norm"):
//   x_out = x + gate (.) f   (gate per sample like scale/shift; one fp32/fp64 fma, rounded to T)
//   y     = AdaLN(x_out)     (statistics of the rounded x_out: y is bit-identical to the plain
//                             kernel applied to x_out)
// reads x and f, writes x_out and y (+ mean, rstd): 4 N*D element moves where the unfused pair
// (residual add, then the norm) moves 5 (7 with an eager mul + add).  x_out is stored in
// pass 3 next to y, so no store sits between the row loads.
template <typename T, int VPL, bool PACKED, bool PREFETCH = false, bool STAGED = false,
          bool RESID = false>
__global__ void __launch_bounds__(STAGED ? 512 : 256, RESID ? 2 : 0) adaln_fwd_rows(const FwdParams p) {
  pdl_enter();
  ts_begin(p.ts);
  static_assert(!(RESID && STAGED), "the gated residual is not staged");
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int EPV = Traits<T>::EPV;
  constexpr int NP = EPV / 2;  // pairs per 16-byte vector
  // (1+scale, shift[, gate]) staging: interleaved, pair e of vector c at c * NP + e.  (The
  // planar layout of rows2/rows16 removes the 2-way bank conflict of 16-bit rows but measured
  // 2-4 % slower here at D = 5120, long sequences -- profiles/r1_fwd_variants.jsonl.)
  auto mi = [](int c, int e) { return c * NP + e; };
  constexpr bool SHIFT = sizeof(T) >= 4;
  extern __shared__ __align__(16) uint8_t smem[];
  P* s1 = reinterpret_cast<P*>(smem);  // [nvec * NP] : 1 + scale
  P* sh = s1 + p.nvec * NP;            // [nvec * NP] : shift
  P* gt = sh + p.nvec * NP;            // [nvec * NP] : gate (RESID only)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT eps = static_cast<CT>(p.eps);
  const int RB = p.row_bytes;
  bool nf = false;

  // STAGED: each warp's next row is streamed by a 1-D TMA bulk copy into a private
  // shared-memory row buffer while the current row is being computed (one-row lookahead per
  // warp; the row itself still lives in registers for the three passes).
  uint8_t* rowbuf = smem + 2 * static_cast<size_t>(p.nvec) * NP * sizeof(P) +
                    static_cast<size_t>(warp) * RB;
  uint64_t* rbar = reinterpret_cast<uint64_t*>(smem + 2 * static_cast<size_t>(p.nvec) * NP *
                                                          sizeof(P) +
                                               static_cast<size_t>(nwarp) * RB) + warp;
  uint32_t rph = 0;
  uint64_t pol = 0;
  if constexpr (STAGED) {
    if (lane == 0) {
      mbar_init(rbar, 1);
      fence_mbar_init();
      pol = policy_evict_first();
    }
    __syncwarp();
  }

  // expand vector i of the row; with PACKED the expansion depends on the runtime zero z
  auto expand = [&](const uint4& raw, uint32_t z, P* q) {
    if constexpr (PACKED) unpack2_dep<T>(raw, z, q);
    else unpack2<T>(raw, q);
  };

  uint4 v[VPL];
  int64_t row0 = r0;
  while (row0 < r1) {
    const int64_t g = row0 / p.S_grp;
    const int64_t seg_end = min(r1, (g + 1) * p.S_grp);
    // issue this warp's first row of the segment before staging the modulation, so the HBM
    // latency of the first row overlaps the CTA prologue
    bool have_row = false;
    if constexpr (!STAGED && !RESID) {
      if (row0 + warp < seg_end) {
        const uint8_t* xr0 = static_cast<const uint8_t*>(p.x) + (row0 + warp) * RB;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          v[i] = c < p.nvec ? ld_global_nc_v4(xr0 + c * 16) : make_uint4(0, 0, 0, 0);
        }
        have_row = true;
      }
    }
    __syncthreads();  // every warp is done with the previous group's modulation
    {
      const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
      const uint8_t* sf = static_cast<const uint8_t*>(p.shift) + g * p.mod_stride * sizeof(T);
      const uint8_t* ga = static_cast<const uint8_t*>(p.gate) + g * p.mod_stride * sizeof(T);
      for (int c = tid; c < p.nvec; c += blockDim.x) {
        P a[NP], b[NP];
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sc) + c), a);
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sf) + c), b);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          nf |= !(finite_ct(a[e].x) && finite_ct(a[e].y) && finite_ct(b[e].x) && finite_ct(b[e].y));
          s1[mi(c, e)] = add2(a[e], splat2(CT(1)));
          sh[mi(c, e)] = b[e];
        }
        if constexpr (RESID) {
          unpack2<T>(__ldg(reinterpret_cast<const uint4*>(ga) + c), a);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            nf |= !(finite_ct(a[e].x) && finite_ct(a[e].y));
            gt[mi(c, e)] = a[e];
          }
        }
      }
    }
    __syncthreads();
    if constexpr (STAGED) {
      if (lane == 0 && row0 + warp < seg_end) {
        mbar_arrive_expect_tx(rbar, static_cast<uint32_t>(RB));
        bulk_g2s(rowbuf, static_cast<const uint8_t*>(p.x) + (row0 + warp) * RB, RB, rbar, pol);
      }
    }
    for (int64_t row = row0 + warp; row < seg_end; row += nwarp) {
      const uint8_t* xr = static_cast<const uint8_t*>(p.x) + row * RB;
      // optional: warm L2 with this warp's next row (measured slower on B200: off by default)
      if (PREFETCH && lane == 0 && row + nwarp < seg_end) prefetch_l2_bulk(xr + nwarp * RB, RB);
      if constexpr (STAGED) {
        mbar_wait(rbar, rph);
        rph ^= 1;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          v[i] = c < p.nvec ? ld_shared_v4(rowbuf + c * 16) : make_uint4(0, 0, 0, 0);
        }
      } else if (have_row) {
        have_row = false;  // first row of the segment: already in flight
      } else if constexpr (RESID) {
        // branch-free (predicated loads, clamped smem index): x lands in v[] exactly as in the
        // plain kernel, then f streams in and is folded in place, so at most one row of x plus
        // the in-flight f vectors are live (fits 128 registers -> 16 warps per SM)
        const uint8_t* fr = static_cast<const uint8_t*>(p.f) + row * RB;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          v[i] = c < p.nvec ? ld_global_nc_v4(xr + c * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          const bool ok = c < p.nvec;
          const int cc = ok ? c : 0;
          const uint4 fw = ok ? ld_global_nc_v4(fr + c * 16) : make_uint4(0, 0, 0, 0);
          P xa[NP], fa[NP];
          unpack2<T>(v[i], xa);
          unpack2<T>(fw, fa);
#pragma unroll
          for (int e = 0; e < NP; ++e) xa[e] = fma2(gt[mi(cc, e)], fa[e], xa[e]);
          v[i] = pack2<T>(xa);
        }
      } else {
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c = lane + 32 * i;
          v[i] = c < p.nvec ? ld_global_nc_v4(xr + c * 16) : make_uint4(0, 0, 0, 0);
        }
      }
      // 32-bit/64-bit inputs: statistics of (x - K), K = the row's first element, so that rows
      // with a large common offset keep full precision in the fp32 sums (x - K is exact for
      // clustered values).  16-bit inputs skip the shift: their own rounding dominates.
      CT K = CT(0);
      if constexpr (SHIFT) {
        P q0[NP];
        unpack2<T>(v[0], q0);
        K = __shfl_sync(0xffffffffu, q0[0].x, 0);
      }
      const P nK = splat2(-K);
      // pass 1: mean (zero-filled tail vectors add nothing)
      P acc[4] = {splat2(CT(0)), splat2(CT(0)), splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        if (!SHIFT || lane + 32 * i < p.nvec) {
          P q[NP];
          expand(v[i], 0u, q);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            if constexpr (SHIFT) q[e] = add2(q[e], nK);
            acc[(i * NP + e) & 3] = add2(acc[(i * NP + e) & 3], q[e]);
          }
        }
      }
      P t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
      const CT md = warp_sum(t.x + t.y) * invD;  // mean of (x - K)
      if constexpr (STAGED) {
        // every lane has consumed its share of the row buffer (pass 1 read all of v[] before
        // the shuffles): hand the buffer back to the async proxy for the next row
        if (lane == 0 && row + nwarp < seg_end) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(rbar, static_cast<uint32_t>(RB));
          bulk_g2s(rowbuf, xr + static_cast<int64_t>(nwarp) * RB, RB, rbar, pol);
        }
      }
      const CT mean = K + md;
      const P nm = splat2(SHIFT ? -md : -mean);
      const uint32_t z1 = PACKED ? runtime_zero(md) : 0u;
      // pass 2: sum of squared deviations (valid vectors only)
      acc[0] = acc[1] = acc[2] = acc[3] = splat2(CT(0));
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        if (lane + 32 * i < p.nvec) {
          P q[NP];
          expand(v[i], z1, q);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            if constexpr (SHIFT) q[e] = add2(q[e], nK);
            const P d = add2(q[e], nm);
            acc[(i * NP + e) & 3] = fma2(d, d, acc[(i * NP + e) & 3]);
          }
        }
      }
      t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
      const CT m2 = warp_sum(t.x + t.y);
      const CT rs = CT(1) / sqrt(m2 * invD + eps);
      const P rs2 = splat2(rs);
      const uint32_t z2 = PACKED ? runtime_zero(rs) : 0u;
      // pass 3: y = (x - mean) * rstd * (1 + scale) + shift
      uint8_t* yr = static_cast<uint8_t*>(p.y) + row * RB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < p.nvec) {
          if constexpr (RESID) st_global_cs(static_cast<uint8_t*>(p.x_out) + row * RB + c * 16, v[i]);
          P q[NP], a[NP], b[NP];
          expand(v[i], z2, q);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            a[e] = s1[mi(c, e)];
            b[e] = sh[mi(c, e)];
          }
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            if constexpr (SHIFT) q[e] = add2(q[e], nK);
            q[e] = fma2(mul2(add2(q[e], nm), rs2), a[e], b[e]);
          }
          st_global_cs(yr + c * 16, pack2<T>(q));
        }
      }
      if (lane == 0) {
        static_cast<CT*>(p.mean)[row] = mean;
        static_cast<CT*>(p.rstd)[row] = rs;
        nf |= !(finite_ct(mean) && finite_ct(m2));
      }
    }
    row0 = seg_end;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// =====================================================================================
// Forward, two rows per warp (variant 6).  Like adaln_fwd_rows<PACKED> but each warp holds
// rows (r, r+1) at once: every (1+scale, shift) shared-memory read feeds two rows (half the
// LDS traffic -- the forward's top stall is short_scoreboard on those reads), the two row
// statistics share one reduce-scatter, and the per-row loop overhead halves.  Twice the
// registers per warp, half the warps: the same bytes in flight per SM.
// =====================================================================================
template <typename T, int VPL>
__global__ void __launch_bounds__(256) adaln_fwd_rows2(const FwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int EPV = Traits<T>::EPV;
  constexpr int NP = EPV / 2;
  // interleaved (1+scale, shift) staging, as adaln_fwd_rows (planar measured ~2 % slower here)
  auto mi = [](int c, int e) { return c * NP + e; };
  constexpr bool SHIFT = sizeof(T) >= 4;
  extern __shared__ __align__(16) uint8_t smem[];
  P* s1 = reinterpret_cast<P*>(smem);
  P* sh = s1 + p.nvec * NP;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT eps = static_cast<CT>(p.eps);
  const int RB = p.row_bytes;
  bool nf = false;

  uint4 v[2][VPL];
  int64_t row0 = r0;
  while (row0 < r1) {
    const int64_t g = row0 / p.S_grp;
    const int64_t seg_end = min(r1, (g + 1) * p.S_grp);
    __syncthreads();
    {
      const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
      const uint8_t* sf = static_cast<const uint8_t*>(p.shift) + g * p.mod_stride * sizeof(T);
      for (int c = tid; c < p.nvec; c += blockDim.x) {
        P a[NP], b[NP];
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sc) + c), a);
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sf) + c), b);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          nf |= !(finite_ct(a[e].x) && finite_ct(a[e].y) && finite_ct(b[e].x) && finite_ct(b[e].y));
          s1[mi(c, e)] = add2(a[e], splat2(CT(1)));
          sh[mi(c, e)] = b[e];
        }
      }
    }
    __syncthreads();
    for (int64_t row = row0 + 2 * warp; row < seg_end; row += 2 * nwarp) {
      const bool two = row + 1 < seg_end;
      const uint8_t* xr = static_cast<const uint8_t*>(p.x) + row * RB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        v[0][i] = c < p.nvec ? ld_global_nc_v4(xr + c * 16) : make_uint4(0, 0, 0, 0);
        v[1][i] = (two && c < p.nvec) ? ld_global_nc_v4(xr + RB + c * 16) : make_uint4(0, 0, 0, 0);
      }
      CT K[2] = {CT(0), CT(0)};
      if constexpr (SHIFT) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          P q0[NP];
          unpack2<T>(v[q][0], q0);
          K[q] = __shfl_sync(0xffffffffu, q0[0].x, 0);
        }
      }
      // pass 1: means
      CT part[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const P nK = splat2(-K[q]);
        P acc[4] = {splat2(CT(0)), splat2(CT(0)), splat2(CT(0)), splat2(CT(0))};
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (!SHIFT || lane + 32 * i < p.nvec) {
            P t[NP];
            unpack2_dep<T>(v[q][i], 0u, t);
#pragma unroll
            for (int e = 0; e < NP; ++e)
              acc[(i * NP + e) & 3] = add2(acc[(i * NP + e) & 3], SHIFT ? add2(t[e], nK) : t[e]);
          }
        }
        const P t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
        part[q] = t.x + t.y;
      }
      CT md[2];
      {
        const CT u = warp_reduce_scatter<2>(part, lane);
        md[0] = __shfl_sync(0xffffffffu, u, 0) * invD;
        md[1] = __shfl_sync(0xffffffffu, u, 16) * invD;
      }
      // pass 2: squared deviations
      const uint32_t z1 = runtime_zero(md[0] + md[1]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const P nK = splat2(-K[q]), nm = splat2(-md[q]);
        P acc[4] = {splat2(CT(0)), splat2(CT(0)), splat2(CT(0)), splat2(CT(0))};
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (lane + 32 * i < p.nvec) {
            P t[NP];
            unpack2_dep<T>(v[q][i], z1, t);
#pragma unroll
            for (int e = 0; e < NP; ++e) {
              const P d = add2(SHIFT ? add2(t[e], nK) : t[e], nm);
              acc[(i * NP + e) & 3] = fma2(d, d, acc[(i * NP + e) & 3]);
            }
          }
        }
        const P t = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
        part[q] = t.x + t.y;
      }
      CT rs[2], mean[2], m2[2];
      {
        const CT u = warp_reduce_scatter<2>(part, lane);
        m2[0] = __shfl_sync(0xffffffffu, u, 0);
        m2[1] = __shfl_sync(0xffffffffu, u, 16);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          rs[q] = CT(1) / sqrt(m2[q] * invD + eps);
          mean[q] = K[q] + md[q];
        }
      }
      // pass 3: y for both rows from one read of (1+scale, shift)
      const uint32_t z2 = runtime_zero(rs[0] + rs[1]);
      const P nK0 = splat2(-K[0]), nK1 = splat2(-K[1]);
      const P nm0 = splat2(-md[0]), nm1 = splat2(-md[1]);
      const P rs0 = splat2(rs[0]), rs1 = splat2(rs[1]);
      uint8_t* yr = static_cast<uint8_t*>(p.y) + row * RB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        if (c < p.nvec) {
          P a[NP], b[NP], t0[NP], t1[NP];
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            a[e] = s1[mi(c, e)];
            b[e] = sh[mi(c, e)];
          }
          unpack2_dep<T>(v[0][i], z2, t0);
          unpack2_dep<T>(v[1][i], z2, t1);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            t0[e] = fma2(mul2(add2(SHIFT ? add2(t0[e], nK0) : t0[e], nm0), rs0), a[e], b[e]);
            t1[e] = fma2(mul2(add2(SHIFT ? add2(t1[e], nK1) : t1[e], nm1), rs1), a[e], b[e]);
          }
          st_global_cs(yr + c * 16, pack2<T>(t0));
          if (two) st_global_cs(yr + RB + c * 16, pack2<T>(t1));
        }
      }
      if (lane == 0) {
        static_cast<CT*>(p.mean)[row] = mean[0];
        static_cast<CT*>(p.rstd)[row] = rs[0];
        nf |= !(finite_ct(mean[0]) && finite_ct(m2[0]));
        if (two) {
          static_cast<CT*>(p.mean)[row + 1] = mean[1];
          static_cast<CT*>(p.rstd)[row + 1] = rs[1];
          nf |= !(finite_ct(mean[1]) && finite_ct(m2[1]));
        }
      }
    }
    row0 = seg_end;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// =====================================================================================
// Forward, row-in-registers path for 16-bit rows (bf16 / fp16): the row stays packed in
// registers and is consumed by mixed-precision adds (FHADD.{BF16,F16}: 16-bit operand, fp32
// result), so there is no separate expansion step.  Exact two-pass statistics from the
// registers (mean, then the centred sum of squares), then y = (x - mean) * rstd * (1 + scale)
// + shift.  About 5.5 instructions per element instead of 8 for the unpacking kernel.
// =====================================================================================
template <typename T, int VPL, bool RESID = false>
__global__ void __launch_bounds__(256, 2) adaln_fwd_rows16(const FwdParams p) {
  pdl_enter();
  ts_begin(p.ts);
  if (threadIdx.x == 0) AL_TRACE(0, 0);
  static_assert(sizeof(T) == 2, "16-bit rows only");
  using P = float2;
  constexpr int NP = 4;  // pairs per 16-byte vector
  // (1+scale, shift) staging in shared memory, planar by 16-byte chunk: pair e of vector c
  // lives in plane e / HP, so the per-lane 16-byte reads of one plane are consecutive across
  // the warp (no 2-way bank conflict: 16-bit vectors expand to 32 bytes of fp32 pairs).
  // Measured +6-8 % at short sequences (cfg3 S <= 3600), where this kernel is selected.
  constexpr int HP = 16 / static_cast<int>(sizeof(P));
  const int nvec_ = p.nvec;
  auto mi = [nvec_](int c, int e) { return ((e / HP) * nvec_ + c) * HP + (e % HP); };
  extern __shared__ __align__(16) uint8_t smem[];
  P* s1 = reinterpret_cast<P*>(smem);  // [nvec * NP] : 1 + scale
  P* sh = s1 + p.nvec * NP;            // [nvec * NP] : shift
  P* gt = sh + p.nvec * NP;            // [nvec * NP] : gate (RESID: the gated-residual twin)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int64_t k = blockIdx.x;
  // static head: rows [0, N_static) split evenly over the CTAs; dynamic tail: rows
  // [N_static, N) handed out one row per warp from a global ticket counter (p.sched)
  const int64_t r0 = part_begin(k, p.N_static, p.G), r1 = part_begin(k + 1, p.N_static, p.G);
  const float invD = 1.0f / static_cast<float>(p.D);
  const float eps = static_cast<float>(p.eps);
  const int RB = p.row_bytes;
  bool nf = false;

  auto mod_smem = [&](int c, P* a, P* b) {
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      a[e] = s1[mi(c, e)];
      b[e] = sh[mi(c, e)];
    }
  };
  // one row by one warp
  auto do_row = [&](int64_t row) {
    const uint8_t* xr = static_cast<const uint8_t*>(p.x) + row * RB;
    uint4 v[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      v[i] = c < p.nvec ? ld_global_nc_v4(xr + c * 16) : make_uint4(0, 0, 0, 0);
    }
    if constexpr (RESID) {
      // x_out = x + gate * f: one fp32 fma per element, rounded to T (as adaln_fwd_rows<RESID>),
      // folded into v[] vector by vector while f streams in; the statistics below are then those
      // of the rounded x_out, so y equals this kernel's forward on x_out bit for bit
      const uint8_t* fr = static_cast<const uint8_t*>(p.f) + row * RB;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = lane + 32 * i;
        const bool ok = c < p.nvec;
        const int cc = ok ? c : 0;
        const uint4 fw = ok ? ld_global_nc_v4(fr + c * 16) : make_uint4(0, 0, 0, 0);
        P xa[NP], fa[NP];
        unpack2<T>(v[i], xa);
        unpack2<T>(fw, fa);
#pragma unroll
        for (int e = 0; e < NP; ++e) xa[e] = fma2(gt[mi(cc, e)], fa[e], xa[e]);
        v[i] = pack2<T>(xa);
      }
    }
    // Exact two-pass statistics from the register-resident row (the reference's order of
    // operations, _kernels_numba.py:22-30): pass 1 the mean, pass 2 the centred sum of squares
    // -- no E[x^2] - E[x]^2 cancellation whatever the row's offset or outliers.  Both passes
    // read the packed 16-bit row through mixed-precision adds (FHADD: 16-bit operand, fp32
    // result), so neither needs an unpack step.
    float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      if (lane + 32 * i < p.nvec) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = acc16x2_f32<T>(w[e], make_float2(s4[(2 * e) & 3], s4[(2 * e + 1) & 3]));
          s4[(2 * e) & 3] = a.x;
          s4[(2 * e + 1) & 3] = a.y;
        }
      }
    }
    const float mean = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3])) * invD;
    P q[2] = {splat2(0.0f), splat2(0.0f)};
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      if (lane + 32 * i < p.nvec) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const P dd = sub16x2_f32<T>(w[e], -mean);
          q[e & 1] = fma2(dd, dd, q[e & 1]);
        }
      }
    }
    const P tq = add2(q[0], q[1]);
    const float sq = warp_sum(tq.x + tq.y);
    const float m2 = sq;
    const float rs = 1.0f / sqrtf(m2 * invD + eps);
    const P rs2 = splat2(rs);
    // pass 2: y = (x - mean) * rstd * (1 + scale) + shift
    uint8_t* yr = static_cast<uint8_t*>(p.y) + row * RB;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < p.nvec) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        P a[NP], b[NP], o[NP];
        mod_smem(c, a, b);
#pragma unroll
        for (int e = 0; e < NP; ++e) o[e] = fma2(mul2(sub16x2_f32<T>(w[e], -mean), rs2), a[e], b[e]);
        if constexpr (RESID) st_global_cs(static_cast<uint8_t*>(p.x_out) + row * RB + c * 16, v[i]);
        st_global_cs(yr + c * 16, pack2<T>(o));
      }
    }
    if (lane == 0) {
      static_cast<float*>(p.mean)[row] = mean;
      static_cast<float*>(p.rstd)[row] = rs;
      nf |= !(finite_ct(mean) && finite_ct(sq));
    }
  };

  // stage (1 + scale, shift) of group g; the caller brackets it with __syncthreads
  auto stage_group = [&](int64_t g) {
    const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
    const uint8_t* sf = static_cast<const uint8_t*>(p.shift) + g * p.mod_stride * sizeof(T);
    for (int c = tid; c < p.nvec; c += blockDim.x) {
      P a[NP], b[NP];
      unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sc) + c), a);
      unpack2<T>(__ldg(reinterpret_cast<const uint4*>(sf) + c), b);
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        nf |= !(finite_ct(a[e].x) && finite_ct(a[e].y) && finite_ct(b[e].x) && finite_ct(b[e].y));
        s1[mi(c, e)] = add2(a[e], splat2(1.0f));
        sh[mi(c, e)] = b[e];
      }
      if constexpr (RESID) {
        const uint8_t* ga = static_cast<const uint8_t*>(p.gate) + g * p.mod_stride * sizeof(T);
        unpack2<T>(__ldg(reinterpret_cast<const uint4*>(ga) + c), a);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          nf |= !(finite_ct(a[e].x) && finite_ct(a[e].y));
          gt[mi(c, e)] = a[e];
        }
      }
    }
  };

  int64_t staged = -1;
  int64_t row0 = r0;
  while (row0 < r1) {
    const int64_t g = row0 / p.S_grp;
    const int64_t seg_end = min(r1, (g + 1) * p.S_grp);
    __syncthreads();  // every warp is done with the previous group's modulation
    stage_group(g);
    __syncthreads();
    staged = g;
    for (int64_t row = row0 + warp; row < seg_end; row += nwarp) do_row(row);
    row0 = seg_end;
  }

  if (p.sched != nullptr && p.dyn_groups) {
    // Multi-group dynamic tail (multi-sample launches): whole groups [N_static / S_grp, ...)
    // cut into chunks of 2 rows per warp that never cross a group; the CTA draws one chunk per
    // ticket (thread 0, one chunk ahead, double-buffered in shared memory), restages the
    // modulation when the chunk's group changes, and its warps split the chunk's rows.  One
    // barrier per chunk; every row runs the same code as in the static part.  (Per-warp tickets
    // with the modulation read from global memory instead measured 16-20 % slower.)
    __shared__ long long s_tk[2];
    const int CH = 2 * nwarp;
    const int64_t g0 = p.N_static / p.S_grp;
    const int64_t cpg = (p.S_grp + CH - 1) / CH;
    const int64_t nch = ((p.N + p.S_grp - 1) / p.S_grp - g0) * cpg;
    if (tid == 0) s_tk[0] = static_cast<long long>(atomicAdd(p.sched, 1u));
    __syncthreads();
    int buf = 0;
    while (true) {
      const int64_t t = s_tk[buf];
      if (t >= nch) break;
      if (tid == 0) s_tk[buf ^ 1] = static_cast<long long>(atomicAdd(p.sched, 1u));
      const int64_t g = g0 + t / cpg;
      const int64_t rs0 = g * p.S_grp + (t % cpg) * CH;
      const int64_t re = min(min(rs0 + CH, (g + 1) * p.S_grp), p.N);
      if (g != staged) {  // CTA-uniform; the previous chunk ended with a barrier
        stage_group(g);
        __syncthreads();
        staged = g;
      }
      for (int64_t row = rs0 + warp; row < re; row += nwarp) do_row(row);
      __syncthreads();  // the staging and the ticket buffer may be reused
      buf ^= 1;
    }
  } else if (p.sched != nullptr) {
    // Dynamic tail: bandwidth is not shared evenly between SMs once the kernel is
    // memory-bound (per-CTA end times of a fully static split spread 87..122 us at cfg2), so
    // the last rows go to whichever warps are free.  The host keeps the tail inside the last
    // modulation group, staged here once.  The next ticket is requested before the current
    // row is processed, hiding the atomic's round trip.  Every row runs the same instruction
    // sequence wherever it lands, so results do not depend on the assignment.
    const int64_t gl = (p.N - 1) / p.S_grp;
    if (staged != gl) {
      __syncthreads();
      stage_group(gl);
      __syncthreads();
    }
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(p.sched, 1u);
    int64_t row = p.N_static + __shfl_sync(0xffffffffu, t, 0);
    while (row < p.N) {
      unsigned int tn = 0;
      if (lane == 0) tn = atomicAdd(p.sched, 1u);
      do_row(row);
      row = p.N_static + __shfl_sync(0xffffffffu, tn, 0);
    }
  }
  if (p.sched != nullptr) {
    // the last CTA out re-arms the counter pair for the next launch that draws this slot
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1u) == static_cast<unsigned int>(p.G - 1)) {
        atomicExch(p.sched, 0u);
        atomicExch(p.sched + 1, 0u);
      }
    }
  }
#ifdef AL_CTA_TRACE
  __syncthreads();
  if (tid == 0) AL_TRACE(0, 1);
#endif
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
  if (p.ts != nullptr) {
    __syncthreads();
    if (tid == 0) ts_end(p.ts);
  }
}

// =====================================================================================
// Forward, wide-row TMA ring path (rows too wide for registers).
// blockDim = nc consumers (multiple of 32) + 1 producer warp.  Stage = R rows streamed into
// shared memory by 1-D bulk copies; consumer thread t owns 16-byte vectors t + i*nc.
// Statistics: per-thread two-pass over (x - K) with K = the row's first element (shifted data:
// exact differences for clustered rows), merged across lanes and warps with the parallel
// variance identity M2 = sum_i [M2_i + n_i (m_i - m)^2].
// =====================================================================================
template <typename T, int V, int R>
__global__ void __launch_bounds__(512) adaln_fwd_wide(const FwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  constexpr int EPV = Traits<T>::EPV;
  extern __shared__ __align__(128) uint8_t smem[];

  const int nc = blockDim.x - 32;
  const int ncw = nc >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = p.nstages;
  const int RB = p.row_bytes;
  const int stage_bytes = R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * stage_bytes);
  uint64_t* empty = full + NS;
  CT* red = reinterpret_cast<CT*>(empty + NS);  // [2][ncw][R][2] : (warp mean, warp M2)
  CT* wcnt = red + 2 * ncw * R * 2;             // [ncw] elements per warp

  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);

  uint32_t vmask = 0;
  int nown = 0;
  if (tid < nc) {
#pragma unroll
    for (int j = 0; j < V; ++j)
      if (tid + j * nc < p.nvec) {
        vmask |= 1u << j;
        ++nown;
      }
    const CT nw = warp_sum(static_cast<CT>(nown * EPV));
    if (lane == 0) wcnt[warp] = nw;
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == ncw) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* xb = static_cast<const uint8_t*>(p.x);
      StageWalker w;
      w.init(r0, r1, p.S_grp);
      int s = 0;
      uint32_t f = 0;
      while (!w.done()) {
        int64_t start, g;
        const int rows = w.next(R, start, g);
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows * RB));
        uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
        for (int rr = 0; rr < rows; ++rr)
          bulk_g2s(dst + rr * RB, xb + (start + rr) * RB, RB, &full[s], pol);
        if (++s == NS) {
          s = 0;
          ++f;
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const CT n_t = static_cast<CT>(nown * EPV);
  const CT inv_nt = nown ? CT(1) / n_t : CT(0);
  const CT inv_nw = CT(1) / wcnt[warp];
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT eps = static_cast<CT>(p.eps);
  bool nf = false;

  CT s1[V][EPV], sh[V][EPV];
  int64_t cur_g = -1;

  StageWalker w;
  w.init(r0, r1, p.S_grp);
  int s = 0;
  uint32_t ph = 0;
  int it = 0;
  while (!w.done()) {
    int64_t rb, g;
    const int rows = w.next(R, rb, g);
    if (g != cur_g) {  // uniform: reload (1+scale), shift of the owned columns
      cur_g = g;
      const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
      const uint8_t* sf = static_cast<const uint8_t*>(p.shift) + g * p.mod_stride * sizeof(T);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (vmask >> j & 1) {
          const size_t off = static_cast<size_t>(tid + j * nc) * 16;
          unpack<T>(__ldg(reinterpret_cast<const uint4*>(sc + off)), s1[j]);
          unpack<T>(__ldg(reinterpret_cast<const uint4*>(sf + off)), sh[j]);
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            nf |= !(finite_ct(s1[j][e]) && finite_ct(sh[j][e]));
            s1[j][e] += CT(1);
          }
        }
      }
    }
    mbar_wait(&full[s], ph);
    const uint8_t* st = smem + static_cast<size_t>(s) * stage_bytes;
    CT* rd = red + (it & 1) * (ncw * R * 2);

    // phase 1: per-row statistics of the owned elements (shifted by K), merged within the warp
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr < rows) {
        CT kk[EPV];
        unpack<T>(ld_shared_v4(st + rr * RB), kk);
        const CT K = kk[0];
        CT v[V][EPV];
        CT sum = CT(0);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            unpack<T>(ld_shared_v4(st + rr * RB + (tid + j * nc) * 16), v[j]);
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              v[j][e] -= K;
              sum += v[j][e];
            }
          }
        }
        const CT mt = sum * inv_nt;
        CT m2 = CT(0);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              const CT d = v[j][e] - mt;
              m2 = fma(d, d, m2);
            }
          }
        }
        const CT mw = warp_sum(sum) * inv_nw;
        const CT dm = mt - mw;
        const CT q = warp_sum(fma(n_t * dm, dm, m2));
        if (lane == 0) {
          rd[(warp * R + rr) * 2 + 0] = mw;
          rd[(warp * R + rr) * 2 + 1] = q;
        }
      }
    }
    named_bar_sync(1, nc);

    // phase 2: merge warps (fixed order), normalise, modulate, store
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr < rows) {
        const int64_t row = rb + rr;
        CT kk[EPV];
        unpack<T>(ld_shared_v4(st + rr * RB), kk);
        const CT K = kk[0];
        CT md = CT(0);  // mean of (x - K)
        for (int q = 0; q < ncw; ++q) md = fma(wcnt[q], rd[(q * R + rr) * 2], md);
        md *= invD;
        CT m2 = CT(0);
        for (int q = 0; q < ncw; ++q) {
          const CT d = rd[(q * R + rr) * 2] - md;
          m2 += fma(wcnt[q] * d, d, rd[(q * R + rr) * 2 + 1]);
        }
        const CT rs = CT(1) / sqrt(m2 * invD + eps);
        uint8_t* yrow = static_cast<uint8_t*>(p.y) + row * RB;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            CT v[EPV];
            unpack<T>(ld_shared_v4(st + rr * RB + (tid + j * nc) * 16), v);
#pragma unroll
            for (int e = 0; e < EPV; ++e) v[e] = fma(((v[e] - K) - md) * rs, s1[j][e], sh[j][e]);
            st_global_cs(yrow + (tid + j * nc) * 16, pack<T>(v));
          }
        }
        if (tid == 0) {
          const CT mean = K + md;
          static_cast<CT*>(p.mean)[row] = mean;
          static_cast<CT*>(p.rstd)[row] = rs;
          nf |= !(finite_ct(mean) && finite_ct(m2));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    ++it;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// =====================================================================================
// Forward, TMA ring in the backward's mould (variant 7; the default for 32-bit rows of
// D >= 2048 and for 16-bit rows wider than the rows kernels take).
// One producer lane streams R rows of x per stage into an NS-deep shared-memory ring with 1-D
// bulk copies; consumer thread t owns 16-byte column vectors t + j*nc.  Per stage: the owned
// vectors of the R rows are read once from shared memory and kept PACKED in registers, the row
// sums are reduce-scattered within the warp and combined across warps through a named barrier,
// the slot is released, and y = (x - mean) * rstd * (1 + scale) + shift is written from the
// registers.  Packed fp32 pair math; (1 + scale, shift) of the owned columns live in registers.
// Statistics of d = x - K (K = the row's first element), exact two passes from the registers
// (sum d, barrier, sum (d - mean_d)^2, barrier) for every dtype -- a single pass of sum d and
// sum d^2 can lose the variance of rows whose first element is a far outlier.
// =====================================================================================
template <typename T, int V, int R>
__global__ void __launch_bounds__(384) adaln_fwd_ring(const FwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int NP = Traits<T>::EPV / 2;
  constexpr bool TWO = true;  // exact two-pass statistics (the one-pass branch is kept for A/B)
  constexpr int NV = TWO ? R : 2 * R;  // row sums reduced per barrier
  extern __shared__ __align__(128) uint8_t smem[];

  const int nc = blockDim.x - 32;
  const int ncw = nc >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = p.nstages;
  const int RB = p.row_bytes;
  const int stage_bytes = R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * stage_bytes);
  uint64_t* empty = full + NS;
  // [2 parities][ncw][2R]: (sum d, sum d^2) per row; two-pass rows use the halves for the
  // two passes
  CT* red = reinterpret_cast<CT*>(empty + NS);

  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == ncw) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* xb = static_cast<const uint8_t*>(p.x);
      StageWalker w;
      w.init(r0, r1, p.S_grp);
      int s = 0;
      uint32_t f = 0;
      while (!w.done()) {
        int64_t start, g;
        const int rows = w.next(R, start, g);
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows * RB));
        uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
        for (int rr = 0; rr < rows; ++rr)
          bulk_g2s(dst + rr * RB, xb + (start + rr) * RB, RB, &full[s], pol);
        if (++s == NS) {
          s = 0;
          ++f;
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  uint32_t vmask = 0u;
  int coff[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    coff[j] = (tid + j * nc) * 16;
    if (tid + j * nc < p.nvec) vmask |= 1u << j;
  }
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT eps = static_cast<CT>(p.eps);
  const uint32_t ring_u = smem_addr(smem);
  bool nf = false;

  // warp reduce-scatter of NV row sums, then the cross-warp totals spread over the lanes
  auto reduce_rows = [&](const CT* v, CT* buf, CT* out) {
    constexpr int GRP = 32 / NV;
    const CT u = warp_reduce_scatter<NV>(v, lane);
    if ((lane & (GRP - 1)) == 0) buf[warp * NV + lane / GRP] = u;
    named_bar_sync(1, nc);
    return [=](CT* o) {
      const int nval = ncw * NV;
      CT s_l = CT(0);
      for (int i = lane; i < nval; i += 32) s_l += buf[i];
#pragma unroll
      for (int off = NV; off < 32; off <<= 1) s_l += __shfl_xor_sync(0xffffffffu, s_l, off);
#pragma unroll
      for (int q = 0; q < NV; ++q) o[q] = __shfl_sync(0xffffffffu, s_l, q);
    };
  };

  P s1[V][NP], shv[V][NP];
  int64_t cur_g = -1;
  StageWalker w;
  w.init(r0, r1, p.S_grp);
  int s = 0;
  uint32_t ph = 0;
  int it = 0;
  while (!w.done()) {
    int64_t rb, g;
    const int rows = w.next(R, rb, g);
    if (g != cur_g) {
      cur_g = g;
      const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
      const uint8_t* sf = static_cast<const uint8_t*>(p.shift) + g * p.mod_stride * sizeof(T);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = vmask >> j & 1;
        unpack2<T>(ok ? __ldg(reinterpret_cast<const uint4*>(sc + coff[j])) : make_uint4(0, 0, 0, 0), s1[j]);
        unpack2<T>(ok ? __ldg(reinterpret_cast<const uint4*>(sf + coff[j])) : make_uint4(0, 0, 0, 0), shv[j]);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          nf |= !(finite_ct(s1[j][e].x) && finite_ct(s1[j][e].y) && finite_ct(shv[j][e].x) &&
                  finite_ct(shv[j][e].y));
          s1[j][e] = add2(s1[j][e], splat2(CT(1)));
        }
      }
    }
    mbar_wait(&full[s], ph);
    const uint32_t st = ring_u + static_cast<uint32_t>(s * stage_bytes);
    CT* rd = red + (it & 1) * (ncw * 2 * R);

    // phase 1: first-pass sums from the packed row slice, kept in registers
    uint4 xr[R][V];
    CT K[R], rowsum[2 * R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const bool live = rr < rows;
      {
        P k0[NP];
        unpack2<T>(live ? ld_shared_v4_u32(st + rr * RB) : make_uint4(0, 0, 0, 0), k0);
        K[rr] = k0[0].x;
      }
      const P nK = splat2(-K[rr]);
      P a1[2] = {splat2(CT(0)), splat2(CT(0))}, a2[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = live && (vmask >> j & 1);
        xr[rr][j] = ok ? ld_shared_v4_u32(st + static_cast<uint32_t>(rr * RB + coff[j]))
                       : make_uint4(0, 0, 0, 0);
        if (ok) {
          P q[NP];
          unpack2<T>(xr[rr][j], q);
#pragma unroll
          for (int e = 0; e < NP; ++e) {
            const P d = add2(q[e], nK);
            a1[e & 1] = add2(a1[e & 1], d);
            if constexpr (!TWO) a2[e & 1] = fma2(d, d, a2[e & 1]);
          }
        }
      }
      const P t1 = add2(a1[0], a1[1]), t2 = add2(a2[0], a2[1]);
      if constexpr (TWO) {
        rowsum[rr] = t1.x + t1.y;
      } else {
        rowsum[2 * rr] = t1.x + t1.y;
        rowsum[2 * rr + 1] = t2.x + t2.y;
      }
    }
    auto fin1 = reduce_rows(rowsum, rd, nullptr);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage is in registers: hand the slot back

    CT md[R], m2v[R];
    {
      CT tot[2 * R];
      fin1(tot);
      if constexpr (TWO) {
        // second pass: centred squares from the registers
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          md[rr] = tot[rr] * invD;
          const P nK = splat2(-K[rr]), nmd = splat2(-md[rr]);
          P a2[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if (rr < rows && (vmask >> j & 1)) {
              P q[NP];
              unpack2<T>(xr[rr][j], q);
#pragma unroll
              for (int e = 0; e < NP; ++e) {
                const P d = add2(add2(q[e], nK), nmd);
                a2[e & 1] = fma2(d, d, a2[e & 1]);
              }
            }
          }
          const P t2 = add2(a2[0], a2[1]);
          rowsum[rr] = t2.x + t2.y;
        }
        auto fin2 = reduce_rows(rowsum, rd + ncw * R, nullptr);
        fin2(m2v);
      } else {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          md[rr] = tot[2 * rr] * invD;
          m2v[rr] = fmax(tot[2 * rr + 1] - tot[2 * rr] * md[rr], CT(0));
        }
      }
    }

    // phase 2: y = ((x - K) - mean_d) * rstd * (1 + scale) + shift
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr < rows) {
        const int64_t row = rb + rr;
        const CT rs = CT(1) / sqrt(m2v[rr] * invD + eps);
        const P nK = splat2(-K[rr]), nmd = splat2(-md[rr]), rs2 = splat2(rs);
        uint8_t* yrow = static_cast<uint8_t*>(p.y) + row * RB;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            P q[NP];
            unpack2<T>(xr[rr][j], q);
#pragma unroll
            for (int e = 0; e < NP; ++e)
              q[e] = fma2(mul2(add2(add2(q[e], nK), nmd), rs2), s1[j][e], shv[j][e]);
            st_global_cs(yrow + coff[j], pack2<T>(q));
          }
        }
        if (tid == 0) {
          static_cast<CT*>(p.mean)[row] = K[rr] + md[rr];
          static_cast<CT*>(p.rstd)[row] = rs;
          nf |= !(finite_ct(md[rr]) && finite_ct(m2v[rr]));
        }
      }
    }
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    ++it;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// =====================================================================================
// Fused stage 2 (cooperative launch only: every CTA of the grid is co-resident).
// After its stage-1 partials are stored, each CTA passes a grid barrier (one atomic per CTA
// on a host-zeroed counter), then reduces a contiguous share of the (group, 16-byte column
// vector) items over the CTAs that cover the group: one warp per item, each lane summing a
// strided subset of the slots in fp64, combined by a fixed butterfly -- deterministic, and
// the same fp64 sum order for every call with the same launch geometry.
// =====================================================================================
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename CT>
__device__ void fused_stage2(const BwdParams& p, int nc, int tid) {
  constexpr int VE = 16 / sizeof(CT);
  const int lane = tid & 31, warp = tid >> 5, ncw = nc >> 5;
  __threadfence();
  named_bar_sync(1, nc);
  if (tid == 0) {
    atomicAdd(p.counter, 1u);
    while (ld_acquire_gpu(p.counter) < static_cast<unsigned int>(p.G)) __nanosleep(64);
  }
  named_bar_sync(1, nc);
  const int64_t nvecs = p.D / VE;
  const int64_t ngroups = (p.N + p.S_grp - 1) / p.S_grp;
  const int64_t items = ngroups * nvecs;
  const int64_t per = (items + p.G - 1) / p.G;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t i1 = min(items, i0 + per);
  const CT* ws = static_cast<const CT*>(p.ws);
  for (int64_t it = i0 + warp; it < i1; it += ncw) {
    const int64_t g = it / nvecs, cv = it % nvecs;
    const int64_t first_row = g * p.S_grp;
    const int64_t last_row = min((g + 1) * p.S_grp, p.N) - 1;
    const int64_t kf = part_owner(first_row, p.N, p.G), kl = part_owner(last_row, p.N, p.G);
    const CT* sc = ws + (kf + g) * p.D + cv * VE;
    const CT* sh = ws + (p.nslots + kf + g) * p.D + cv * VE;
    double a[VE], b[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) a[e] = b[e] = 0.0;
    for (int64_t s = lane; s <= kl - kf; s += 32) {
      const uint4 va = __ldcg(reinterpret_cast<const uint4*>(sc + s * p.D));
      const uint4 vb = __ldcg(reinterpret_cast<const uint4*>(sh + s * p.D));
      const CT* pa = reinterpret_cast<const CT*>(&va);
      const CT* pb = reinterpret_cast<const CT*>(&vb);
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        a[e] += static_cast<double>(pa[e]);
        b[e] += static_cast<double>(pb[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      a[e] = warp_sum(a[e]);
      b[e] = warp_sum(b[e]);
    }
    if (lane == 0) {
      CT* ds = static_cast<CT*>(p.dscale) + g * p.D + cv * VE;
      CT* dh = static_cast<CT*>(p.dshift) + g * p.D + cv * VE;
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        ds[e] = static_cast<CT>(a[e]);
        dh[e] = static_cast<CT>(b[e]);
      }
    }
  }
}

// =====================================================================================
// Backward stage 1, TMA ring path.  Stage layout: [x: R rows][dy: R rows].
// Consumer thread t owns 16-byte column vectors t + i*nc (i < V): per row it forms
// xhat = (x - mu) * rstd and g = dy * (1 + scale) once, keeps both in registers across the
// row-sum barrier, folds dy and dy*xhat into its column accumulators, and after the barrier
// writes dx = rstd * (g - mean(g) - xhat * mean(g*xhat)).  Packed fp32 pair math.
//
// Static head + optional dynamic tail (p.sched != nullptr): rows [0, N_static) are split
// evenly over the CTAs, accumulated per (CTA, group) into slot k + g (deterministic).  Rows
// [N_static, N) -- inside the last group -- are handed out one stage at a time by a global
// ticket counter that the producer lane draws from; the producer passes each stage's row
// index, count and statistics to the consumers in a per-stage header next to the ring.  The
// tail's partials go to the CTA's tail slot tail_slot0 + k; their sum order depends on which
// CTA drew which stage, so dscale/dshift of the last group are reproducible only to fp32
// rounding in this mode (dx is bit-identical either way).
// =====================================================================================
// GW: the group-sequential walk instance (p.interleave == 2); kept out of the other instances,
// whose code it would otherwise change (+5 registers, 2 % slower at cfg2).  (Written as a
// runtime test on p.interleave rather than `if constexpr`: that form of the GW instance
// measured 7 % slower on the walk itself, a code-generation effect -- profiles/r2_bwd_group_walk.jsonl)
template <typename T, int V, int R, bool FULL, bool DYN, bool GW = false>
__global__ void __launch_bounds__(V == 1 ? 704 : 384) adaln_bwd_tma(const BwdParams p) {
  pdl_enter();
  ts_begin(p.ts);
  if (threadIdx.x == 0) AL_TRACE(1, 0);
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int EPV = Traits<T>::EPV;
  constexpr int NP = EPV / 2;
  extern __shared__ __align__(128) uint8_t smem[];

  const int nc = blockDim.x - 32;
  const int ncw = nc >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = p.nstages;
  const int RB = p.row_bytes;
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * stage_bytes);
  uint64_t* empty = full + NS;
  CT* red = reinterpret_cast<CT*>(empty + NS);  // [2][ncw][R][2] : (sum g, sum g*xhat)
  // dynamic-tail stage headers: row, rows, mean[R], rstd[R] per ring slot
  int64_t* h_row = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(red + 2 * ncw * R * 2) + 7) & ~uintptr_t(7));
  int* h_n = reinterpret_cast<int*>(h_row + NS);
  CT* h_m = reinterpret_cast<CT*>(
      (reinterpret_cast<uintptr_t>(h_n + NS) + 7) & ~uintptr_t(7));
  CT* h_r = h_m + NS * R;

  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N_static, p.G), r1 = part_begin(k + 1, p.N_static, p.G);
  const bool dyn = DYN && p.sched != nullptr;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == ncw) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* xb = static_cast<const uint8_t*>(p.x);
      const uint8_t* db = static_cast<const uint8_t*>(p.dy);
      StageWalker w;
      if (GW && p.interleave == 2) w.init(0, 0, p.S_grp);  // empty: the group walk below
      else if (p.interleave) w.init_interleaved(k, p.G, p.N, R);
      else w.init(r0, r1, p.S_grp);
      int s = 0;
      uint32_t f = 0;
      auto issue = [&](int64_t start, int rows) {
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(2 * rows * RB));
        uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
        for (int rr = 0; rr < rows; ++rr) {
          bulk_g2s(dst + rr * RB, xb + (start + rr) * RB, RB, &full[s], pol);
          bulk_g2s(dst + (R + rr) * RB, db + (start + rr) * RB, RB, &full[s], pol);
        }
        if (++s == NS) {
          s = 0;
          ++f;
        }
      };
      if (GW && p.interleave == 2) {
        // group-sequential interleaved walk (multi-sample launches of long samples): the
        // interleaved walk of group 0, then of group 1, ... (same order as the consumers)
        const int64_t ng = (p.N + p.S_grp - 1) / p.S_grp;
        for (int64_t gi = 0; gi < ng; ++gi) {
          const int64_t g0 = gi * p.S_grp, g1 = g0 + p.S_grp < p.N ? g0 + p.S_grp : p.N;
          const int64_t nst = (g1 - g0 + R - 1) / R;
          for (int64_t st = k; st < nst; st += p.G) {
            const int64_t start = g0 + st * R;
            const int rows = g1 - start < R ? static_cast<int>(g1 - start) : R;
            if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
            issue(start, rows);
          }
        }
      }
      while (!w.done()) {
        int64_t start, g;
        const int rows = w.next(R, start, g);
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        issue(start, rows);
      }
      if (dyn) {
        // tickets and their statistics are fetched one stage ahead, so neither the atomic's
        // nor the loads' round trip sits between two stage issues
        const CT* mean_p = static_cast<const CT*>(p.mean);
        const CT* rstd_p = static_cast<const CT*>(p.rstd);
        auto stats = [&](int64_t start, CT* m, CT* r) {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const bool ok = start + rr < p.N;
            m[rr] = ok ? mean_p[start + rr] : CT(0);
            r[rr] = ok ? rstd_p[start + rr] : CT(0);
          }
        };
        int64_t start = p.N_static + static_cast<int64_t>(atomicAdd(p.sched, 1u)) * R;
        CT m[R], r[R];
        stats(start, m, r);
        unsigned int tn = atomicAdd(p.sched, 1u);
        while (true) {
          const int rows = start < p.N ? static_cast<int>(p.N - start < R ? p.N - start : R) : 0;
          if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
          h_row[s] = start;
          h_n[s] = rows;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            h_m[s * R + rr] = m[rr];
            h_r[s * R + rr] = r[rr];
          }
          if (rows == 0) {  // end marker: completes the slot's phase without data
            mbar_arrive(&full[s]);
            break;
          }
          issue(start, rows);
          start = p.N_static + static_cast<int64_t>(tn) * R;
          if (start < p.N) {
            stats(start, m, r);
            tn = atomicAdd(p.sched, 1u);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // FULL: every consumer owns all V vectors (nvec == V * nc), so ownership tests fold away
  uint32_t vmask = FULL ? (1u << V) - 1 : 0u;
  int coff[V];  // byte offset of owned vector j inside a row
#pragma unroll
  for (int j = 0; j < V; ++j) {
    coff[j] = (tid + j * nc) * 16;
    if (!FULL && tid + j * nc < p.nvec) vmask |= 1u << j;
  }
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT* mean_p = static_cast<const CT*>(p.mean);
  const CT* rstd_p = static_cast<const CT*>(p.rstd);
  CT* ws_sc = static_cast<CT*>(p.ws);
  CT* ws_sh = ws_sc + p.nslots * p.D;
  bool nf = false;

  P s1[V][NP], acc_sc[V][NP], acc_sh[V][NP];
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));

  auto flush = [&](int64_t slot) {
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
          acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));
        }
      }
    }
  };
  auto load_scale = [&](int64_t g) {
    const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
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
    }
  };

  if constexpr (DYN) {
  int s = 0;
  uint32_t ph = 0;
  int it = 0;

  // One ring stage (the caller has waited on full[s]): `rows` rows from rb, statistics in
  // mc/rc.  ALL (compile time) = the stage holds R rows, so no row predicates or zero fills
  // are emitted on the common path; short stages take the predicated instance.
  auto stage = [&](auto all_tag, int64_t rb, int rows, const CT* mc, const CT* rc) {
    constexpr bool ALL = decltype(all_tag)::value;
    // 32-bit shared-window addresses: no generic->shared conversion per load (+1.3 %)
    const uint32_t stx_u = smem_addr(smem) + static_cast<uint32_t>(s * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    CT* rd = red + (it & 1) * (ncw * R * 2);

    // phase 1: row sums of g and g*xhat; column accumulators of dy and dy*xhat.
    // Rows past `rows` (stage tail) and columns past D read as zero, so every lane runs the
    // same instruction stream and the shuffles below are convergent.
    // the stage's x and dy vectors into registers first
    uint4 rawx[R][V], rawd[R][V];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = (ALL || rr < rows) && (vmask >> j & 1);
        const uint32_t o = static_cast<uint32_t>(rr * RB + coff[j]);
        rawx[rr][j] = ok ? ld_shared_v4_u32(stx_u + o) : make_uint4(0, 0, 0, 0);
        rawd[rr][j] = ok ? ld_shared_v4_u32(std_u + o) : make_uint4(0, 0, 0, 0);
      }
    P xh[R][V][NP], gg[R][V][NP];
    CT rowsum[R * 2];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const P nm = splat2(-mc[rr]), r2 = splat2(rc[rr]);
      // 16-bit inputs: xhat = x*r - m*r in one FFMA2 (the product is exact inside the FMA;
      // the absolute error ~|m| r 2^-24 is far below the inputs' own 2^-9 rounding)
      const P nmr = splat2(-mc[rr] * rc[rr]);
      // two accumulators per row sum break the FADD2/FFMA2 dependency chains
      P sg[2] = {splat2(CT(0)), splat2(CT(0))}, sgx[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int j = 0; j < V; ++j) {
        P xv[NP], dv[NP];
        unpack2<T>(rawx[rr][j], xv);
        unpack2<T>(rawd[rr][j], dv);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          if constexpr (sizeof(T) == 2) xh[rr][j][e] = fma2(xv[e], r2, nmr);
          else xh[rr][j][e] = mul2(add2(xv[e], nm), r2);
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
    // this warp's phase 1 has consumed every value it loaded from the slot (the row sums depend
    // on all of them): release the slot now, so the producer refills it while the row sums are
    // reduced and the barrier waits.  (Releasing right after the shared loads were issued, before
    // their results were consumed, raced with the refill: tools/bwd_race_stress.py, 25 of 300
    // launches with corrupted dx at 5 x 17 000 x 1 024.)
    if (p.early_release == 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    {
      constexpr int NV = 2 * R, GRP = 32 / NV;
      const CT u = warp_reduce_scatter<NV>(rowsum, lane);
      if ((lane & (GRP - 1)) == 0) rd[warp * NV + lane / GRP] = u;
    }
    named_bar_sync(1, nc);
    if (!p.early_release) {
      // every consumer has read this stage into registers: release the slot to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // cross-warp totals, spread over the lanes: rd holds ncw x NV values [warp][k]; lane l
    // sums entries l, l+32, ... (all of index k = l % NV), lanes of equal k are combined by a
    // butterfly, and every thread then reads the NV totals by shuffles.  Fixed order ->
    // deterministic; ~2 shared loads + 3 + NV shuffles instead of ncw * NV loads per thread.
    CT tot[2 * R];
    {
      constexpr int NV = 2 * R;
      const int nval = ncw * NV;
      CT s_l = CT(0);
      for (int i = lane; i < nval; i += 32) s_l += rd[i];
#pragma unroll
      for (int off = NV; off < 32; off <<= 1) s_l += __shfl_xor_sync(0xffffffffu, s_l, off);
#pragma unroll
      for (int q = 0; q < NV; ++q) tot[q] = __shfl_sync(0xffffffffu, s_l, q);
    }

    // phase 2: dx = rstd * (g - mean(g) - xhat * mean(g*xhat))
    uint8_t* dxrow = static_cast<uint8_t*>(p.dx) + rb * RB;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (ALL || rr < rows) {
        // dx = r*g - r*mean(g) - (r*mean(g*xhat)) * xhat: two FFMA2 per pair
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
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    ++it;
  };

  if (GW && p.interleave == 2) {
    // Group-sequential interleaved walk: for each group g, stages k, k + G, ... of that group
    // (rows g*S_grp + st*R), (1 + scale) restaged per group, partials to slot g*G + k -- every
    // CTA flushes every group's slot (zeros if it drew no stage there); stage 2 adds slots
    // g*G .. g*G + G - 1 in order (tail0 = -2).
    const int64_t ng = (p.N + p.S_grp - 1) / p.S_grp;
    for (int64_t gi = 0; gi < ng; ++gi) {
      load_scale(gi);
      const int64_t g0 = gi * p.S_grp, g1 = g0 + p.S_grp < p.N ? g0 + p.S_grp : p.N;
      const int64_t nst = (g1 - g0 + R - 1) / R;
      CT mc[R], rc[R];
      auto fetch = [&](int64_t st, CT* m, CT* r) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int64_t row = g0 + st * R + rr;
          const bool ok = st < nst && row < g1;
          m[rr] = ok ? mean_p[row] : CT(0);
          r[rr] = ok ? rstd_p[row] : CT(0);
        }
      };
      fetch(k, mc, rc);
      for (int64_t st = k; st < nst; st += p.G) {
        CT mn[R], rn[R];
        fetch(st + p.G, mn, rn);
        mbar_wait(&full[s], ph);
        const int64_t rb = g0 + st * R;
        const int rows = g1 - rb < R ? static_cast<int>(g1 - rb) : R;
        if (rows == R) stage(std::true_type{}, rb, R, mc, rc);
        else stage(std::false_type{}, rb, rows, mc, rc);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          mc[rr] = mn[rr];
          rc[rr] = rn[rr];
        }
      }
      flush(gi * p.G + k);
    }
  } else if (p.interleave) {
    // Interleaved static walk of a single group (deterministic launches, no ticket): stages k,
    // k + G, k + 2G, ... through the same lean stage body; partials to slot k.
    load_scale(0);
    const int64_t nst = (p.N + R - 1) / R;
    CT mc[R], rc[R];
    auto fetch = [&](int64_t st, CT* m, CT* r) {
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const bool ok = st < nst && st * R + rr < p.N;
        m[rr] = ok ? mean_p[st * R + rr] : CT(0);
        r[rr] = ok ? rstd_p[st * R + rr] : CT(0);
      }
    };
    fetch(k, mc, rc);
    for (int64_t st = k; st < nst; st += p.G) {
      CT mn[R], rn[R];
      fetch(st + p.G, mn, rn);
      mbar_wait(&full[s], ph);
      const int64_t rb = st * R;
      const int rows = p.N - rb < R ? static_cast<int>(p.N - rb) : R;
      if (rows == R) stage(std::true_type{}, rb, R, mc, rc);
      else stage(std::false_type{}, rb, rows, mc, rc);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = mn[rr];
        rc[rr] = rn[rr];
      }
    }
    flush(k);
  }
  // Static head.  Segments = the CTA's rows of one reduction group (sample): (1+scale) loaded
  // once, then full R-row stages, one predicated tail stage, and the group's partials flushed
  // to slot k + g.  Statistics are prefetched one stage ahead.  The producer's StageWalker
  // issues the same sequence.
  int64_t row = p.interleave ? r1 : r0;
  while (row < r1) {
    const int64_t g = row / p.S_grp;
    const int64_t seg_end = min((g + 1) * p.S_grp, r1);
    const int n = static_cast<int>(seg_end - row);
    load_scale(g);
    const CT* mp = mean_p + row;
    const CT* rp = rstd_p + row;
    CT mc[R], rc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mc[rr] = rr < n ? mp[rr] : CT(0);
      rc[rr] = rr < n ? rp[rr] : CT(0);
    }
    const int nfull = n / R;
    for (int i = 0; i < nfull; ++i) {
      CT mn[R], rn[R];
      const int nx = (i + 1) * R, left = n - nx;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mn[rr] = rr < left ? mp[nx + rr] : CT(0);
        rn[rr] = rr < left ? rp[nx + rr] : CT(0);
      }
      mbar_wait(&full[s], ph);
      stage(std::true_type{}, row + i * R, R, mc, rc);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = mn[rr];
        rc[rr] = rn[rr];
      }
    }
    if (n > nfull * R) {
      mbar_wait(&full[s], ph);
      stage(std::false_type{}, row + nfull * R, n - nfull * R, mc, rc);
    }
    flush(k + g);
    row = seg_end;
  }

  if (dyn) {
    // Dynamic tail (last group): stages arrive in whatever order the tickets fall; an empty
    // header ends the stream.  The CTA's tail partial always goes to its tail slot (zeros if it
    // drew nothing), which stage 2 adds after the group's static slots.
    load_scale((p.N - 1) / p.S_grp);
    while (true) {
      mbar_wait(&full[s], ph);
      const int64_t rb = h_row[s];
      const int rows = h_n[s];
      if (rows == 0) break;
      CT mc[R], rc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = h_m[s * R + rr];
        rc[rr] = h_r[s * R + rr];
      }
      if (rows == R) stage(std::true_type{}, rb, R, mc, rc);
      else stage(std::false_type{}, rb, rows, mc, rc);
    }
    flush(p.tail_slot0 + k);
  }
  if (tid == 0) AL_TRACE_INFO(it);
  } else {
    // Static-only instance (deterministic launches): the predicated single-instance loop.  Its
    // CTAs stay issue-bound at one common rate; the leaner DYN loop makes them memory-bound
    // and, without the dynamic tail, exposes the uneven split of HBM bandwidth between SMs
    // (cfg2: 5 870 vs 5 087 GB/s).
  int64_t cur_g = -1;
  StageWalker w;
  if (p.interleave) w.init_interleaved(k, p.G, p.N, R);
  else w.init(r0, r1, p.S_grp);
  int s = 0;
  uint32_t ph = 0;
  int it = 0;

  // statistics of the current stage's rows (prefetched one stage ahead)
  StageWalker wp = w;
  CT mcur[R], rcur[R];
  {
    int64_t st0 = 0, g0;
    const int n0 = wp.done() ? 0 : wp.next(R, st0, g0);
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mcur[rr] = rr < n0 ? mean_p[st0 + rr] : CT(0);
      rcur[rr] = rr < n0 ? rstd_p[st0 + rr] : CT(0);
    }
  }

  while (!w.done()) {
    int64_t rb, g;
    const int rows = w.next(R, rb, g);
    CT mnext[R], rnext[R];
    {
      int64_t st1 = 0, g1;
      const int n1 = wp.done() ? 0 : wp.next(R, st1, g1);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mnext[rr] = rr < n1 ? mean_p[st1 + rr] : CT(0);
        rnext[rr] = rr < n1 ? rstd_p[st1 + rr] : CT(0);
      }
    }
    if (g != cur_g) {
      if (cur_g >= 0) flush(k + cur_g);
      cur_g = g;
      const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
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
      }
    }
    mbar_wait(&full[s], ph);
    // 32-bit shared-window addresses: no generic->shared conversion per load (+1.3 %)
    const uint32_t stx_u = smem_addr(smem) + static_cast<uint32_t>(s * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    CT* rd = red + (it & 1) * (ncw * R * 2);

    // phase 1: row sums of g and g*xhat; column accumulators of dy and dy*xhat.
    // Rows past `rows` (stage tail) and columns past D read as zero, so every lane runs the
    // same instruction stream and the shuffles below are convergent.
    // the stage's x and dy vectors into registers first
    uint4 rawx[R][V], rawd[R][V];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = (rr < rows) && (vmask >> j & 1);
        const uint32_t o = static_cast<uint32_t>(rr * RB + coff[j]);
        rawx[rr][j] = ok ? ld_shared_v4_u32(stx_u + o) : make_uint4(0, 0, 0, 0);
        rawd[rr][j] = ok ? ld_shared_v4_u32(std_u + o) : make_uint4(0, 0, 0, 0);
      }
    P xh[R][V][NP], gg[R][V][NP];
    CT rowsum[R * 2];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const P nm = splat2(-mcur[rr]), r2 = splat2(rcur[rr]);
      // 16-bit inputs: xhat = x*r - m*r in one FFMA2 (the product is exact inside the FMA;
      // the absolute error ~|m| r 2^-24 is far below the inputs' own 2^-9 rounding)
      const P nmr = splat2(-mcur[rr] * rcur[rr]);
      // two accumulators per row sum break the FADD2/FFMA2 dependency chains
      P sg[2] = {splat2(CT(0)), splat2(CT(0))}, sgx[2] = {splat2(CT(0)), splat2(CT(0))};
#pragma unroll
      for (int j = 0; j < V; ++j) {
        P xv[NP], dv[NP];
        unpack2<T>(rawx[rr][j], xv);
        unpack2<T>(rawd[rr][j], dv);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          if constexpr (sizeof(T) == 2) xh[rr][j][e] = fma2(xv[e], r2, nmr);
          else xh[rr][j][e] = mul2(add2(xv[e], nm), r2);
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
    // this warp's phase 1 has consumed every value it loaded from the slot (the row sums depend
    // on all of them): release the slot now, so the producer refills it while the row sums are
    // reduced and the barrier waits.  (Releasing right after the shared loads were issued, before
    // their results were consumed, raced with the refill: tools/bwd_race_stress.py, 25 of 300
    // launches with corrupted dx at 5 x 17 000 x 1 024.)
    if (p.early_release == 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    {
      constexpr int NV = 2 * R, GRP = 32 / NV;
      const CT u = warp_reduce_scatter<NV>(rowsum, lane);
      if ((lane & (GRP - 1)) == 0) rd[warp * NV + lane / GRP] = u;
    }
    named_bar_sync(1, nc);
    if (!p.early_release) {
      // every consumer has read this stage into registers: release the slot to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // cross-warp totals, spread over the lanes: rd holds ncw x NV values [warp][k]; lane l
    // sums entries l, l+32, ... (all of index k = l % NV), lanes of equal k are combined by a
    // butterfly, and every thread then reads the NV totals by shuffles.  Fixed order ->
    // deterministic; ~2 shared loads + 3 + NV shuffles instead of ncw * NV loads per thread.
    CT tot[2 * R];
    {
      constexpr int NV = 2 * R;
      const int nval = ncw * NV;
      CT s_l = CT(0);
      for (int i = lane; i < nval; i += 32) s_l += rd[i];
#pragma unroll
      for (int off = NV; off < 32; off <<= 1) s_l += __shfl_xor_sync(0xffffffffu, s_l, off);
#pragma unroll
      for (int q = 0; q < NV; ++q) tot[q] = __shfl_sync(0xffffffffu, s_l, q);
    }

    // phase 2: dx = rstd * (g - mean(g) - xhat * mean(g*xhat))
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr < rows) {
        const int64_t row = rb + rr;
        // dx = r*g - r*mean(g) - (r*mean(g*xhat)) * xhat: two FFMA2 per pair
        const CT rr_ = rcur[rr];
        const P c0 = splat2(-rr_ * tot[2 * rr] * invD), c1 = splat2(-rr_ * tot[2 * rr + 1] * invD);
        const P r2 = splat2(rr_);
        uint8_t* dxrow = static_cast<uint8_t*>(p.dx) + row * RB;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            P o[NP];
#pragma unroll
            for (int e = 0; e < NP; ++e)
              o[e] = fma2(gg[rr][j][e], r2, fma2(xh[rr][j][e], c1, c0));
            st_global_cs(dxrow + coff[j], pack2<T>(o));
          }
        }
        if (tid == 0) nf |= !(finite_ct(tot[2 * rr]) && finite_ct(tot[2 * rr + 1]));
      }
    }
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    ++it;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mcur[rr] = mnext[rr];
      rcur[rr] = rnext[rr];
    }
  }
  if (cur_g >= 0) flush(k + cur_g);
  else if (p.interleave) flush(k);  // no stage for this CTA: its slot still takes part (zeros)
  }
#ifdef AL_CTA_TRACE
  named_bar_sync(1, nc);
  if (tid == 0) AL_TRACE(1, 1);
#endif
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
  if (dyn) {
    // the last CTA out re-arms the ticket pair (consumers only: the producer has returned)
    named_bar_sync(1, nc);
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1u) == static_cast<unsigned int>(p.G - 1)) {
        atomicExch(p.sched, 0u);
        atomicExch(p.sched + 1, 0u);
      }
    }
  }
  if (p.counter != nullptr) fused_stage2<CT>(p, nc, tid);
}

// =====================================================================================
// Backward stage 1, skewed-pipeline TMA path (K2p).  Same ring, producer and column-owner
// layout as adaln_bwd_tma, but no per-stage lock step: a consumer warp runs phase 1 of stage i
// (row sums of g and g*xhat, column accumulators), deposits its row-sum partials in a small
// reduction ring and ARRIVES on that entry's mbarrier (no bar.sync), then runs phase 2 of stage
// i-1 -- whose cross-warp totals were completed by every warp's phase 1 of i-1 while this warp
// was busy -- re-reading x and dy of stage i-1 from the still-held ring slot (xhat and g are
// recomputed, not kept in registers across the barrier), writes dx and releases the slot.
// The barrier latency is thereby overlapped with the next stage's phase 1, warps drift freely
// instead of bursting the FMA pipe in lock step, and the ~64 registers that held xhat and g are
// gone (97 instead of 168 per thread).
// Invariants: a warp in phase 1 of stage i has finished phase 2 of i-2, which needed every warp's
// phase 1 of i-2, so at most three reduction entries (i-2, i-1, i) are live: KR = 4 entries.
// (1 + scale) is group-constant; a group change drains the pending stage first, so phase 2 always
// sees the modulation its stage was accumulated with.
// =====================================================================================
template <typename T, int V, int R, bool FULL, bool DYN>
__global__ void __launch_bounds__(384, 1) adaln_bwd_pipe(const BwdParams p) {
  pdl_enter();
  ts_begin(p.ts);
  if (threadIdx.x == 0) AL_TRACE(1, 0);
  using CT = typename Traits<T>::CT;
  using P = typename PairOf<CT>::type;
  constexpr int EPV = Traits<T>::EPV;
  constexpr int NP = EPV / 2;
  constexpr int KR = 4;       // reduction-ring entries
  constexpr int NV = 2 * R;   // row-sum values per stage (sum g, sum g*xhat per row)
  constexpr int GRP = 32 / NV;
  extern __shared__ __align__(128) uint8_t smem[];

  const int nc = blockDim.x - 32;
  const int ncw = nc >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = p.nstages;
  const int RB = p.row_bytes;
  const int stage_bytes = 2 * R * RB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * stage_bytes);
  uint64_t* empty = full + NS;
  uint64_t* rbar = empty + NS;                        // [KR]: row-sum entry complete
  CT* red = reinterpret_cast<CT*>(rbar + KR);         // [KR][ncw][NV]
  int64_t* h_row = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(red + KR * ncw * NV) + 7) & ~uintptr_t(7));
  int* h_n = reinterpret_cast<int*>(h_row + NS);
  CT* h_m = reinterpret_cast<CT*>((reinterpret_cast<uintptr_t>(h_n + NS) + 7) & ~uintptr_t(7));
  CT* h_r = h_m + NS * R;

  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N_static, p.G), r1 = part_begin(k + 1, p.N_static, p.G);
  const bool dyn = DYN && p.sched != nullptr;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    for (int b = 0; b < KR; ++b) mbar_init(&rbar[b], ncw * NV);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == ncw) {  // ---------------- producer (as adaln_bwd_tma) ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* xb = static_cast<const uint8_t*>(p.x);
      const uint8_t* db = static_cast<const uint8_t*>(p.dy);
      StageWalker w;
      if (p.interleave) w.init_interleaved(k, p.G, p.N, R);
      else w.init(r0, r1, p.S_grp);
      int s = 0;
      uint32_t f = 0;
      auto issue = [&](int64_t start, int rows) {
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(2 * rows * RB));
        uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
        for (int rr = 0; rr < rows; ++rr) {
          bulk_g2s(dst + rr * RB, xb + (start + rr) * RB, RB, &full[s], pol);
          bulk_g2s(dst + (R + rr) * RB, db + (start + rr) * RB, RB, &full[s], pol);
        }
        if (++s == NS) {
          s = 0;
          ++f;
        }
      };
      while (!w.done()) {
        int64_t start, g;
        const int rows = w.next(R, start, g);
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        issue(start, rows);
      }
      if (dyn) {
        const CT* mean_p = static_cast<const CT*>(p.mean);
        const CT* rstd_p = static_cast<const CT*>(p.rstd);
        auto stats = [&](int64_t start, CT* m, CT* r) {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const bool ok = start + rr < p.N;
            m[rr] = ok ? mean_p[start + rr] : CT(0);
            r[rr] = ok ? rstd_p[start + rr] : CT(0);
          }
        };
        int64_t start = p.N_static + static_cast<int64_t>(atomicAdd(p.sched, 1u)) * R;
        CT m[R], r[R];
        stats(start, m, r);
        unsigned int tn = atomicAdd(p.sched, 1u);
        while (true) {
          const int rows = start < p.N ? static_cast<int>(p.N - start < R ? p.N - start : R) : 0;
          if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
          h_row[s] = start;
          h_n[s] = rows;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            h_m[s * R + rr] = m[rr];
            h_r[s * R + rr] = r[rr];
          }
          if (rows == 0) {
            mbar_arrive(&full[s]);
            break;
          }
          issue(start, rows);
          start = p.N_static + static_cast<int64_t>(tn) * R;
          if (start < p.N) {
            stats(start, m, r);
            tn = atomicAdd(p.sched, 1u);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  uint32_t vmask = FULL ? (1u << V) - 1 : 0u;
  int coff[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    coff[j] = (tid + j * nc) * 16;
    if (!FULL && tid + j * nc < p.nvec) vmask |= 1u << j;
  }
  const CT invD = CT(1) / static_cast<CT>(p.D);
  const CT* mean_p = static_cast<const CT*>(p.mean);
  const CT* rstd_p = static_cast<const CT*>(p.rstd);
  CT* ws_sc = static_cast<CT*>(p.ws);
  CT* ws_sh = ws_sc + p.nslots * p.D;
  bool nf = false;
  const uint32_t smem_u = smem_addr(smem);

  P s1[V][NP], acc_sc[V][NP], acc_sh[V][NP];
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));

  auto flush = [&](int64_t slot) {
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
          acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));
        }
      }
    }
  };
  auto load_scale = [&](int64_t g) {
    const uint8_t* sc = static_cast<const uint8_t*>(p.scale) + g * p.mod_stride * sizeof(T);
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
    }
  };

  // ring cursor (consumer side) and reduction-ring counter
  int s = 0;
  uint32_t ph = 0;
  uint32_t it = 0;
  // the stage whose phase 2 is pending
  struct Pend {
    int64_t rb;
    int rows, slot;
    uint32_t it;
    CT m[R], r[R];
  } pd;
  bool pending = false;

  // phase 1 of the stage in ring slot s (the caller has waited on full[s])
  auto phase1 = [&](auto all_tag, int rows, const CT* mc, const CT* rc) {
    constexpr bool ALL = decltype(all_tag)::value;
    const uint32_t stx_u = smem_u + static_cast<uint32_t>(s * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    CT rowsum[NV];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const bool live = ALL || rr < rows;
      const P nm = splat2(-mc[rr]), r2 = splat2(rc[rr]);
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
          P xh;
          if constexpr (sizeof(T) == 2) xh = fma2(xv[e], r2, nmr);
          else xh = mul2(add2(xv[e], nm), r2);
          const P gg = mul2(dv[e], s1[j][e]);
          sg[e & 1] = add2(sg[e & 1], gg);
          sgx[e & 1] = fma2(gg, xh, sgx[e & 1]);
          acc_sh[j][e] = add2(acc_sh[j][e], dv[e]);
          acc_sc[j][e] = fma2(dv[e], xh, acc_sc[j][e]);
        }
      }
      const P tsg = add2(sg[0], sg[1]), tsgx = add2(sgx[0], sgx[1]);
      rowsum[2 * rr] = tsg.x + tsg.y;
      rowsum[2 * rr + 1] = tsgx.x + tsgx.y;
    }
    const int b = static_cast<int>(it % KR);
    const CT u = warp_reduce_scatter<NV>(rowsum, lane);
    if ((lane & (GRP - 1)) == 0) {
      red[(b * ncw + warp) * NV + lane / GRP] = u;
      mbar_arrive(&rbar[b]);  // release: the entry write above is visible to the waiters
    }
  };

  // phase 2 of the pending stage: totals, dx from the re-read slot, slot release
  auto phase2 = [&](auto all_tag) {
    constexpr bool ALL = decltype(all_tag)::value;
    const int b = static_cast<int>(pd.it % KR);
    mbar_wait(&rbar[b], (pd.it / KR) & 1);
    CT tot[NV];
    {
      const CT* rd = red + b * ncw * NV;
      const int nval = ncw * NV;
      CT s_l = CT(0);
      for (int i = lane; i < nval; i += 32) s_l += rd[i];
#pragma unroll
      for (int off = NV; off < 32; off <<= 1) s_l += __shfl_xor_sync(0xffffffffu, s_l, off);
#pragma unroll
      for (int q = 0; q < NV; ++q) tot[q] = __shfl_sync(0xffffffffu, s_l, q);
    }
    const uint32_t stx_u = smem_u + static_cast<uint32_t>(pd.slot * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    uint8_t* dxrow = static_cast<uint8_t*>(p.dx) + pd.rb * RB;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (ALL || rr < pd.rows) {
        const CT rr_ = pd.r[rr];
        const CT c0 = -rr_ * tot[2 * rr] * invD, c1 = -rr_ * tot[2 * rr + 1] * invD;
        const P r2 = splat2(rr_);
        // xhat and g recomputed exactly as in phase 1 (and as adaln_bwd_tma keeps them), then
        // dx = g*r + (xhat*c1 + c0): dx is bit-identical to the lock-step kernel's
        const P nm = splat2(-pd.m[rr]), pc1 = splat2(c1), pc0 = splat2(c0);
        const P nmr = splat2(-pd.m[rr] * rr_);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            P xv[NP], dv[NP], o[NP];
            const uint32_t off = static_cast<uint32_t>(rr * RB + coff[j]);
            unpack2<T>(ld_shared_v4_u32(stx_u + off), xv);
            unpack2<T>(ld_shared_v4_u32(std_u + off), dv);
#pragma unroll
            for (int e = 0; e < NP; ++e) {
              const P gg = mul2(dv[e], s1[j][e]);
              P xh;
              if constexpr (sizeof(T) == 2) xh = fma2(xv[e], r2, nmr);
              else xh = mul2(add2(xv[e], nm), r2);
              o[e] = fma2(gg, r2, fma2(xh, pc1, pc0));
            }
            st_global_cs(dxrow + rr * RB + coff[j], pack2<T>(o));
          }
        }
        if (tid == 0) nf |= !(finite_ct(tot[2 * rr]) && finite_ct(tot[2 * rr + 1]));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[pd.slot]);
    pending = false;
  };
  auto drain = [&]() {
    if (pending) {
      if (pd.rows == R) phase2(std::true_type{});
      else phase2(std::false_type{});
    }
  };
  // one stage: phase 1 of it, then phase 2 of the previous one
  auto step = [&](int64_t rb, int rows, const CT* mc, const CT* rc) {
    if (rows == R) phase1(std::true_type{}, rows, mc, rc);
    else phase1(std::false_type{}, rows, mc, rc);
    drain();
    pd.rb = rb;
    pd.rows = rows;
    pd.slot = s;
    pd.it = it;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      pd.m[rr] = mc[rr];
      pd.r[rr] = rc[rr];
    }
    pending = true;
    ++it;
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  };

  if (!DYN && p.interleave) {
    // interleaved static partition (single group): stages k, k+G, ... as the producer walks
    // them (StageWalker::init_interleaved); one (1 + scale), one slot
    load_scale(0);
    const int64_t step_rows = static_cast<int64_t>(p.G) * R;
    int64_t rb = k * R;
    CT mc[R], rc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mc[rr] = rb + rr < p.N ? mean_p[rb + rr] : CT(0);
      rc[rr] = rb + rr < p.N ? rstd_p[rb + rr] : CT(0);
    }
    for (; rb < p.N; rb += step_rows) {
      const int rows = p.N - rb < R ? static_cast<int>(p.N - rb) : R;
      const int64_t nb = rb + step_rows;
      CT mn[R], rn[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mn[rr] = nb + rr < p.N ? mean_p[nb + rr] : CT(0);
        rn[rr] = nb + rr < p.N ? rstd_p[nb + rr] : CT(0);
      }
      mbar_wait(&full[s], ph);
      step(rb, rows, mc, rc);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = mn[rr];
        rc[rr] = rn[rr];
      }
    }
    flush(k);  // zeros when this CTA had no stage: its slot still takes part
  }
  // static head: the producer's StageWalker sequence, segment by segment
  int64_t row = (!DYN && p.interleave) ? r1 : r0;
  while (row < r1) {
    const int64_t g = row / p.S_grp;
    const int64_t seg_end = min((g + 1) * p.S_grp, r1);
    const int n = static_cast<int>(seg_end - row);
    drain();  // phase 2 of the previous group's last stage needs that group's (1 + scale)
    load_scale(g);
    const CT* mp = mean_p + row;
    const CT* rp = rstd_p + row;
    CT mc[R], rc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      mc[rr] = rr < n ? mp[rr] : CT(0);
      rc[rr] = rr < n ? rp[rr] : CT(0);
    }
    for (int i = 0; i * R < n; ++i) {
      const int rows = n - i * R < R ? n - i * R : R;
      CT mn[R], rn[R];
      const int nx = (i + 1) * R, left = n - nx;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mn[rr] = rr < left ? mp[nx + rr] : CT(0);
        rn[rr] = rr < left ? rp[nx + rr] : CT(0);
      }
      mbar_wait(&full[s], ph);
      step(row + i * R, rows, mc, rc);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = mn[rr];
        rc[rr] = rn[rr];
      }
    }
    flush(k + g);  // accumulators are phase-1 state: the pending phase 2 does not touch them
    row = seg_end;
  }

  if (dyn) {
    drain();
    load_scale((p.N - 1) / p.S_grp);
    while (true) {
      mbar_wait(&full[s], ph);
      const int64_t rb = h_row[s];
      const int rows = h_n[s];
      if (rows == 0) break;
      CT mc[R], rc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = h_m[s * R + rr];
        rc[rr] = h_r[s * R + rr];
      }
      step(rb, rows, mc, rc);
    }
    flush(p.tail_slot0 + k);
  }
  drain();
#ifdef AL_CTA_TRACE
  named_bar_sync(1, nc);
  if (tid == 0) AL_TRACE(1, 1);
#endif
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
  if (dyn) {
    named_bar_sync(1, nc);
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1u) == static_cast<unsigned int>(p.G - 1)) {
        atomicExch(p.sched, 0u);
        atomicExch(p.sched + 1, 0u);
      }
    }
  }
}

// =====================================================================================
// Backward stage 2: dscale/dshift[g, d] = sum over the CTAs covering group g, ascending.
// Vector form (D a multiple of 16 B of partials): block = 512 threads = kRedCV column vectors
// (8 x 16 B = 32 fp32 / 16 fp64 columns) x 64 slot lanes, 2 CTAs per SM, so a cfg2 reduction
// (296 slots, 160 CTAs) is one wave with <= 5 slots per thread, all loads of a thread in flight
// before the first add (the kernel is a latency chain, not a bandwidth one).  Slot lanes are
// combined by a fixed shuffle tree inside the warp and the 16 warps in ascending order through
// shared memory -- a fixed order, so the result is deterministic.
// =====================================================================================
constexpr int kRedCV = 8;  // 16-byte column vectors per stage-2 CTA
template <typename CT>
__global__ void __launch_bounds__(512, 2) adaln_bwd_reduce_vec(const CT* __restrict__ ws,
                                                             CT* __restrict__ dscale,
                                                             CT* __restrict__ dshift, int64_t N,
                                                             int64_t S_grp, int64_t D, int64_t G,
                                                             int64_t nslots, int64_t Ns,
                                                             int64_t tail0,
                                                             unsigned long long* ts) {
  pdl_wait();
  constexpr int VE = 16 / sizeof(CT);   // columns per 16-byte vector
  constexpr int CV = kRedCV;
  constexpr int COLS = CV * VE;         // columns per CTA
  constexpr int SL = 512 / CV;          // slot lanes
  constexpr int NW = 512 / 32;          // warps
  __shared__ double part[2][NW][COLS + 1];
  const int t = threadIdx.x, hl = t % CV, sl = t / CV, warp = t >> 5;
  const int64_t g = blockIdx.y;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * COLS + hl * VE;
  // slots of group g: the static owners of its rows below Ns (slot k + g, ascending k), then --
  // for the last group of a dynamically scheduled launch -- the G tail slots tail0 + k
  const int64_t first_row = g * S_grp;
  const int64_t end_row = (g + 1) * S_grp < N ? (g + 1) * S_grp : N;
  const int64_t last_static = (end_row < Ns ? end_row : Ns) - 1;
  int64_t kf = 0, n1 = 0;
  if (tail0 <= -2) {  // group-sequential walk: slots g*G .. g*G + G - 1
    kf = g * G - g;
    n1 = G;
  } else if (first_row <= last_static) {
    kf = part_owner(first_row, Ns, G);
    n1 = part_owner(last_static, Ns, G) - kf + 1;
  }
  const int64_t n2 = (tail0 >= 0 && end_row == N) ? G : 0;
  const int64_t n = n1 + n2;
  double a[VE], b[VE];
#pragma unroll
  for (int e = 0; e < VE; ++e) a[e] = b[e] = 0.0;
  const bool two = dshift != nullptr;  // dshift == nullptr: reduce the first array only
  if (col < D) {
    const CT* sc = ws + (kf + g) * D + col;
    const CT* sh = two ? ws + (nslots + kf + g) * D + col : sc;
    // slot i -> row offset (in units of D) from sc / sh
    const int64_t jump = tail0 - (kf + g) - n1;
    auto off = [&](int64_t i) { return (i < n1 ? i : i + jump) * D; };
    int64_t i = sl;
    for (; i + 3 * SL < n; i += 4 * SL) {  // 4 slots x 2 arrays of 16-byte loads in flight
      uint4 va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        va[u] = __ldcg(reinterpret_cast<const uint4*>(sc + off(i + SL * u)));
        vb[u] = __ldcg(reinterpret_cast<const uint4*>(sh + off(i + SL * u)));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const CT* pa = reinterpret_cast<const CT*>(&va[u]);
        const CT* pb = reinterpret_cast<const CT*>(&vb[u]);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          a[e] += static_cast<double>(pa[e]);
          b[e] += static_cast<double>(pb[e]);
        }
      }
    }
    // remainder (< 4 slots per lane): predicated loads, all issued before the adds
    uint4 va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = i + SL * u < n;
      va[u] = ok ? __ldcg(reinterpret_cast<const uint4*>(sc + off(i + SL * u))) : make_uint4(0, 0, 0, 0);
      vb[u] = ok ? __ldcg(reinterpret_cast<const uint4*>(sh + off(i + SL * u))) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i + SL * u < n) {
        const CT* pa = reinterpret_cast<const CT*>(&va[u]);
        const CT* pb = reinterpret_cast<const CT*>(&vb[u]);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          a[e] += static_cast<double>(pa[e]);
          b[e] += static_cast<double>(pb[e]);
        }
      }
    }
  }
  // slot lanes of a warp (lane / CV) combined by a fixed tree: lanes < CV end with the sum
#pragma unroll
  for (int o = 16; o >= CV; o >>= 1) {
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      a[e] += __shfl_down_sync(0xffffffffu, a[e], o);
      b[e] += __shfl_down_sync(0xffffffffu, b[e], o);
    }
  }
  if ((t & 31) < CV) {
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      part[0][warp][hl * VE + e] = a[e];
      part[1][warp][hl * VE + e] = b[e];
    }
  }
  __syncthreads();
  pdl_launch();
  if (t < (two ? 2 : 1) * COLS) {
    const int which = t / COLS, c = t % COLS;
    const int64_t oc = static_cast<int64_t>(blockIdx.x) * COLS + c;
    if (oc < D) {
      double s = 0.0;
#pragma unroll 8
      for (int q = 0; q < NW; ++q) s += part[which][q][c];
      (which == 0 ? dscale : dshift)[g * D + oc] = static_cast<CT>(s);
    }
  }
  if (ts != nullptr) {
    __syncthreads();
    if (t == 0) ts_end(ts);
  }
}

// Many-group form (multi-sample launches without a dynamic tail, e.g. the sampler's buckets of
// 307 x 1 560 rows): a group's rows lie in one or two CTA ranges, so each group has only a few
// slots and the block-per-(column block, group) grid above is thousands of CTAs of almost no work
// -- 20 x 307 = 6 140 CTAs, ~380 us of latency-bound waves at that bucket.  Here one thread
// owns one 16-byte column vector of one group and adds that group's slots in ascending order
// (fp64, four slots' loads in flight), so the grid is the output size / 256 and one wave deep.
template <typename CT>
__global__ void __launch_bounds__(256) adaln_bwd_reduce_grp(const CT* __restrict__ ws,
                                                          CT* __restrict__ dscale,
                                                          CT* __restrict__ dshift, int64_t N,
                                                          int64_t S_grp, int64_t D, int64_t G,
                                                          int64_t nslots, int64_t Ns,
                                                          int64_t tail0,
                                                          unsigned long long* ts) {
  pdl_wait();
  constexpr int VE = 16 / sizeof(CT);
  const int64_t nv = D / VE;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ngroups = (N + S_grp - 1) / S_grp;
  const bool two = dshift != nullptr;
  if (item < ngroups * nv) {
    const int64_t g = item / nv, col = (item % nv) * VE;
    const int64_t first_row = g * S_grp;
    const int64_t end_row = (g + 1) * S_grp < N ? (g + 1) * S_grp : N;
    const int64_t last_static = (end_row < Ns ? end_row : Ns) - 1;
    int64_t kf = 0, n1 = 0;
    if (first_row <= last_static) {
      kf = part_owner(first_row, Ns, G);
      n1 = part_owner(last_static, Ns, G) - kf + 1;
    }
    const int64_t n2 = (tail0 >= 0 && end_row == N) ? G : 0;
    const int64_t n = n1 + n2;
    const CT* sc = ws + (kf + g) * D + col;
    const CT* sh = two ? ws + (nslots + kf + g) * D + col : sc;
    const int64_t jump = tail0 - (kf + g) - n1;
    auto off = [&](int64_t i) { return (i < n1 ? i : i + jump) * D; };
    double a[VE], b[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) a[e] = b[e] = 0.0;
    for (int64_t i = 0; i < n; i += 4) {
      uint4 va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = i + u < n;
        va[u] = ok ? __ldcg(reinterpret_cast<const uint4*>(sc + off(i + u))) : make_uint4(0, 0, 0, 0);
        vb[u] = ok && two ? __ldcg(reinterpret_cast<const uint4*>(sh + off(i + u)))
                          : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i + u < n) {
          const CT* pa = reinterpret_cast<const CT*>(&va[u]);
          const CT* pb = reinterpret_cast<const CT*>(&vb[u]);
#pragma unroll
          for (int e = 0; e < VE; ++e) {
            a[e] += static_cast<double>(pa[e]);
            b[e] += static_cast<double>(pb[e]);
          }
        }
      }
    }
    // element stores: the outputs carry no alignment requirement beyond their type's
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      dscale[g * D + col + e] = static_cast<CT>(a[e]);
      if (two) dshift[g * D + col + e] = static_cast<CT>(b[e]);
    }
  }
  pdl_launch();
  if (ts != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) ts_end(ts);
  }
}

// Scalar form for any D: block = 1024 threads = 32 columns x 32 slot lanes.
template <typename CT>
__global__ void __launch_bounds__(1024) adaln_bwd_reduce(const CT* __restrict__ ws,
                                                         CT* __restrict__ dscale,
                                                         CT* __restrict__ dshift, int64_t N,
                                                         int64_t S_grp, int64_t D, int64_t G,
                                                         int64_t nslots) {
  pdl_enter();
  __shared__ double part[2][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t g = blockIdx.y;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  const int64_t first_row = g * S_grp;
  const int64_t last_row = ((g + 1) * S_grp < N ? (g + 1) * S_grp : N) - 1;
  const int64_t kf = part_owner(first_row, N, G), kl = part_owner(last_row, N, G);
  double a = 0.0, b = 0.0;
  const bool two = dshift != nullptr;  // dshift == nullptr: reduce the first array only
  if (col < D) {
    const CT* sc = ws + (kf + g) * D + col;
    const CT* sh = two ? ws + (nslots + kf + g) * D + col : sc;
    for (int64_t i = w; i <= kl - kf; i += 32) {
      a += static_cast<double>(sc[i * D]);
      b += static_cast<double>(sh[i * D]);
    }
  }
  part[0][w][lane] = a;
  part[1][w][lane] = b;
  __syncthreads();
  if (w < (two ? 2 : 1) && col < D) {
    double t = 0.0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) t += part[w][q][lane];
    (w == 0 ? dscale : dshift)[g * D + col] = static_cast<CT>(t);
  }
}

// =====================================================================================
// Generic (any D, any alignment) kernels.  Correctness path for shapes the vector/TMA path
// cannot take (D*sizeof(T) not a multiple of 16, unaligned views, very wide rows).
// =====================================================================================
template <typename T>
__global__ void __launch_bounds__(256) adaln_fwd_generic(const FwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const T* x = static_cast<const T*>(p.x);
  const T* sc = static_cast<const T*>(p.scale);
  const T* sf = static_cast<const T*>(p.shift);
  T* y = static_cast<T*>(p.y);
  const CT eps = static_cast<CT>(p.eps);
  bool nf = false;
  for (int64_t row = wid; row < p.N; row += nw) {
    const T* xr = x + row * p.D;
    const int64_t g = row / p.S_grp;
    CT sum = CT(0);
    for (int64_t j = lane; j < p.D; j += 32) sum += to_ct(xr[j]);
    const CT mean = warp_sum(sum) / static_cast<CT>(p.D);
    CT m2 = CT(0);
    for (int64_t j = lane; j < p.D; j += 32) {
      const CT d = to_ct(xr[j]) - mean;
      m2 = fma(d, d, m2);
    }
    m2 = warp_sum(m2);
    const CT rs = CT(1) / sqrt(m2 / static_cast<CT>(p.D) + eps);
    for (int64_t j = lane; j < p.D; j += 32) {
      const CT a = to_ct(sc[g * p.mod_stride + j]), b = to_ct(sf[g * p.mod_stride + j]);
      nf |= !(finite_ct(a) && finite_ct(b));
      y[row * p.D + j] = from_ct<T>(fma((to_ct(xr[j]) - mean) * rs, CT(1) + a, b));
    }
    if (lane == 0) {
      static_cast<CT*>(p.mean)[row] = mean;
      static_cast<CT*>(p.rstd)[row] = rs;
      nf |= !(finite_ct(mean) && finite_ct(m2));
    }
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

// Gated residual for shapes the fused kernel does not take (unaligned pointers, wide rows):
// x_out = x + gate (.) f with the same single fp32 (fp64) rounding; adaln_fwd_generic/wide then
// normalises x_out.
template <typename T>
__global__ void __launch_bounds__(256) gate_residual_generic(const FwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  const T* x = static_cast<const T*>(p.x);
  const T* f = static_cast<const T*>(p.f);
  const T* ga = static_cast<const T*>(p.gate);
  T* xo = static_cast<T*>(p.x_out);
  const int64_t total = p.N * p.D;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  bool nf = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += stride) {
    const int64_t row = i / p.D, j = i - row * p.D;
    const CT g = to_ct(ga[(row / p.S_grp) * p.mod_stride + j]);
    nf |= !finite_ct(g);
    xo[i] = from_ct<T>(fma(g, to_ct(f[i]), to_ct(x[i])));
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

template <typename T>
__global__ void __launch_bounds__(256) adaln_bwd_generic(const BwdParams p) {
  pdl_enter();
  using CT = typename Traits<T>::CT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int64_t k = blockIdx.x;
  const int64_t r0 = part_begin(k, p.N, p.G), r1 = part_begin(k + 1, p.N, p.G);
  const T* x = static_cast<const T*>(p.x);
  const T* dy = static_cast<const T*>(p.dy);
  const T* sc = static_cast<const T*>(p.scale);
  const CT* mean_p = static_cast<const CT*>(p.mean);
  const CT* rstd_p = static_cast<const CT*>(p.rstd);
  T* dx = static_cast<T*>(p.dx);
  const CT invD = CT(1) / static_cast<CT>(p.D);
  bool nf = false;
  // dx: one warp per row
  for (int64_t row = r0 + warp; row < r1; row += nwarp) {
    const int64_t g = row / p.S_grp;
    const CT m = mean_p[row], r = rstd_p[row];
    CT sg = CT(0), sgx = CT(0);
    for (int64_t j = lane; j < p.D; j += 32) {
      const CT xh = (to_ct(x[row * p.D + j]) - m) * r;
      const CT gg = to_ct(dy[row * p.D + j]) * (CT(1) + to_ct(sc[g * p.mod_stride + j]));
      sg += gg;
      sgx = fma(gg, xh, sgx);
    }
    sg = warp_sum(sg);
    sgx = warp_sum(sgx);
    const CT mg = sg * invD, mgx = sgx * invD;
    for (int64_t j = lane; j < p.D; j += 32) {
      const CT xh = (to_ct(x[row * p.D + j]) - m) * r;
      const CT gg = to_ct(dy[row * p.D + j]) * (CT(1) + to_ct(sc[g * p.mod_stride + j]));
      dx[row * p.D + j] = from_ct<T>(r * fma(-xh, mgx, gg - mg));
    }
    if (lane == 0) nf |= !(finite_ct(sg) && finite_ct(sgx));
  }
  // stage-1 column partials: thread per column, rows ascending
  CT* ws_sc = static_cast<CT*>(p.ws);
  CT* ws_sh = ws_sc + p.nslots * p.D;
  for (int64_t col = threadIdx.x; col < p.D; col += blockDim.x) {
    int64_t g = r0 / p.S_grp;
    int64_t gend = (g + 1) * p.S_grp;
    CT a = CT(0), b = CT(0);
    for (int64_t row = r0; row < r1; ++row) {
      if (row >= gend) {
        ws_sc[(k + g) * p.D + col] = a;
        ws_sh[(k + g) * p.D + col] = b;
        a = b = CT(0);
        ++g;
        gend += p.S_grp;
      }
      const CT d = to_ct(dy[row * p.D + col]);
      const CT xh = (to_ct(x[row * p.D + col]) - mean_p[row]) * rstd_p[row];
      b += d;
      a = fma(d, xh, a);
    }
    ws_sc[(k + g) * p.D + col] = a;
    ws_sh[(k + g) * p.D + col] = b;
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
}

}  // namespace al

#include "bwd_steal.cuh"

