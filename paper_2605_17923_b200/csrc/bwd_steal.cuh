// bwd_steal.cuh -- backward stage 1 with DETERMINISTIC dynamic load balancing (K2s).
//
// Why: once the backward is memory-bound, HBM bandwidth is not shared evenly between SMs, so a
// static row partition waits for the slowest SM (cfg2: 173 us static vs 157 us with a dynamic
// tail).  The round-1 dynamic tail handed rows to whichever CTA was free and summed the tail's
// dscale/dshift per CTA, so their fp32 rounding depended on the (timing-dependent) assignment.
//
// Here every CTA k still OWNS a fixed row range (the static partition), and the last segment
// of that range is cut into fixed chunks of C rows.  The owner's partial sums for its last
// segment are accumulated chunk by chunk in a fixed order,
//        slot[k] = ((pre + c_0) + c_1) + ... + c_{nch-1}          (per column, fp32)
// where c_j is chunk j's column sums computed in FRESH accumulators, rows in order.  A CTA that
// finishes its own range may steal chunks from the END of a slower owner's range (owner takes
// chunks from the head, thieves from the tail of a per-owner [head, tail) claim word); it
// computes c_j with exactly the same per-thread arithmetic (thread t owns the same columns in
// every CTA), writes it to a pool slot and publishes it with an epoch-tagged flag.  The owner,
// after its own chunks, adds the stolen c_j in chunk order.  The sums therefore do not depend
// on who computed which chunk: dscale/dshift are bit-identical run to run, while the tail of
// the kernel is balanced at chunk granularity (C = 32 rows by default).
//
// Selected automatically (adaln_capi.cu bwd_steal_mode) for multi-sample launches: there the
// alternative is a static contiguous partition, and stealing measured 6 % faster (307 x 1 560
// ... 15 x 14 040 rows, profiles/r2_steal_buckets_ab.jsonl) and bit-reproducible.  Single-sample
// launches keep the dynamic tail / interleaved static walk of adaln_bwd_tma.
//
// Protocol state lives in a per-stream slot of device memory (StealSlot, zero at module load):
//  * epoch: each launch uses E = epoch + 1 (read by every CTA at entry; the previous launch on
//    the stream has completed -- griddepcontrol.wait -- and its last CTA stored its epoch);
//  * word[k] = (E << 32) | (head << 16) | tail, written by owner k at entry; a word carrying an
//    older epoch means "owner not started yet" to the thieves;
//  * flag[k][j] = E once chunk j of owner k has been published (pidx[k][j] = its pool slot);
//  * pool / done: pool slots handed out / CTAs finished in this launch, reset by the last CTA.
// Owners only wait for chunks a thief has already claimed; thieves never wait: no deadlock.
//
// Producer: a whole warp (lane 0 drives the TMA ring; all lanes scan the claim words when
// stealing).  Every ring slot carries a header (rows, statistics, control events), so the
// consumers follow whatever the producer decided: EV_SCALE (load 1 + scale of a group),
// EV_FLUSH (owner partial -> slot, set or add), EV_MERGE (add stolen chunks), EV_PUBLISH
// (thief partial -> pool + flag), EV_END.
#pragma once

namespace al {

constexpr int kStealSlots = 32;   // concurrently usable protocol states (streams / captures)
constexpr int kStealMaxG = 296;   // CTAs per launch (<= 2 per SM)
constexpr int kStealMaxC = 64;    // stealable chunks per owner

struct StealSlot {
  unsigned long long word[kStealMaxG];
  unsigned int flag[kStealMaxG][kStealMaxC];
  unsigned int pidx[kStealMaxG][kStealMaxC];
  unsigned int epoch;
  unsigned int pool;
  unsigned int done;
  unsigned int stolen;  // chunks stolen over all launches on this slot (diagnostics)
};
__device__ StealSlot g_steal[kStealSlots];

struct ChunkGeo {
  int64_t cstart;  // first chunked row (contiguous layout: the last nch * C rows of the range)
  int64_t group;   // group of the range's last segment
  int nch;
  bool il;         // interleaved layout: chunk j of owner k is global chunk j * G + k
};

// Chunk geometry of owner k: identical in the owner and in every thief.  Interleaved (single
// group): the whole row range is cut into C-row chunks dealt round robin, chunk j of owner k =
// global chunk j*G + k, so the owners sweep HBM together (the dynamic tail's access order) and
// stolen chunks are the sweep's last ones.  Contiguous: the last segment of the owner's static
// range, cut into its last nch chunks.
__device__ __forceinline__ ChunkGeo chunk_geo(int64_t k, int64_t N, int64_t G, int64_t S_grp, int C,
                                              bool il = false) {
  if (il) {
    const int64_t nc = (N + C - 1) / C;
    ChunkGeo c{0, 0, nc > k ? static_cast<int>((nc - 1 - k) / G + 1) : 0, true};
    return c;
  }
  const int64_t r0 = part_begin(k, N, G), r1 = part_begin(k + 1, N, G);
  ChunkGeo c{r1, 0, 0, false};
  if (r1 <= r0) return c;
  c.group = (r1 - 1) / S_grp;
  const int64_t seg0 = max(r0, c.group * S_grp);
  int64_t n = (r1 - seg0) / C;
  if (n > kStealMaxC) n = kStealMaxC;
  c.nch = static_cast<int>(n);
  c.cstart = r1 - n * C;
  return c;
}
__device__ __forceinline__ int64_t chunk_row0(const ChunkGeo& c, int64_t k, int64_t G, int C, int j) {
  return c.il ? (static_cast<int64_t>(j) * G + k) * C : c.cstart + static_cast<int64_t>(j) * C;
}

__device__ __forceinline__ unsigned long long steal_word(unsigned int e, unsigned int h, unsigned int t) {
  return (static_cast<unsigned long long>(e) << 32) | (static_cast<unsigned long long>(h) << 16) | t;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// data-stage events (packed above the row count in h_n): load (1 + scale) of group h_a before
// the stage; after it, flush the accumulators to slot k + group (an earlier segment) or add
// them to the shared running total (the last segment).  Control-only slots (no rows): merge the
// stolen chunks, publish a stolen chunk (args in h_b), end.
enum : int { kEvScale = 1, kEvFlush = 2, kEvFlushTotal = 4, kEvMerge = 8, kEvPublish = 16,
             kEvEnd = 32 };

// MAXT: the block size bound; 352 (10 consumer warps + the producer, the cfg2 plan) lets ptxas
// use 184 registers per thread instead of 168
template <typename T, int V, int R, bool FULL, int MAXT = 384>
__global__ void __launch_bounds__(MAXT, 1) adaln_bwd_steal(const BwdParams p) {
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
  const int C = p.chunk_rows;
  // shared-memory layout by integer offsets from the shared array (every pointer stays in the
  // shared window, so the header and total accesses compile to LDS/STS, not generic LD/ST)
  size_t off = static_cast<size_t>(NS) * stage_bytes;  // 16-aligned: stage_bytes % 16 == 0
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + off);
  uint64_t* empty = full + NS;
  off += 16 * static_cast<size_t>(NS);
  int64_t* h_row = reinterpret_cast<int64_t*>(smem + off);
  int64_t* h_a = h_row + NS;   // EV_SCALE: group
  int64_t* h_b = h_a + NS;     // EV_MERGE: (group, head, nch); EV_PUBLISH: (victim, chunk, pool)
  off += 24 * static_cast<size_t>(NS);
  CT* h_m = reinterpret_cast<CT*>(smem + off);
  CT* h_r = h_m + NS * R;
  off += (2 * static_cast<size_t>(NS) * R * sizeof(CT) + 15) & ~size_t(15);
  int* h_n = reinterpret_cast<int*>(smem + off);  // rows | events << 8
  int* s_bcast = h_n + 2 * NS;
  off += (8 * static_cast<size_t>(NS) + 4 + 15) & ~size_t(15);
  CT* red = reinterpret_cast<CT*>(smem + off);  // [2][ncw][R][2]
  off += (2 * static_cast<size_t>(ncw) * R * 2 * sizeof(CT) + 15) & ~size_t(15);
  // the owner's running total of its last segment, [2][D] (dscale | dshift): chunk partials are
  // added here in chunk order (a shared-memory RMW -- a global one would put an L2 round trip
  // under saturated HBM traffic on the consumers' path once per chunk)
  CT* tot_sc = reinterpret_cast<CT*>(smem + off);
  CT* tot_sh = tot_sc + p.D;

  StealSlot* st = p.steal;
  const unsigned int E = *reinterpret_cast<volatile unsigned int*>(&st->epoch) + 1u;
  const int64_t k = blockIdx.x;
  const int64_t G = p.G;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == ncw) {  // ---------------- producer warp ----------------
    // All 32 lanes follow the control flow (the claim results are broadcast by shuffles and
    // the victim scan is warp-wide); lane 0 alone touches the ring, the statistics and the
    // claim words.  The owner claims its next chunk with one atomicAdd on the head, issued a
    // chunk ahead of use (it cannot fail, so it needs no CAS loop); only thieves use CAS.
    const ChunkGeo mine = chunk_geo(k, p.N, G, p.S_grp, C, p.interleave != 0);
    if (lane == 0) atomicExch(&st->word[k], steal_word(E, 0u, static_cast<unsigned int>(mine.nch)));
    const uint64_t pol = policy_evict_first();
    const uint8_t* xb = static_cast<const uint8_t*>(p.x);
    const uint8_t* db = static_cast<const uint8_t*>(p.dy);
    const CT* mean_p = static_cast<const CT*>(p.mean);
    const CT* rstd_p = static_cast<const CT*>(p.rstd);
    int s = 0;
    uint32_t f = 0;

    auto emit = [&](int64_t row, int rows, int ev, int64_t a, int64_t b) {
      CT m[R], r[R];
      if (lane == 0) {
        // the row statistics are loaded by lane 0 alone, issued before it waits for the ring
        // slot (the wait hides their round trip); no warp-wide step on the per-stage path
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const bool ok = rr < rows;
          m[rr] = ok ? mean_p[row + rr] : CT(0);
          r[rr] = ok ? rstd_p[row + rr] : CT(0);
        }
        if (f > 0) mbar_wait(&empty[s], (f - 1) & 1);
        h_row[s] = row;
        h_a[s] = a;
        h_b[s] = b;
        h_n[s] = rows | (ev << 8);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          h_m[s * R + rr] = rows > 0 ? m[rr] : CT(0);
          h_r[s * R + rr] = rows > 0 ? r[rr] : CT(0);
        }
        if (rows > 0) {
          mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(2 * rows * RB));
          uint8_t* dst = smem + static_cast<size_t>(s) * stage_bytes;
          for (int rr = 0; rr < rows; ++rr) {
            bulk_g2s(dst + rr * RB, xb + (row + rr) * RB, RB, &full[s], pol);
            bulk_g2s(dst + (R + rr) * RB, db + (row + rr) * RB, RB, &full[s], pol);
          }
        } else {
          mbar_arrive(&full[s]);  // control-only slot: completes the phase without data
        }
      }
      if (++s == NS) {
        s = 0;
        ++f;
      }
    };
    // Events travel in control-only slots of their own, so the consumers' data-stage loop is
    // the round-1 dynamic loop verbatim (no per-stage event decoding on the hot path).
    auto data = [&](int64_t row, int rows) { emit(row, rows, 0, 0, 0); };
    auto ctrl = [&](int ev, int64_t a, int64_t b) { emit(0, 0, ev, a, b); };
    // one chunk's stages [row0, min(row0 + C, N)), optionally preceded by a scale load
    auto emit_chunk = [&](int64_t row0, bool scale, int64_t g, int last_ev) {
      if (scale) ctrl(kEvScale, g, 0);
      const int64_t end = row0 + C < p.N ? row0 + C : p.N;
      for (int64_t row = row0; row < end; row += R)
        data(row, end - row < R ? static_cast<int>(end - row) : R);
      if (last_ev) ctrl(last_ev, 0, 0);
    };

    // ---- 1. the static part: earlier segments and the pre part of the last segment ----
    const int64_t r0 = mine.il ? 0 : part_begin(k, p.N, G);
    int64_t scaled = -1;
    if (mine.il && mine.nch == 0) {  // no chunk for this CTA: its slot still takes part (zeros)
      ctrl(kEvScale, 0, 0);
      ctrl(kEvFlush, 0, 0);
    }
    {
      StageWalker w;
      w.init(r0, mine.il ? 0 : mine.cstart, p.S_grp);
      int64_t prev_g = -1;
      while (!w.done()) {
        int64_t start, g;
        const int rows = w.next(R, start, g);
        if (g != prev_g) {
          ctrl(kEvScale, g, 0);
          scaled = g;
        }
        data(start, rows);
        const int64_t seg_end = min((g + 1) * p.S_grp, mine.cstart);
        if (start + rows >= seg_end)  // the last segment's pre part feeds the running total
          ctrl((g == mine.group && mine.nch > 0) ? kEvFlushTotal : kEvFlush, g, 0);
        prev_g = g;
      }
    }
    // ---- 2. own chunks from the head, the next claim always in flight ----
    if (mine.nch > 0) {
      unsigned long long claim = 0;
      if (lane == 0) claim = atomicAdd(&st->word[k], 1ull << 16);
      unsigned int own_head = 0;
      while (true) {
        const unsigned long long c = __shfl_sync(0xffffffffu, claim, 0);
        const unsigned int h = static_cast<unsigned int>(c >> 16) & 0xffffu;
        const unsigned int t = static_cast<unsigned int>(c) & 0xffffu;
        if (h >= t) break;
        own_head = h + 1;
        if (lane == 0) claim = atomicAdd(&st->word[k], 1ull << 16);  // the next one, ahead
        const bool first = scaled != mine.group;
        scaled = mine.group;
        emit_chunk(chunk_row0(mine, k, G, C, h), first, mine.group, kEvFlushTotal);
      }
      // the chunks thieves took, [own_head, nch), are added in order by the consumers
      ctrl(kEvMerge, 0, (mine.group << 32) | (static_cast<int64_t>(own_head) << 16) | mine.nch);
    }
    // ---- 3. steal: from the owner with the most unclaimed chunks (>= 2, so that owner keeps
    //         working while this CTA computes the stolen one), one chunk off its tail ----
    unsigned int pool_p = 0xffffffffu;
    while (true) {
      if (pool_p == 0xffffffffu) {
        unsigned int q = 0;
        if (lane == 0) q = atomicAdd(&st->pool, 1u);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= static_cast<unsigned int>(p.pool_cap)) break;
        pool_p = q;
      }
      int best_v = -1;
      unsigned int best_rem = 1;
      for (int v = lane; v < G; v += 32) {
        const unsigned long long wv = ld_volatile_u64(&st->word[v]);
        if (static_cast<unsigned int>(wv >> 32) != E) continue;
        const unsigned int h = static_cast<unsigned int>(wv >> 16) & 0xffffu;
        const unsigned int t = static_cast<unsigned int>(wv) & 0xffffu;
        const unsigned int rem = t > h ? t - h : 0;
        if (rem > best_rem) {
          best_rem = rem;
          best_v = v;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned int orem = __shfl_xor_sync(0xffffffffu, best_rem, o);
        const int ov = __shfl_xor_sync(0xffffffffu, best_v, o);
        if (orem > best_rem || (orem == best_rem && ov >= 0 && (best_v < 0 || ov < best_v))) {
          best_rem = orem;
          best_v = ov;
        }
      }
      if (best_v < 0) break;
      unsigned int got = 0xffffffffu;
      if (lane == 0) {
        unsigned long long old = ld_volatile_u64(&st->word[best_v]);
        while (static_cast<unsigned int>(old >> 32) == E) {
          const unsigned int h = static_cast<unsigned int>(old >> 16) & 0xffffu;
          const unsigned int t = static_cast<unsigned int>(old) & 0xffffu;
          if (t < h + 2) break;
          const unsigned long long prev = atomicCAS(&st->word[best_v], old, steal_word(E, h, t - 1));
          if (prev == old) {
            got = t - 1;
            break;
          }
          old = prev;
        }
      }
      got = __shfl_sync(0xffffffffu, got, 0);
      if (got == 0xffffffffu) continue;  // lost the race: scan again
      if (lane == 0) atomicAdd(&st->stolen, 1u);
      const ChunkGeo vg = chunk_geo(best_v, p.N, G, p.S_grp, C, p.interleave != 0);
      emit_chunk(chunk_row0(vg, best_v, G, C, got), true, vg.group, 0);
      ctrl(kEvPublish, 0,
           (static_cast<int64_t>(best_v) << 48) | (static_cast<int64_t>(got) << 32) | pool_p);
      scaled = vg.group;
      pool_p = 0xffffffffu;
    }
    ctrl(kEvEnd, 0, 0);
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
  CT* ws_sc = static_cast<CT*>(p.ws);
  CT* ws_sh = ws_sc + p.nslots * p.D;
  bool nf = false;

  P s1[V][NP], acc_sc[V][NP], acc_sh[V][NP];
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));

  auto col_of = [&](int j) { return static_cast<int64_t>(coff[j] / 16) * EPV; };
  // global slot <- acc, this thread's columns; acc cleared
  auto flush_to = [&](int64_t slot) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (vmask >> j & 1) {
        P* a = reinterpret_cast<P*>(ws_sc + slot * p.D + col_of(j));
        P* b = reinterpret_cast<P*>(ws_sh + slot * p.D + col_of(j));
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          a[e] = acc_sc[j][e];
          b[e] = acc_sh[j][e];
          acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));
        }
      }
    }
  };
  // shared running total <- acc (set) or total += acc (add); acc cleared
  auto total_add = [&](bool add) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (vmask >> j & 1) {
        P* a = reinterpret_cast<P*>(tot_sc + col_of(j));
        P* b = reinterpret_cast<P*>(tot_sh + col_of(j));
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          a[e] = add ? add2(a[e], acc_sc[j][e]) : acc_sc[j][e];
          b[e] = add ? add2(b[e], acc_sh[j][e]) : acc_sh[j][e];
          acc_sc[j][e] = acc_sh[j][e] = splat2(CT(0));
        }
      }
    }
  };
  // global slot <- shared running total (this thread's columns)
  auto total_to = [&](int64_t slot) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (vmask >> j & 1) {
        const P* a = reinterpret_cast<const P*>(tot_sc + col_of(j));
        const P* b = reinterpret_cast<const P*>(tot_sh + col_of(j));
        P* ga = reinterpret_cast<P*>(ws_sc + slot * p.D + col_of(j));
        P* gb = reinterpret_cast<P*>(ws_sh + slot * p.D + col_of(j));
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          ga[e] = a[e];
          gb[e] = b[e];
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

  int s = 0;
  uint32_t ph = 0;
  int it = 0;

  // One ring stage (as adaln_bwd_tma's dynamic instance): phase 1 row sums + column
  // accumulators, cross-warp totals, slot release, phase 2 dx from registers.
  auto stage = [&](auto all_tag, int64_t rb, int rows, const CT* mc, const CT* rc) {
    constexpr bool ALL = decltype(all_tag)::value;
    const uint32_t stx_u = smem_addr(smem) + static_cast<uint32_t>(s * stage_bytes);
    const uint32_t std_u = stx_u + static_cast<uint32_t>(R * RB);
    CT* rd = red + (it & 1) * (ncw * R * 2);
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
      const P nmr = splat2(-mc[rr] * rc[rr]);
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
    if (p.early_release == 1) {  // as in adaln_bwd_tma: release once this warp's loads are consumed
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
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
    uint8_t* dxrow = static_cast<uint8_t*>(p.dx) + rb * RB;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (ALL || rr < rows) {
        const CT rr_ = rc[rr];
        const P c0 = splat2(-rr_ * tot[2 * rr] * invD), c1 = splat2(-rr_ * tot[2 * rr + 1] * invD);
        const P r2 = splat2(rr_);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          if (vmask >> j & 1) {
            P o[NP];
#pragma unroll
            for (int e = 0; e < NP; ++e) o[e] = fma2(gg[rr][j][e], r2, fma2(xh[rr][j][e], c1, c0));
            st_global_cs(dxrow + rr * RB + coff[j], pack2<T>(o));
          }
        }
        if (tid == 0) nf |= !(finite_ct(tot[2 * rr]) && finite_ct(tot[2 * rr + 1]));
      }
    }
    ++it;
  };

  int64_t cur_g = -1;
  bool slot_init = false;  // has slot k + cur_g (or the shared total) been written
  while (true) {
    // ---- data stages: the round-1 dynamic loop, verbatim ----
    int hn;
    while (true) {
      mbar_wait(&full[s], ph);
      hn = h_n[s];
      if (hn == 0 || hn > R) break;  // a control slot
      const int64_t rb = h_row[s];
      CT mc[R], rc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        mc[rr] = h_m[s * R + rr];
        rc[rr] = h_r[s * R + rr];
      }
      if (hn == R) stage(std::true_type{}, rb, R, mc, rc);
      else stage(std::false_type{}, rb, hn, mc, rc);
      if (++s == NS) {
        s = 0;
        ph ^= 1;
      }
    }
    // ---- a control slot (rare) ----
    const int ev = hn >> 8;
    if (ev & kEvEnd) break;
    const int64_t a = h_a[s], b = h_b[s];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
    if (ev & kEvScale) {
      cur_g = a;
      load_scale(cur_g);
      slot_init = false;
    } else if (ev & kEvFlushTotal) {
      total_add(slot_init);  // written to the slot after the merge (kEvMerge)
      slot_init = true;
    } else if (ev & kEvFlush) {
      flush_to(k + cur_g);
      slot_init = true;
    } else if (ev & kEvPublish) {  // a stolen chunk: pool slot, then the owner's flag
      const int v = static_cast<int>(b >> 48);
      const int j = static_cast<int>((b >> 32) & 0xffff);
      const unsigned int q = static_cast<unsigned int>(b & 0xffffffffu);
      flush_to(p.tail_slot0 + q);
      named_bar_sync(1, nc);
      if (tid == 0) {
        __threadfence();
        st->pidx[v][j] = q;
        st_release_u32(&st->flag[v][j], E);
      }
    } else if (ev & kEvMerge) {  // the chunks thieves took from this range, in chunk order
      const int64_t g = b >> 32;
      const int h0 = static_cast<int>((b >> 16) & 0xffff), nch = static_cast<int>(b & 0xffff);
      for (int j = h0; j < nch; ++j) {
        if (tid == 0) {
          while (ld_acquire_u32(&st->flag[k][j]) != E) __nanosleep(32);
          *s_bcast = static_cast<int>(ld_acquire_u32(&st->pidx[k][j]));
        }
        named_bar_sync(1, nc);
        const int64_t q = p.tail_slot0 + *s_bcast;
#pragma unroll
        for (int jj = 0; jj < V; ++jj) {
          if (vmask >> jj & 1) {
            const int64_t col = col_of(jj);
#pragma unroll
            for (int e = 0; e < NP; ++e) {  // L2 reads: written by another SM
              acc_sc[jj][e] = __ldcg(reinterpret_cast<const P*>(ws_sc + q * p.D + col + 2 * e));
              acc_sh[jj][e] = __ldcg(reinterpret_cast<const P*>(ws_sh + q * p.D + col + 2 * e));
            }
          }
        }
        total_add(slot_init);
        slot_init = true;
        named_bar_sync(1, nc);  // everyone has read s_bcast before the next chunk's write
      }
      total_to(k + g);
    }
  }
  if (nf && p.nonfinite) atomicExch(p.nonfinite, 1);
  named_bar_sync(1, nc);
  if (tid == 0) AL_TRACE(1, 1);
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&st->done, 1u) == static_cast<unsigned int>(G - 1)) {
      // last CTA out: every owner has merged, every thief has published
      st->pool = 0u;
      st->done = 0u;
      __threadfence();
      st_release_u32(&st->epoch, E);
    }
  }
}

}  // namespace al
