// Flat SpMM for large degree-ordered graphs, chunks of <= 32 probes (the narrow class: gathered rows
// of <= 128 bytes in fp32, <= 256 bytes in fp64): the C5 gather.  Described for its main shape, fp32
// rows of 17..32 probes (128 bytes, 8 lanes per row, four CSR rows per warp); see L and VT below for
// 64-byte and 256-byte rows.
//
// The warp-per-row kernel (engine.cuh: spmm_kernel) walks offsets -> columns -> gathers -> epilogue
// as one dependent chain per row and holds the gathered rows in registers, so a warp keeps ~10 line
// requests in flight and the DRAM misses run at ~0.6 of the random-line rate the B200 sustains.
// Here the gathered rows are STAGED IN SHARED MEMORY by cp.async (LDGSTS, 16 bytes per lane): a
// QUARTER-warp (8 lanes x 16 bytes = one 128-byte row of the vector) owns one CSR row, a warp walks a
// QUAD of four consecutive rows in lockstep (the degree-ordered fold makes neighbouring rows equally
// long), and the nonzeros of successive quads are FLATTENED into batches of kFlatU slots per quarter
// (32 line requests per warp and batch).  A ring of kFlatNB batches per warp keeps kFlatNB - 1 batches
// in flight whatever the row lengths are, at no register cost.
//
//   * work items (atomic counter): quads of long-row segments first, then graph-fixed fine row tiles;
//   * a batch is kFlatU slots of one quad: slot q of quarter i gathers the vector row of nonzero
//     j + q of the quarter's row; slots past the row's end are zero-filled by the copy (src-size 0),
//     so consumption is one unconditional unrolled loop; a batch starts at an even j, so a slot's
//     chain (even / odd position) is a compile-time choice;
//   * the quad's last batch also copies the rows' own values, degree and dinv, and its consumption
//     ends with the operator epilogue and the store (or the store of a segment's partial sums);
//   * lane `sub` of a quarter loads the column index of the quarter's slot `sub` two batches ahead of
//     the copies; row ends come from a register block of 32 prefetched offsets;
//   * loop: wait for the oldest batch (cp.async.wait_group), consume it from shared memory, issue
//     the newest batch into the buffer freed one iteration ago, generate the batch after that.
//
// Arithmetic = the narrow class of gather_range (engine.cuh): a row is summed as two chains (even /
// odd positions from the row start, ascending), acc = s_even + s_odd, then the same epilogue, so the
// results are bitwise those of spmm_kernel's HALF2 / full-warp mappings (adding the +0.0 of a
// zero-filled slot never changes an accumulator, which starts at +0.0 and so is never -0.0).
#include "engine.cuh"

namespace slq {

#ifndef SLQ_FLAT_NB
#define SLQ_FLAT_NB 3
#endif
#ifndef SLQ_FLAT_WARPS
#define SLQ_FLAT_WARPS 8
#endif
#ifndef SLQ_FLAT_CTAS
#define SLQ_FLAT_CTAS 2
#endif
#ifndef SLQ_FLAT_CVT
#define SLQ_FLAT_CVT 1   // 1: integer widening + DFMA instead of F2F.F64.F32 + DADD (same bits for finite inputs)
#endif
#ifndef SLQ_FLAT_MIX
#define SLQ_FLAT_MIX 0
#endif
constexpr int kFlatU = 8;
constexpr int kFlatNB = SLQ_FLAT_NB;           // batches in the ring (kFlatNB - 1 in flight)
constexpr int kFlatThreads = 32 * SLQ_FLAT_WARPS;
constexpr int kFlatCtasPerSm = SLQ_FLAT_CTAS;
constexpr int kFlatBatchBytes = kFlatU * 4 * 128;   // gathered rows of one batch
constexpr int kFlatOwnBytes = 512 + 8 * 16;         // own rows + (degree, dinv) of up to 8 rows
constexpr int kFlatWarpBytes = kFlatNB * (kFlatBatchBytes + kFlatOwnBytes);
constexpr int kFlatSmem = SLQ_FLAT_WARPS * kFlatWarpBytes;

constexpr int PH_NZ = 0, PH_ITEM = 2, PH_DONE = 3;
// Operator-pair chunk (slq_rules_pair): columns < a.split run the normalized Laplacian (prescaled
// gathers / first-step records), the others the density matrix on the SAME probes -- one 128-byte
// gather per nonzero serves both Lanczos runs.  a.split is a multiple of 4 (a lane = 4 columns).
constexpr int kPair = 5;
constexpr int GF_OK = 1, GF_LIVE = 2, GF_END = 4, GF_SEG = 8;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds128d(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// BITS: the first step.  u_0 is the +-1 probe bitmask (bits[row][kBitWords], word 0 = probes 0..31);
// a slot gathers one 16-byte bitmask row -- for the normalized Laplacian the 32-byte [bits | dinv]
// record (a.rec), so dinv[col] comes from the same sector -- copied by ONE lane (lane `sub` copies its
// quarter's slot `sub`: the column index it loaded itself), 32 bytes of shared memory per slot.
//
// L = lanes per row of the vector: 8 (128-byte rows: a quad of CSR rows per warp), 4 (64-byte rows:
// eight CSR rows per warp; a lane then loads the column indices of two slots) or 16 (256-byte rows of
// 17..32 fp64 probes: two CSR rows per warp).  Shared-memory addressing is the same: a slot's rows of all the warp's CSR rows are 512
// contiguous bytes, lane l's 16 bytes at offset 16 l.
// VT = float (4 probes per lane) or double (2 probes per lane: rows of <= 16 fp64 probes).
template <typename VT, int KIND, bool BITS, int L>
__global__ void __launch_bounds__(kFlatThreads, kFlatCtasPerSm) spmm_flat_kernel(SpmmArgs a) {
  constexpr int EPL = 16 / static_cast<int>(sizeof(VT));   // probes per lane (one 16-byte piece of a row)
  static_assert(L == 16 || L == 8 || L == 4, "lanes per gathered row");
  constexpr int RPW = 32 / L;            // CSR rows a warp walks in lockstep
  constexpr int kOffBlock = 32 - RPW;    // rows per offsets block (32 prefetched offsets: RPW + 1 per group)
  constexpr unsigned FULL = 0xffffffffu;
  constexpr bool NL = nl_kind<KIND>() || KIND == kPair;   // dinv[row] in the epilogue
  constexpr bool REC = KIND == SLQ_NORMALIZED_LAPLACIAN || KIND == kPair;   // BITS: gathers [bits | dinv] records
  const int lane = threadIdx.x & 31;
  const int sub = lane & (L - 1);
  const int qid = lane / L;
  const int qbase = lane & ~(L - 1);

  // probes EPL sub .. EPL sub + EPL - 1 of the chunk
  bool pv[EPL];
  double rj[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    pv[j] = EPL * sub + j < a.c;
    rj[j] = pv[j] ? __ldg(a.r + EPL * sub + j) : 1.0;
  }
  const bool all4 = pv[EPL - 1];
  const bool lane_nl = KIND != kPair || EPL * sub < a.split;   // pair chunk: this lane's operator
  // 16 bytes of a row per lane; lanes past the row's end copy nothing (zero fill)
  const int lane_bytes = EPL * sub + EPL - 1 < a.ldc_in ? 16 : 0;
  const uint32_t strideb = static_cast<uint32_t>(a.ldc_in) * static_cast<uint32_t>(sizeof(VT));   // row stride in bytes
  const char* __restrict__ ugb =
      static_cast<const char*>((KIND == kNLPre || KIND == kPair) ? a.upre : a.u) + (lane_bytes ? 16 * sub : 0);   // gathered vector
  const char* __restrict__ uob = static_cast<const char*>(a.u) + (lane_bytes ? 16 * sub : 0);   // own values
  // keep the per-lane base pointers whole, so a gather address is one IMAD.WIDE (col * stride + base)
  asm volatile("" : "+l"(ugb));
  asm volatile("" : "+l"(uob));
  extern __shared__ __align__(128) unsigned char flat_smem[];
  const uint32_t sm_warp = static_cast<uint32_t>(__cvta_generic_to_shared(flat_smem)) +
                           (threadIdx.x >> 5) * kFlatWarpBytes;   // BITS: + buf * batch + (q * RPW + qid) * 32
  const unsigned char* __restrict__ recb = reinterpret_cast<const unsigned char*>(
      (BITS && REC) ? a.rec : a.bits);
  constexpr uint32_t rec_stride = 4u * ((BITS && REC) ? kRecWords : kBitWords);
  const uint32_t sm_ring = static_cast<uint32_t>(__cvta_generic_to_shared(flat_smem)) +
                           (threadIdx.x >> 5) * kFlatWarpBytes + lane * 16;        // + buf * batch + q * 512
  const uint32_t sm_own = static_cast<uint32_t>(__cvta_generic_to_shared(flat_smem)) +
                          (threadIdx.x >> 5) * kFlatWarpBytes + kFlatNB * kFlatBatchBytes;   // + buf * own
  VT* __restrict__ w = static_cast<VT*>(a.w) + EPL * sub;
  const int64_t* __restrict__ off = a.offsets;
  const int32_t* __restrict__ cols = a.cols;
  const double scale = (KIND == SLQ_DENSITY || KIND == kPair) ? a.dscal[3] : 0.0;
  const bool has_long = a.long_counts != nullptr;
  const long long nseg = has_long ? a.long_counts[1] : 0;
  const long long nsq = (nseg + RPW - 1) / RPW;   // groups of RPW segments
  const long long nitems = nsq + a.nftiles;
  const int64_t nrows = a.n_rows;   // offsets has nrows + 1 entries

  // ---- cursor: warp-uniform control; qpos / dq / rowok are per quarter
  int phase = PH_ITEM;
  bool isseg = false;
  int R = 0, Rend = 0;        // first row (segment) of the current quad, end of the item
  int obase = 0;
  int64_t offA = 0, offB = 0;   // off[obase + lane], off[obase + kOffBlock + lane]
  int64_t qpos = 0;           // first nonzero of this quarter's row (segment)
  int dq = 0, dmax = 0, dmin = 0, j = 0;
  bool rowok = false;

  auto load_off = [&](int64_t r) -> int64_t { return __ldg(off + (r < nrows ? r : nrows)); };
  auto enter_quad = [&]() {
    if (R >= Rend) { phase = PH_ITEM; return; }
    if (isseg) {
      const int sg = R + qid;
      rowok = sg < Rend;
      int64_t p0 = 0, p1 = 0;
      if (rowok) {
        p0 = a.seg_begin[sg];
        const int64_t re = __ldg(off + a.seg_row[sg] + 1);
        p1 = p0 + kSeg < re ? p0 + kSeg : re;
      }
      qpos = p0;
      dq = static_cast<int>(p1 - p0);
    } else {
      int idx = R - obase;
      if (idx >= kOffBlock) {
        obase += kOffBlock;
        idx -= kOffBlock;
        offA = offB;
        offB = load_off(static_cast<int64_t>(obase) + kOffBlock + lane);
      }
      const int64_t p0 = __shfl_sync(FULL, offA, idx + qid);
      const int64_t p1 = __shfl_sync(FULL, offA, idx + qid + 1);
      rowok = R + qid < Rend;
      int64_t d = rowok ? p1 - p0 : 0;
      if (has_long && d > kLongRow) { rowok = false; d = 0; }   // summed from its segments
      qpos = p0;
      dq = static_cast<int>(d);
    }
    dmax = __reduce_max_sync(FULL, dq);
    dmin = __reduce_min_sync(FULL, dq);
    j = 0;
    phase = PH_NZ;
  };
  auto fetch_item = [&]() {
    for (;;) {
      long long item = 0;
      if (lane == 0) item = static_cast<long long>(atomicAdd(a.work, 1ull));
      item = __shfl_sync(FULL, item, 0);
      if (item >= nitems) { phase = PH_DONE; return; }
#if SLQ_FLAT_MIX
      // the item list runs from the long rows to the shortest ones (degree order): take items from
      // both ends alternately, so the low-parallelism batches of short rows overlap the full ones
      item = (item & 1) ? nitems - 1 - (item >> 1) : (item >> 1);
#endif
      if (item < nsq) {
        isseg = true;
        R = static_cast<int>(RPW * item);
        Rend = static_cast<int>(R + RPW < nseg ? R + RPW : nseg);
      } else {
        const long long t = item - nsq;
        const int64_t rb = a.ftile_rows[t], re = a.ftile_rows[t + 1];
        if (rb >= re) continue;
        isseg = false;
        R = static_cast<int>(rb);
        Rend = static_cast<int>(re);
        obase = R;
        offA = load_off(static_cast<int64_t>(obase) + lane);
        offB = load_off(static_cast<int64_t>(obase) + kOffBlock + lane);
      }
      enter_quad();
      return;
    }
  };

  // ---- one batch: nv = bit mask of the slots this lane copies, r0 = the quad's first row / segment (uniform),
  // flags: GF_OK (this quarter has a row), uniform GF_LIVE / GF_END (the quad's last batch) / GF_SEG
  struct Group { int nv, r0, fl; };
  auto gen = [&](Group& g, int64_t& mypos, int64_t& mypos2) {
    if (phase == PH_ITEM) fetch_item();
    mypos = -1;
    mypos2 = -1;
    g.nv = 0;
    g.r0 = R;
    g.fl = 0;
    if (phase == PH_DONE) return;
    const int rem = dq - j;
    const int nv = rem < 0 ? 0 : (rem > kFlatU ? kFlatU : rem);
    if (sub < nv) mypos = qpos + j + sub;
    if (L == 4 && sub + 4 < nv) mypos2 = qpos + j + sub + 4;   // 4 lanes per row: two slots per lane
    // slots this lane copies (the others are zero-filled); BITS: the quarter's valid slots
    g.nv = (BITS || lane_bytes) ? (1 << nv) - 1 : 0;
    j += kFlatU;
    g.fl = GF_LIVE | (rowok ? GF_OK : 0) | (isseg ? GF_SEG : 0);
    if (j >= dmax) {
      g.fl |= GF_END;
      R += RPW;
      enter_quad();
    }
  };

  // ---- consumer state
  double ae[EPL], ao[EPL];
#pragma unroll
  for (int jj = 0; jj < EPL; ++jj) ae[jj] = ao[jj] = 0.0;

  auto finish_row = [&](int64_t r, const double (&own)[EPL], double d, double dis) {
    VT y[EPL];
#pragma unroll
    for (int jj = 0; jj < EPL; ++jj) {
      const double tot = ae[jj] + ao[jj];
      const double x = __dmul_rn(own[jj], rj[jj]);
      const double sc = __dmul_rn(tot, rj[jj]);
      if constexpr (KIND == kPair)
        y[jj] = from_f64<VT>(lane_nl ? op_epilogue<SLQ_NORMALIZED_LAPLACIAN>(x, sc, d, dis, scale)
                                     : op_epilogue<SLQ_DENSITY>(x, sc, d, dis, scale));
      else
        y[jj] = from_f64<VT>(op_epilogue<KIND>(x, sc, d, dis, scale));
    }
    VT* dst = w + r * a.ldc_out;
    if (all4) {
      if constexpr (EPL == 4) *reinterpret_cast<float4*>(dst) = make_float4(y[0], y[1], y[2], y[3]);
      else *reinterpret_cast<double2*>(dst) = make_double2(y[0], y[1]);
    } else {
#pragma unroll
      for (int jj = 0; jj < EPL; ++jj)
        if (pv[jj]) dst[jj] = y[jj];
    }
  };
  auto finish_seg = [&](int64_t sg) {
    double* dst = a.segpart + sg * a.cpad + EPL * sub;
#pragma unroll
    for (int jj = 0; jj < EPL; ++jj)
      if (pv[jj]) dst[jj] = ae[jj] + ao[jj];
  };
  auto consume = [&](const Group& g, int buf) {
    if constexpr (BITS) {
      const uint32_t base = sm_warp + buf * kFlatBatchBytes + qid * 32;
      constexpr int kSlotRec = RPW * 32;   // bytes of one slot's records
#pragma unroll
      for (int q = 0; q < kFlatU; ++q) {
        const uint32_t wd = lds32(base + q * kSlotRec) >> (EPL * sub);
        // s_c: dinv[col] (normalized Laplacian; a zero-filled slot has dinv = 0), else 1 for a valid
        // slot and 0 for a zero-filled one: fma(s_c, +-1, acc) is the reference term or acc itself
        const double one = ((g.nv >> q) & 1) ? 1.0 : 0.0;
        const double sk = KIND == SLQ_NORMALIZED_LAPLACIAN ? lds64(base + q * kSlotRec + 16)
                          : (KIND == kPair ? (lane_nl ? lds64(base + q * kSlotRec + 16) : one) : one);
#pragma unroll
        for (int jj = 0; jj < EPL; ++jj) {
          const double x = ((wd >> jj) & 1u) ? 1.0 : -1.0;
          if (q & 1) ao[jj] = fma(sk, x, ao[jj]); else ae[jj] = fma(sk, x, ae[jj]);
        }
      }
    } else {
      const uint32_t base = sm_ring + buf * kFlatBatchBytes;
#pragma unroll
      for (int q = 0; q < kFlatU; ++q) {
        if constexpr (EPL == 2) {
          const double2 x = lds128d(base + q * 512);
          if (q & 1) { ao[0] += x.x; ao[1] += x.y; } else { ae[0] += x.x; ae[1] += x.y; }
        } else {
        const float4 x = lds128(base + q * 512);
#if SLQ_FLAT_CVT
        // acc + double(x) without the conversion instruction (the XU pipe converts 4 lanes per clock):
        // the double with exponent field = x's 8-bit exponent and mantissa = x's (three integer
        // instructions) is x * 2^-896 exactly -- also for zeros and subnormals, whose exponent field
        // is 0 in both formats -- and fma(that, 2^896, acc) rounds acc + x once, like the add.
        // (Inf/NaN inputs come out as 2^128 * 1.m: still non-finite after the fp32 store.)
        const double k896 = __hiloint2double(0x77f00000, 0);   // 2^896
        auto wide = [](float v) {
          const int f = __float_as_int(v);
          return __hiloint2double((f >> 3) & static_cast<int>(0x8fffffffu), f << 29);
        };
        if (q & 1) {
          ao[0] = fma(wide(x.x), k896, ao[0]); ao[1] = fma(wide(x.y), k896, ao[1]);
          ao[2] = fma(wide(x.z), k896, ao[2]); ao[3] = fma(wide(x.w), k896, ao[3]);
        } else {
          ae[0] = fma(wide(x.x), k896, ae[0]); ae[1] = fma(wide(x.y), k896, ae[1]);
          ae[2] = fma(wide(x.z), k896, ae[2]); ae[3] = fma(wide(x.w), k896, ae[3]);
        }
#else
        if (q & 1) {
          ao[0] += static_cast<double>(x.x); ao[1] += static_cast<double>(x.y);
          ao[2] += static_cast<double>(x.z); ao[3] += static_cast<double>(x.w);
        } else {
          ae[0] += static_cast<double>(x.x); ae[1] += static_cast<double>(x.y);
          ae[2] += static_cast<double>(x.z); ae[3] += static_cast<double>(x.w);
        }
#endif
        }
      }
    }
    if (g.fl & GF_END) {
      if (g.fl & GF_OK) {
        if (g.fl & GF_SEG) {
          finish_seg(static_cast<int64_t>(g.r0) + qid);
        } else {
          const uint32_t ob = sm_own + buf * kFlatOwnBytes;
          double ownv[EPL];
          if constexpr (BITS) {
            const uint32_t wd = lds32(ob + qid * (L * 16)) >> (EPL * sub);
#pragma unroll
            for (int jj = 0; jj < EPL; ++jj) ownv[jj] = ((wd >> jj) & 1u) ? 1.0 : -1.0;
          } else if constexpr (EPL == 2) {
            const double2 v = lds128d(ob + lane * 16);
            ownv[0] = v.x; ownv[1] = v.y;
          } else {
            const float4 v = lds128(ob + lane * 16);
            ownv[0] = static_cast<double>(v.x); ownv[1] = static_cast<double>(v.y);
            ownv[2] = static_cast<double>(v.z); ownv[3] = static_cast<double>(v.w);
          }
          const double d = lds64(ob + 512 + qid * 16);
          const double dis = NL ? lds64(ob + 512 + qid * 16 + 8) : 0.0;
          finish_row(static_cast<int64_t>(g.r0) + qid, ownv, d, dis);
        }
      }
#pragma unroll
      for (int jj = 0; jj < EPL; ++jj) ae[jj] = ao[jj] = 0.0;
    }
  };
  auto issue = [&](const Group& g, int32_t col, int32_t col2, int buf) {
    if (g.fl & GF_LIVE) {
      if constexpr (BITS) {
        // this lane's own slot: the column index it loaded; invalid slots are zero-filled
        const uint32_t dst = sm_warp + buf * kFlatBatchBytes + (sub * RPW + qid) * 32;
        const unsigned char* src = recb + static_cast<uint64_t>(static_cast<uint32_t>(col)) * rec_stride;
        const int nb = ((g.nv >> sub) & 1) ? 16 : 0;
        if (L <= kFlatU || sub < kFlatU) {
          cp_async16(dst, src, nb);
          if (REC) cp_async16(dst + 16, src + 16, nb);
        }
        if (L == 4) {   // this lane's second slot
          const uint32_t dst2 = dst + 4 * RPW * 32;
          const unsigned char* src2 = recb + static_cast<uint64_t>(static_cast<uint32_t>(col2)) * rec_stride;
          const int nb2 = ((g.nv >> (sub + 4)) & 1) ? 16 : 0;
          cp_async16(dst2, src2, nb2);
          if (REC) cp_async16(dst2 + 16, src2 + 16, nb2);
        }
      } else {
        const uint32_t base = sm_ring + buf * kFlatBatchBytes;
#pragma unroll
        for (int q = 0; q < kFlatU; ++q) {
          const uint32_t c = static_cast<uint32_t>(__shfl_sync(FULL, q < L ? col : col2, qbase | (q & (L - 1))));
          cp_async16(base + q * 512, ugb + static_cast<uint64_t>(c) * strideb, ((g.nv >> q) & 1) ? 16 : 0);
        }
      }
      if ((g.fl & (GF_END | GF_SEG | GF_OK)) == (GF_END | GF_OK)) {
        const int64_t r = static_cast<int64_t>(g.r0) + qid;
        const uint32_t ob = sm_own + buf * kFlatOwnBytes;
        if constexpr (BITS) {
          if (sub == 2) cp_async16(ob + qid * (L * 16), a.bits + r * kBitWords, 16);
        } else {
          cp_async16(ob + lane * 16, uob + static_cast<uint64_t>(r) * strideb, lane_bytes);
        }
        if (sub == 0) cp_async8(ob + 512 + qid * 16, a.degree + r);
        if (NL && sub == 1) cp_async8(ob + 512 + qid * 16 + 8, a.dinv + r);
      }
    }
    cp_async_commit();
  };

  // g0: consumed this iteration; g1 (g2): in flight; gi: issued this iteration; gp: generated, its
  // column indices loading.  Live batches are contiguous: once a dead batch is generated (no items
  // left) every later one is dead, so the loop runs while the batch to consume is live.
  static_assert(kFlatNB == 3 || kFlatNB == 4, "ring depth");
  Group g0, g1, g2, gi, gp;
  int64_t mypos, mypos2;
  int32_t col_i, col_p, col2_i = 0, col2_p = 0;
  auto next = [&](Group& g, int32_t& col, int32_t& col2) {
    gen(g, mypos, mypos2);
    col = mypos >= 0 ? __ldg(cols + mypos) : 0;
    if (L == 4) col2 = mypos2 >= 0 ? __ldg(cols + mypos2) : 0;
  };
  // prologue: issue the first NB - 1 batches
  next(g0, col_i, col2_i);
  issue(g0, col_i, col2_i, 0);
  next(g1, col_i, col2_i);
  issue(g1, col_i, col2_i, 1);
  if (kFlatNB == 4) {
    next(g2, col_i, col2_i);
    issue(g2, col_i, col2_i, 2);
  }
  next(gi, col_i, col2_i);
  next(gp, col_p, col2_p);
  int cbuf = 0;            // buffer of the batch consumed this iteration
  int ibuf = kFlatNB - 1;  // buffer of the batch issued this iteration (consumed one iteration ago)
  while (g0.fl & GF_LIVE) {
    cp_async_wait<kFlatNB - 2>();
    __syncwarp();
    consume(g0, cbuf);
    issue(gi, col_i, col2_i, ibuf);
    ibuf = cbuf;
    cbuf = cbuf + 1 == kFlatNB ? 0 : cbuf + 1;
    g0 = g1;
    if (kFlatNB == 4) { g1 = g2; g2 = gi; } else { g1 = gi; }
    gi = gp;
    col_i = col_p;
    col2_i = col2_p;
    next(gp, col_p, col2_p);
  }
  cp_async_wait<0>();
}

template <typename VT, int KIND, bool BITS, int L = 8>
static bool flat_go(const SpmmArgs& a, cudaStream_t st) {
  const dim3 grid(148 * kFlatCtasPerSm);
  static std::atomic<bool> attr[64];
  if (!smem_optin(reinterpret_cast<const void*>(spmm_flat_kernel<VT, KIND, BITS, L>), kFlatSmem, attr)) return false;
  if (a.win_rows <= 0) {
    spmm_flat_kernel<VT, KIND, BITS, L><<<grid, kFlatThreads, kFlatSmem, st>>>(a);
    return true;
  }
  constexpr bool REC = KIND == SLQ_NORMALIZED_LAPLACIAN || KIND == kPair;
  const void* base = BITS ? static_cast<const void*>(REC ? a.rec : a.bits)
                          : ((KIND == kNLPre || KIND == kPair) ? a.upre : a.u);
  const size_t row_bytes = BITS ? sizeof(uint32_t) * (REC ? kRecWords : kBitWords)
                                : sizeof(VT) * static_cast<size_t>(a.ldc_in);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kFlatThreads);
  cfg.dynamicSmemBytes = kFlatSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  at[0].val.accessPolicyWindow.num_bytes = row_bytes * static_cast<size_t>(a.win_rows);
  at[0].val.accessPolicyWindow.hitRatio = 1.0f;
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, spmm_flat_kernel<VT, KIND, BITS, L>, a);
  l2_demote(base, at[0].val.accessPolicyWindow.num_bytes, st);
  return true;
}

// True when the flat kernel took the launch (gathered rows of <= 128 bytes: <= 32 fp32 or <= 16 fp64
// probes, unit weights, the Lanczos path, a graph with fine tiles); the caller falls back to spmm_kernel.
template <typename VT>
static bool launch_flat(int kind, const SpmmArgs& a, cudaStream_t st) {
  constexpr int EPL = 16 / static_cast<int>(sizeof(VT));
  constexpr int kMaxCols = EPL == 2 ? 32 : 32;   // 128-byte rows (fp32), 256-byte rows (fp64): the narrow class
  if (!a.ftile_rows || a.nftiles <= 0 || a.weights || !a.r) return false;
  if (a.ldc_in > kMaxCols || a.ldc_out > kMaxCols || a.c > kMaxCols || (a.ldc_in & (EPL - 1)) || (a.ldc_out & (EPL - 1)) ||
      a.ldc_in < EPL)
    return false;
  const bool narrow = a.ldc_in <= 4 * EPL;   // 64-byte rows: 4 lanes per row
  const bool wide16 = a.ldc_in > 8 * EPL;    // 256-byte rows (17..32 fp64 probes): 16 lanes per row
  if (a.n_rows >= (int64_t(1) << 29) || a.max_seg >= (int64_t(1) << 29)) return false;
  // the normalized Laplacian needs dinv[col] per nonzero: prescaled gathers, or the first step's records
  if (kind == SLQ_NORMALIZED_LAPLACIAN && !(a.bits ? a.rec != nullptr : a.upre != nullptr)) return false;
  const bool pair = a.split < a.c;
  if (pair && (kind != SLQ_NORMALIZED_LAPLACIAN || (a.split & (EPL - 1)) || narrow || EPL != 4)) return false;
  LaunchScope ls(K_SPMM, st);
  if constexpr (EPL == 4) {
    if (pair) return a.bits ? flat_go<VT, kPair, true>(a, st) : flat_go<VT, kPair, false>(a, st);
  }
  if constexpr (EPL == 2) {
    if (wide16) {
      if (a.bits) {
        if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, SLQ_NORMALIZED_LAPLACIAN, true, 16>(a, st);
        if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, true, 16>(a, st);
        return flat_go<VT, SLQ_LAPLACIAN, true, 16>(a, st);
      }
      if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, kNLPre, false, 16>(a, st);
      if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, false, 16>(a, st);
      return flat_go<VT, SLQ_LAPLACIAN, false, 16>(a, st);
    }
  }
  if (narrow) {
    if (a.bits) {
      if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, SLQ_NORMALIZED_LAPLACIAN, true, 4>(a, st);
      if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, true, 4>(a, st);
      return flat_go<VT, SLQ_LAPLACIAN, true, 4>(a, st);
    }
    if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, kNLPre, false, 4>(a, st);
    if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, false, 4>(a, st);
    return flat_go<VT, SLQ_LAPLACIAN, false, 4>(a, st);
  }
  if (a.bits) {
    if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, SLQ_NORMALIZED_LAPLACIAN, true>(a, st);
    if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, true>(a, st);
    return flat_go<VT, SLQ_LAPLACIAN, true>(a, st);
  }
  if (kind == SLQ_NORMALIZED_LAPLACIAN) return flat_go<VT, kNLPre, false>(a, st);
  if (kind == SLQ_DENSITY) return flat_go<VT, SLQ_DENSITY, false>(a, st);
  return flat_go<VT, SLQ_LAPLACIAN, false>(a, st);
}

bool launch_spmm_flat_f32(int kind, const SpmmArgs& a, cudaStream_t st) { return launch_flat<float>(kind, a, st); }
bool launch_spmm_flat_f64(int kind, const SpmmArgs& a, cudaStream_t st) { return launch_flat<double>(kind, a, st); }

}  // namespace slq
