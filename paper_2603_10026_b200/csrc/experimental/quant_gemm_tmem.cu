// EXPERIMENTAL, NOT BUILT INTO librf_cuda (measured slower than qnt2 — see
// profiles/r2_fp8_investigation.md, "Round 2, session 3"). Two FP8 quant GEMM
// variants kept for reference; this is a fragment of gemm_sm100.cu's anonymous
// namespace (it uses tile_of, sw128, qnt::Params with extra `int wb, wr, exp;`
// fields, QTRACE) and compiles only when pasted back there:
//   * quant_gemm_tmem_kernel: e4m3 A written by 8 quantiser warps straight into
//     TMEM (tcgen05.st) and consumed by kind::f8f6f4 TS MMAs; N tiles <= 448
//     (TMEM = accumulator + two 32-column A8 stages). 2136-2162 TFLOP/s vs
//     qnt2's 2302 on one box (9 waves of 448-wide tiles vs 7 of 512; per
//     column ~5 % faster).
//   * quant_gemm_x4_kernel: clusters of two CTA pairs on adjacent N tiles of
//     the same rows, each A half TMA-multicast to both pairs (half the L2 reads
//     of A). 1878-1900 TFLOP/s. (Reading the partner's half with
//     ld.shared::cluster instead: 660 TFLOP/s, ~3600 cycles per 16 KB.)

// ------------------------------------------- QUANT_GEMM, 2-SM, A8 in TMEM --
//
// The 2-SM kernel above is bound by each SM's shared-memory port, not by the
// tensor pipe (profiles/r2_fp8_investigation.md): per K step a CTA moves
// ~176 KB through shared memory, ~48 KB of it the e4m3 A tile (quantiser
// writes + the MMAs' reads, once per N = 256 half). Here the quantiser writes
// its e4m3 row straight into TMEM (tcgen05.st, thread = row = TMEM lane) and
// the MMAs read A from TMEM (kind::f8f6f4 TS form); shared memory carries
// only the TMA-staged bf16 A tile (read once by the quantiser) and W.
// TMEM then holds the accumulator AND two 32-column A8 stages, so a tile is at
// most 448 columns wide (2 MMAs of N <= 224 per K step). N is cut into
// T = ceil(N / 448) tiles of widths wb or wb + 64 (multiples of 64, as even as
// possible): cfg4's N = 8192 is 14 tiles of 448 + 5 of 384.

namespace qnt3 {

using qnt::BK;
constexpr int BNMAX = 448;
constexpr int S8 = 2;
constexpr int NQW = 8;                   // quantiser + epilogue warps (2 per TMEM lane quarter)
constexpr int TMA_WARP = NQW, MMA_WARP = NQW + 1;  // MMA issue (leader) / peer relay
constexpr int NT = 32 * (NQW + 2);
constexpr int ABF_BYTES = BM * BK * 2;        // 32 KB
constexpr int W_BYTES = (BNMAX / 2) * BK;     // 28 KB: this CTA's quarter of each N half
constexpr uint32_t A8_COL = BNMAX;            // TMEM columns [448, 512): A8 stages

template <int SA, int SW>
struct Smem {
  uint8_t abf[SA][ABF_BYTES];
  uint8_t w[SW][W_BYTES];
  uint64_t abf_full[SA], abf_empty[SA], w_full[SW], w_empty[SW], a8_full[S8], a8_empty[S8];
  uint64_t acc_full;
  float xmax[2][2][BM];  // [K step parity][K half][row]: half-tile absmax exchange
  uint32_t tmem_base;
};

__device__ __forceinline__ void mma_f8_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int SA, int SW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    quant_gemm_tmem_kernel(const __grid_constant__ CUtensorMap ta,
                           const __grid_constant__ CUtensorMap tw_hi,
                           const __grid_constant__ CUtensorMap tw_lo,
                           const __grid_constant__ CUtensorMap tc, const qnt::Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem<SA, SW>& s = *reinterpret_cast<Smem<SA, SW>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  int mt, nt;
  tile_of(blockIdx.x >> 1, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const bool wide = nt < p.wr;
  const int wn = wide ? p.wb + 64 : p.wb;  // tile width (N columns)
  const int wq = wn / 4;                   // W rows per CTA per N half
  const int n0 = nt * p.wb + 64 * min(nt, p.wr);
  const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);
  if (threadIdx.x == 0) QTRACE(7, 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&s.abf_full[i], 1);
      mbar_init(&s.abf_empty[i], NQW);
    }
    for (int i = 0; i < SW; ++i) {
      mbar_init(&s.w_full[i], 1);
      mbar_init(&s.w_empty[i], 1);
    }
    for (int i = 0; i < S8; ++i) {
      mbar_init(&s.a8_full[i], leader ? NQW + 1 : NQW);  // leader: + peer relay
      mbar_init(&s.a8_empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (threadIdx.x == 0) QTRACE(7, 3);  // common origin of the pair's clocks

  if (warp == TMA_WARP) {
    if (elect_one()) {
      const CUtensorMap* tw = wide ? &tw_hi : &tw_lo;
      prefetch_tmap(&ta);
      prefetch_tmap(tw);
      prefetch_tmap(&tc);
      const uint32_t wbytes = static_cast<uint32_t>(2 * wq * BK);
      for (int t = 0; t < kt; ++t) {
        const int sa = t % SA, sw = t % SW;
        mbar_wait(&s.abf_empty[sa], ((t / SA) & 1) ^ 1);
        QTRACE(5, t);
        mbar_arrive_expect_tx(&s.abf_full[sa], ABF_BYTES);
        tma_load_2d(s.abf[sa], &ta, &s.abf_full[sa], k0 + t * BK, m0, kEvictFirst);
        tma_load_2d(s.abf[sa] + BM * 128, &ta, &s.abf_full[sa], k0 + t * BK + 64, m0, kEvictFirst);
        mbar_wait(&s.w_empty[sw], ((t / SW) & 1) ^ 1);
        QTRACE(6, t);
        mbar_arrive_expect_tx(&s.w_full[sw], wbytes);
        for (int h = 0; h < 2; ++h)
          tma_load_2d(s.w[sw] + h * wq * 128, tw, &s.w_full[sw], k0 + t * BK,
                      n0 + h * (wn / 2) + static_cast<int>(rank) * wq, kEvictLast);
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader) {
      const uint32_t idesc = idesc_f8(2 * BM, static_cast<uint32_t>(wn / 2));
      const bool el = elect_one();
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        mbar_wait(&s.w_full[sw], (t / SW) & 1);
        if (el) QTRACE(0, t);
        mbar_wait(&s.a8_full[s8], (t / S8) & 1);  // own A8 + peer (W + A8) relay
        if (el) QTRACE(1, t);
        tc_fence_after();
        if (el) {
          const uint32_t a = tmem + A8_COL + 32 * s8, b = smem_u32(s.w[sw]);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks)
              mma_f8_ts_2sm(tmem + h * (wn / 2), a + ks * 8,
                            sdesc_kmajor_sw128(b + h * wq * 128 + ks * 32), idesc, (t | ks) != 0);
          mma_commit_2sm(&s.w_empty[sw]);
          mma_commit_2sm(&s.a8_empty[s8]);
          if (t + 1 == kt) mma_commit_2sm(&s.acc_full);
        }
        __syncwarp();
      }
    } else if (elect_one()) {
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        mbar_wait(&s.w_full[sw], (t / SW) & 1);
        mbar_wait(&s.a8_full[s8], (t / S8) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.a8_full[s8]), 0));
      }
    }
  } else {
    // Quantiser: warps q and q + 4 own TMEM lane quarter q (rows 32q..32q+31,
    // thread = row) and K half kh of every 128-wide tile; the tile absmax of a
    // row is the max of the two halves, exchanged through shared memory.
    const int kh = warp >> 2;
    const int r = threadIdx.x & (BM - 1);
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t pair_bar = 2 + (warp & 3);  // named barriers 2..5: warps q, q + 4
    const int nch = wn / 32;                   // 32-column accumulator chunks
    const int c_lo = kh * (nch / 2), c_hi = c_lo + nch / 2;  // this warp's half of them
    float amax = 0.f, ref = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int sa = t % SA, s8 = t % S8;
      mbar_wait(&s.abf_full[sa], (t / SA) & 1);
      if (threadIdx.x == 0) QTRACE(2, t);
      uint32_t x[32];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint4 q = lds128(smem_u32(s.abf[sa]) + kh * (BM * 128) + sw128(r, v));
        x[4 * v + 0] = q.x;
        x[4 * v + 1] = q.y;
        x[4 * v + 2] = q.z;
        x[4 * v + 3] = q.w;
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.abf_empty[sa]);
      uint32_t mc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mc[i] = qnt::absmax_bf16x2(x[i], x[i + 8]);
#pragma unroll
      for (int i = 16; i < 32; ++i) mc[i & 7] = qnt::absmax_bf16x2(mc[i & 7], x[i]);
#pragma unroll
      for (int w = 4; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) mc[i] = qnt::absmax_bf16x2(mc[i], mc[i + w]);
      const uint32_t mx = mc[0];
      float half_max = fmaxf(__uint_as_float((mx << 16) & 0x7fffffffu),
                             __uint_as_float(mx & 0x7fff0000u));
      s.xmax[t & 1][kh][r] = half_max;
      named_bar_sync(pair_bar, 64);
      const float tile_max = fmaxf(half_max, s.xmax[t & 1][kh ^ 1][r]);
      amax = fmaxf(amax, tile_max);
      const float nref = qnt::pow2_ceil(amax);
      const bool changed = t > 0 && nref != ref;
      if (__any_sync(0xffffffffu, changed)) {
        // In-loop correction ref/ref' of this CTA's accumulator rows, once the
        // MMAs of tile t-1 (the last to use the old scale) have retired.
        const int sp = (t - 1) % S8;
        mbar_wait(&s.a8_empty[sp], ((t - 1) / S8) & 1);
        tc_fence_after();
        const float f = changed ? ref / nref : 1.f;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * f);
          tmem_st32(tmem + lane_off + c * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
      }
      ref = nref;
      const float sc = ref > 0.f ? p.fmax / ref : 0.f;  // see quant_gemm_kernel
      uint64_t sc2;
      asm("mov.b64 %0, {%1, %1};" : "=l"(sc2) : "f"(sc));
      uint32_t q8[16];  // TMEM column 16 kh + j = e4m3 elements 4j .. 4j+3 of this K half
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t lo = qnt::quant_pair(x[2 * j], sc2);
        const uint32_t hi = qnt::quant_pair(x[2 * j + 1], sc2);
        q8[j] = (lo & 0xffffu) | (hi << 16);
      }
      mbar_wait(&s.a8_empty[s8], ((t / S8) & 1) ^ 1);
      if (threadIdx.x == 0) QTRACE(3, t);
      tc_fence_after();
      tmem_st16(tmem + lane_off + A8_COL + 32 * s8 + 16 * kh, q8);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) QTRACE(4, t);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.a8_full[s8]);
    }
    const float fin = p.partial ? ref : ref / amax;
    if (kh == 0) {
      if (p.partial) {
        if (nt == 0) p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = amax;
      } else {
        if (!(amax > 0.f)) atomicExch(p.domain_flag, 1);
        if (nt == 0) p.d1[m0 + r] = amax;
      }
    }
    const int crow = p.partial ? static_cast<int>(blockIdx.y * p.ws_rows) + m0 : m0;
    const uint32_t grp_bar = 6 + kh;  // the 4 warps of this K half
    const bool grp_lead = (threadIdx.x & (BM - 1)) == 0;
    named_bar_sync(grp_bar, BM);
    mbar_wait(&s.acc_full, 0);
    if (threadIdx.x == 0) QTRACE(7, 0);
    tc_fence_after();
    // C tile (128 rows x wn fp32 columns): warp group kh stores chunks
    // [c_lo, c_hi) in rounds of 2 chunks through two 32 KB staging areas of
    // the drained rings (its own pair of them).
    uint8_t* const base = reinterpret_cast<uint8_t*>(&s) + kh * (4 * BM * 128);
    uint8_t* const area[2] = {base, base + 2 * (BM * 128)};
    uint32_t v[2][32];
    tmem_ld32(tmem + lane_off + c_lo * 32, v[0]);
    const int my = c_hi - c_lo;
    const int rounds = (my + 1) / 2;
#pragma unroll 1
    for (int rnd = 0; rnd < rounds; ++rnd) {
      if (rnd >= 2) {
        if (grp_lead) bulk_wait_read1();
        named_bar_sync(grp_bar, BM);
      }
      const uint32_t stage = smem_u32(area[rnd & 1]);
      const int cn = min(2, my - 2 * rnd);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c < cn) {
          const int cc = c_lo + 2 * rnd + c;
          tmem_ld_wait();
          if (cc + 1 < c_hi) tmem_ld32(tmem + lane_off + (cc + 1) * 32, v[(c + 1) & 1]);
          const uint32_t chunk = stage + c * (BM * 128);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            sts128(chunk + sw128(r, u),
                   make_uint4(__float_as_uint(__uint_as_float(v[c & 1][4 * u]) * fin),
                              __float_as_uint(__uint_as_float(v[c & 1][4 * u + 1]) * fin),
                              __float_as_uint(__uint_as_float(v[c & 1][4 * u + 2]) * fin),
                              __float_as_uint(__uint_as_float(v[c & 1][4 * u + 3]) * fin)));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(grp_bar, BM);
      if (grp_lead) {
        for (int c = 0; c < cn; ++c)
          tma_store_2d(&tc, area[rnd & 1] + c * (BM * 128), n0 + 32 * (c_lo + 2 * rnd + c), crow);
        bulk_commit();
      }
    }
    if (grp_lead) bulk_wait0();
    if (threadIdx.x == 0) QTRACE(7, 1);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == MMA_WARP) tmem_dealloc_2sm<512>(tmem);
}

// ------------------------------------------------ cluster of two CTA pairs --
//
// Both kernels above read every A row once per N tile through L2 (bf16, the
// larger operand), and at ~38 B/clk/SM of TMA traffic the whole chip sits near
// the L2 -> SM throughput ceiling (~6000 B/clk, the same ceiling cuBLASLt's
// e4m3 GEMM reaches). Here a cluster holds two CTA pairs on adjacent N tiles
// of the SAME rows: CTA (pair p, rank r) TMA-loads K half p of its rows' bf16
// A tile and multicasts it to itself and its partner (pair 1-p, rank r), so
// each A half is read from L2 once for both N tiles. A slot is refilled only
// when the quantisers of both CTAs released it (abf_empty counts 8 local + 8
// remote warp arrivals). (Measured and dropped: reading the partner's half
// through ld.shared::cluster — ~3600 cycles per 16 KB per CTA.)

template <int SA, int SW>
struct SmemX4 {
  uint8_t abf[SA][ABF_BYTES];
  uint8_t w[SW][W_BYTES];
  uint64_t abf_full[SA], abf_empty[SA], w_full[SW], w_empty[SW], a8_full[S8], a8_empty[S8];
  uint64_t acc_full;
  float xmax[2][2][BM];
  uint32_t tmem_base;
};

template <int SA, int SW>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(NT, 1)
    quant_gemm_x4_kernel(const __grid_constant__ CUtensorMap ta,
                         const __grid_constant__ CUtensorMap tw_hi,
                         const __grid_constant__ CUtensorMap tw_lo,
                         const __grid_constant__ CUtensorMap tc, const qnt::Params p) {
  extern __shared__ uint8_t smem_raw[];
  SmemX4<SA, SW>& s =
      *reinterpret_cast<SmemX4<SA, SW>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1, pr = crank >> 1;  // MMA-pair rank, pair index in the cluster
  const uint32_t partner = crank ^ 2;               // same rows, other N tile
  const bool leader = rank == 0;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pr));
  const uint16_t row_mask = static_cast<uint16_t>((1u << crank) | (1u << partner));
  int mt, ntp;
  tile_of(blockIdx.x >> 2, p.mt_count, p.nt_count / 2, p.group_n, mt, ntp);
  const int nt = 2 * ntp + static_cast<int>(pr);
  const bool wide = nt < p.wr;
  const int wn = wide ? p.wb + 64 : p.wb;
  const int wq = wn / 4;
  const int n0 = nt * p.wb + 64 * min(nt, p.wr);
  const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);
  if (threadIdx.x == 0) QTRACE(7, 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&s.abf_full[i], 1);
      mbar_init(&s.abf_empty[i], 2 * NQW);
    }
    for (int i = 0; i < SW; ++i) {
      mbar_init(&s.w_full[i], 1);
      mbar_init(&s.w_empty[i], 1);
    }
    for (int i = 0; i < S8; ++i) {
      mbar_init(&s.a8_full[i], leader ? NQW + 1 : NQW);
      mbar_init(&s.a8_empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (threadIdx.x == 0) QTRACE(7, 3);

  if (warp == TMA_WARP) {
    if (elect_one()) {
      const CUtensorMap* tw = wide ? &tw_hi : &tw_lo;
      prefetch_tmap(&ta);
      prefetch_tmap(tw);
      prefetch_tmap(&tc);
      const uint32_t wbytes = static_cast<uint32_t>(2 * wq * BK);
      for (int t = 0; t < kt; ++t) {
        const int sa = t % SA, sw = t % SW;
        mbar_wait(&s.abf_empty[sa], ((t / SA) & 1) ^ 1);  // both CTAs' quantisers released it
        QTRACE(5, t);
        mbar_arrive_expect_tx(&s.abf_full[sa], ABF_BYTES);  // our half + the partner's
        tma_load_2d_mc(s.abf[sa] + pr * (BM * 128), &ta, &s.abf_full[sa], k0 + t * BK + 64 * static_cast<int>(pr),
                       m0, row_mask, kEvictFirst);
        mbar_wait(&s.w_empty[sw], ((t / SW) & 1) ^ 1);
        QTRACE(6, t);
        mbar_arrive_expect_tx(&s.w_full[sw], wbytes);
        for (int h = 0; h < 2; ++h)
          tma_load_2d(s.w[sw] + h * wq * 128, tw, &s.w_full[sw], k0 + t * BK,
                      n0 + h * (wn / 2) + static_cast<int>(rank) * wq, kEvictLast);
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader) {
      const uint32_t idesc = idesc_f8(2 * BM, static_cast<uint32_t>(wn / 2));
      const bool el = elect_one();
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        if (!(p.exp & 2)) mbar_wait(&s.w_full[sw], (t / SW) & 1);
        if (el) QTRACE(0, t);
        if (!(p.exp & 1)) mbar_wait(&s.a8_full[s8], (t / S8) & 1);
        if (el) QTRACE(1, t);
        tc_fence_after();
        if (el) {
          const uint32_t a = tmem + A8_COL + 32 * s8, b = smem_u32(s.w[sw]);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks)
              mma_f8_ts_2sm(tmem + h * (wn / 2), a + ks * 8,
                            sdesc_kmajor_sw128(b + h * wq * 128 + ks * 32), idesc, (t | ks) != 0);
          mma_commit_2sm(&s.w_empty[sw], pair_mask);
          mma_commit_2sm(&s.a8_empty[s8], pair_mask);
          if (t + 1 == kt) mma_commit_2sm(&s.acc_full, pair_mask);
        }
        __syncwarp();
      }
    } else if (elect_one()) {
      const uint32_t lead = crank & ~1u;
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        mbar_wait(&s.w_full[sw], (t / SW) & 1);
        mbar_wait(&s.a8_full[s8], (t / S8) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.a8_full[s8]), lead));
      }
    }
  } else {
    const int kh = warp >> 2;
    const int r = threadIdx.x & (BM - 1);
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t pair_bar = 2 + (warp & 3);
    const int nch = wn / 32;
    const int c_lo = kh * (nch / 2), c_hi = c_lo + nch / 2;
    float amax = 0.f, ref = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int sa = t % SA, s8 = t % S8;
      mbar_wait(&s.abf_full[sa], (t / SA) & 1);
      if (threadIdx.x == 0) QTRACE(2, t);
      uint32_t x[32];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint4 q = lds128(smem_u32(s.abf[sa]) + kh * (BM * 128) + sw128(r, v));
        x[4 * v + 0] = q.x;
        x[4 * v + 1] = q.y;
        x[4 * v + 2] = q.z;
        x[4 * v + 3] = q.w;
      }
      uint32_t mc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mc[i] = qnt::absmax_bf16x2(x[i], x[i + 8]);
#pragma unroll
      for (int i = 16; i < 32; ++i) mc[i & 7] = qnt::absmax_bf16x2(mc[i & 7], x[i]);
#pragma unroll
      for (int w = 4; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) mc[i] = qnt::absmax_bf16x2(mc[i], mc[i + w]);
      const uint32_t mx = mc[0];
      // every element of x has been consumed: release the slot in both CTAs
      // (the partner's producer multicasts into ours)
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        mbar_arrive(&s.abf_empty[sa]);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.abf_empty[sa]), partner));
      }
      float half_max = fmaxf(__uint_as_float((mx << 16) & 0x7fffffffu),
                             __uint_as_float(mx & 0x7fff0000u));
      s.xmax[t & 1][kh][r] = half_max;
      named_bar_sync(pair_bar, 64);
      const float tile_max = fmaxf(half_max, s.xmax[t & 1][kh ^ 1][r]);
      amax = fmaxf(amax, tile_max);
      const float nref = qnt::pow2_ceil(amax);
      const bool changed = t > 0 && nref != ref;
      if (__any_sync(0xffffffffu, changed)) {
        const int sp = (t - 1) % S8;
        mbar_wait(&s.a8_empty[sp], ((t - 1) / S8) & 1);
        tc_fence_after();
        const float f = changed ? ref / nref : 1.f;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * f);
          tmem_st32(tmem + lane_off + c * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
      }
      ref = nref;
      const float sc = ref > 0.f ? p.fmax / ref : 0.f;
      uint64_t sc2;
      asm("mov.b64 %0, {%1, %1};" : "=l"(sc2) : "f"(sc));
      uint32_t q8[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t lo = qnt::quant_pair(x[2 * j], sc2);
        const uint32_t hi = qnt::quant_pair(x[2 * j + 1], sc2);
        q8[j] = (lo & 0xffffu) | (hi << 16);
      }
      mbar_wait(&s.a8_empty[s8], ((t / S8) & 1) ^ 1);
      if (threadIdx.x == 0) QTRACE(3, t);
      tc_fence_after();
      if (!(p.exp & 4)) tmem_st16(tmem + lane_off + A8_COL + 32 * s8 + 16 * kh, q8);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) QTRACE(4, t);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.a8_full[s8]);
    }
    const float fin = p.partial ? ref : ref / amax;
    if (kh == 0) {
      if (p.partial) {
        if (nt == 0) p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = amax;
      } else {
        if (!(amax > 0.f)) atomicExch(p.domain_flag, 1);
        if (nt == 0) p.d1[m0 + r] = amax;
      }
    }
    const int crow = p.partial ? static_cast<int>(blockIdx.y * p.ws_rows) + m0 : m0;
    const uint32_t grp_bar = 6 + kh;
    const bool grp_lead = (threadIdx.x & (BM - 1)) == 0;
    named_bar_sync(grp_bar, BM);
    mbar_wait(&s.acc_full, 0);
    if (threadIdx.x == 0) QTRACE(7, 0);
    tc_fence_after();
    // C tile: K-half group kh stores chunks [c_lo, c_hi) one at a time through
    // two 16 KB staging areas in the drained W ring (drained for both CTAs of
    // the MMA pair once acc_full fired).
    uint8_t* const base = reinterpret_cast<uint8_t*>(s.w) + kh * (2 * BM * 128);
    uint8_t* const area[2] = {base, base + BM * 128};
    uint32_t v[2][32];
    tmem_ld32(tmem + lane_off + c_lo * 32, v[0]);
    const int my = c_hi - c_lo;
#pragma unroll 1
    for (int cc = 0; cc < my; ++cc) {
      if (cc >= 2) {
        if (grp_lead) bulk_wait_read1();
        named_bar_sync(grp_bar, BM);
      }
      const uint32_t chunk = smem_u32(area[cc & 1]);
      tmem_ld_wait();
      if (cc + 1 < my) tmem_ld32(tmem + lane_off + (c_lo + cc + 1) * 32, v[(cc + 1) & 1]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        sts128(chunk + sw128(r, u),
               make_uint4(__float_as_uint(__uint_as_float(v[cc & 1][4 * u]) * fin),
                          __float_as_uint(__uint_as_float(v[cc & 1][4 * u + 1]) * fin),
                          __float_as_uint(__uint_as_float(v[cc & 1][4 * u + 2]) * fin),
                          __float_as_uint(__uint_as_float(v[cc & 1][4 * u + 3]) * fin)));
      fence_proxy_async_smem();
      named_bar_sync(grp_bar, BM);
      if (grp_lead) {
        tma_store_2d(&tc, area[cc & 1], n0 + 32 * (c_lo + cc), crow);
        bulk_commit();
      }
    }
    if (grp_lead) bulk_wait0();
    if (threadIdx.x == 0) QTRACE(7, 1);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == MMA_WARP) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace qnt3
