// EXPERIMENTAL, NOT BUILT INTO librf_cuda (measured slower than rms2 — see
// DESIGN.md §3.3, "Round 2: A in TMEM for the RMS / LayerNorm GEMM"). A
// fragment of gemm_sm100.cu's anonymous namespace (uses rms::Params with extra
// `int wb, wr, exp;` fields, tile_of, sw128, rms2::BK); compiles only when
// pasted back there. Parity-green (test_gpu_gemm, fullshape, fused) at
// 1299-1336 TFLOP/s on cfg5 vs rms2's 1449-1465 in same-box A/Bs.

// ------------------------------------------ RMS / LayerNorm, 2-SM, A in TMEM --
//
// The 2-SM kernel above issues bf16 SS MMAs (N = 256), which on this B200 run
// at ~0.73 of the tensor rate even alone (a fixed ~43-cycle operand overhead
// per K = 16 instruction); with A in TMEM (TS) the same MMAs run
// at ~0.9. The statistics warps already read every A row from shared memory
// for sum x^2: here they also write it (bf16, thread = row = TMEM lane) into
// one of two 32-column TMEM stages, and the MMA reads A from there. TMEM per
// CTA = accumulator (<= 192 columns) + 2 A stages = 256, so two CTA pairs
// still share an SM pair and one pair's epilogue overlaps the other's
// mainloop. N is cut into T = ceil(N / 192) tiles of widths wb / wb + 64
// (multiples of 64; cfg5's 11008 = 56 x 192 + 2 x 128).
// Sync: the MMA waits only on a_full (4 own statistics warps + the peer's
// relay of its own a_full): a warp arrives after it saw its TMA tiles land
// and wrote its rows, so a_full also covers both CTAs' W halves. a_empty is
// the MMA's multicast commit (the A stage may be rewritten); `empty` frees the
// shared-memory stage (MMA commit: W read; 4 statistics warps: A read).

namespace rms3 {

using rms2::BK;
constexpr int STAGES = 4;  // the MMA now also waits on the statistics warps: one more stage of lookahead
constexpr int NSW = 8;  // statistics warps: warp w owns TMEM lane quarter w & 3 and K half w >> 2
constexpr int TMA_WARP = NSW, MMA_WARP = NSW + 1;
constexpr int NT = 32 * (NSW + 2);
constexpr int WMAX = 192;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB
constexpr int B_BYTES = (WMAX / 2) * BK * 2;  // 12 KB: this CTA's half of the tile's W rows
constexpr uint32_t A_COL = WMAX;             // TMEM columns [192, 256): four A stages of K = 32
constexpr int NAS = 4;                       // A stages (16 columns = 32 bf16 of K each)

struct Smem {
  uint8_t a[STAGES][A_BYTES];
  uint8_t b[STAGES][B_BYTES];
  uint64_t full[STAGES];   // own TMA bytes (A + W half)
  uint64_t empty[STAGES];  // MMA multicast commit + 8 statistics warps
  uint64_t a_full[NAS];    // 4 statistics warps (one K half) + on the leader the peer's relay
  uint64_t a_empty[NAS];   // MMA multicast commit
  uint64_t acc_full;
  uint32_t tmem_base;
};
// two CTAs of ~113 KB per SM: no alignment slack (the dynamic window starts
// 1024-aligned when there is no static shared memory; checked at entry)
static_assert(2 * (sizeof(Smem) + 1024) <= 228 * 1024, "two CTAs per SM");

// store_acc_f32 with a run-time column count (a multiple of 32 * RND).
template <int RND>
__device__ __forceinline__ void store_acc_f32_n(uint32_t tmem_row, int r, uint8_t* stage_ptr,
                                                const CUtensorMap* tm, int n0, int row0, int ncols) {
  const uint32_t stage = smem_u32(stage_ptr);
#pragma unroll 1
  for (int c0 = 0; c0 < ncols / 32; c0 += RND) {
#pragma unroll 1
    for (int c = 0; c < RND; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem_row + (c0 + c) * 32, v);
      tmem_ld_wait();
      const uint32_t chunk = stage + c * (BM * 128);
#pragma unroll
      for (int u = 0; u < 8; ++u) sts128(chunk + sw128(r, u), make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
      for (int c = 0; c < RND; ++c) tma_store_2d(tm, stage_ptr + c * (BM * 128), n0 + (c0 + c) * 32, row0);
      bulk_commit();
      bulk_wait_read0();
    }
    named_bar_sync(1, 128);
  }
}

template <bool LN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 2)
    rms_gemm_ts_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb_hi,
                       const __grid_constant__ CUtensorMap tb_lo, const __grid_constant__ CUtensorMap ty,
                       const __grid_constant__ CUtensorMap ty4, const rms::Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  int mt, nt;  // mt: 256-row pair tile
  tile_of(blockIdx.x >> 1, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const bool wide = nt < p.wr;
  const int wn = wide ? p.wb + 64 : p.wb;  // tile width
  const int wh = wn / 2;                   // this CTA's W rows
  const int n0 = nt * p.wb + 64 * min(nt, p.wr);
  const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1 + NSW);
    }
    for (int i = 0; i < NAS; ++i) {
      mbar_init(&s.a_full[i], leader ? 4 + 1 : 4);  // the 4 warps of one K half (+ peer relay)
      mbar_init(&s.a_empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc_2sm<256>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == TMA_WARP) {
    if (elect_one()) {
      const CUtensorMap* tb = wide ? &tb_hi : &tb_lo;
      prefetch_tmap(&ta);
      prefetch_tmap(tb);
      prefetch_tmap(&ty);
      if (LN) prefetch_tmap(&ty4);
      const uint32_t bytes = static_cast<uint32_t>(A_BYTES + wh * BK * 2);
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.empty[st], ((t / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[st], bytes);
        tma_load_2d(s.a[st], &ta, &s.full[st], k0 + t * BK, m0, kEvictNormal);
        tma_load_2d(s.b[st], tb, &s.full[st], k0 + t * BK, n0 + static_cast<int>(rank) * wh, kEvictLast);
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader) {
      const uint32_t idesc = idesc_f16(2 * BM, static_cast<uint32_t>(wn), kFmtBF16, false, false);
      const bool el = elect_one();
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        const uint32_t b = smem_u32(s.b[st]);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // K halves of the tile: one A stage each
          const int h = 2 * t + hf, j = h % NAS;
          mbar_wait(&s.a_full[j], (h / NAS) & 1);  // both CTAs: A rows in TMEM, TMA tiles landed
          tc_fence_after();
          if (el) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int ks = 2 * hf + kk;
              mma_f16_ts_2sm(tmem, tmem + A_COL + 16 * j + kk * 8, sdesc_kmajor_sw128(b + ks * 32), idesc,
                             (t | ks) != 0);
            }
            mma_commit_2sm(&s.a_empty[j]);
            if (hf == 1) {
              mma_commit_2sm(&s.empty[st]);
              if (t + 1 == kt) mma_commit_2sm(&s.acc_full);
            }
          }
          __syncwarp();
        }
      }
    } else if (elect_one()) {
      // relay: this CTA's A rows are in TMEM (and its tiles landed) -> the leader
      for (int h = 0; h < 2 * kt; ++h) {
        const int j = h % NAS;
        mbar_wait(&s.a_full[j], (h / NAS) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.a_full[j]), 0));
      }
    }
  } else {
    const int kh = warp >> 2;               // K half: 32 of the tile's 64 columns
    const int r = threadIdx.x & (BM - 1);   // row = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float ss = 0.f, sx = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int st = t % STAGES;
      mbar_wait(&s.full[st], (t / STAGES) & 1);
      const uint32_t row = smem_u32(s.a[st]) + (r >> 3) * 1024 + (r & 7) * 128;
      uint32_t w[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 v = lds128(row + (((4 * kh + u) ^ (r & 7)) << 4));
        w[4 * u] = v.x;
        w[4 * u + 1] = v.y;
        w[4 * u + 2] = v.z;
        w[4 * u + 3] = v.w;
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.empty[st]);  // this warp's A reads are done
      // A half row -> TMEM stage (column c = K elements 2c, 2c + 1) once the
      // MMAs of the stage's previous reader have retired
      const int h = 2 * t + kh, j = h % NAS;
      mbar_wait(&s.a_empty[j], ((h / NAS) & 1) ^ 1);
      tc_fence_after();
      tmem_st16(tmem + lane_off + A_COL + 16 * j, w);
      float ts[4] = {0.f, 0.f, 0.f, 0.f}, tx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float lo = bf_lo(w[q]), hi = bf_hi(w[q]);
        ts[q & 3] = fmaf(lo, lo, ts[q & 3]);
        ts[q & 3] = fmaf(hi, hi, ts[q & 3]);
        if (LN) tx[q & 3] += lo + hi;
      }
      ss += (ts[0] + ts[1]) + (ts[2] + ts[3]);  // per-tile partials: pairwise accumulation
      if (LN) sx += (tx[0] + tx[1]) + (tx[2] + tx[3]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.a_full[j]);
    }
    // row sums: the K-half-1 warps hand theirs to the K-half-0 warps, which
    // run the epilogue, through the last A stage (every statistics read of
    // it is done once all 8 warps passed the first barrier; the Y staging
    // below uses stages 0-2)
    float* xs = reinterpret_cast<float*>(s.a[STAGES - 1]);
    named_bar_sync(2, NSW * 32);
    if (kh == 1) {
      xs[r] = ss;
      if (LN) xs[BM + r] = sx;
    }
    named_bar_sync(2, NSW * 32);
    if (kh == 1) goto stats_done;
    ss += xs[r];
    if (LN) sx += xs[BM + r];
    float inv, mean = 0.f;
    if (p.partial) {  // slice partial state: statistics of the slice only
      if (nt == 0) {
        p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = LN ? sx : ss;
        if (LN) p.ws_d2[blockIdx.y * p.ws_rows + m0 + r] = ss;
      }
      inv = 0.f;
    } else if (LN) {
      mean = sx * p.inv_k;
      inv = rsqrtf(fmaf(ss, p.inv_k, -mean * mean) + p.eps);  // 1/sigma
      if (nt == 0) {
        p.d1[m0 + r] = sx;
        p.d2[m0 + r] = ss;
      }
    } else {
      inv = rsqrtf(fmaf(ss, p.inv_k, p.eps));
      if (nt == 0) p.d1[m0 + r] = ss;
    }
    named_bar_sync(1, 128);
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    const uint32_t stage = smem_u32(s.a[0]);  // drained: 48 KB of A stages for the Y tile
    if (p.partial) {
      // raw accumulator (H' = 1) of the slice, 2 x 16 KB staged per round
      store_acc_f32_n<2>(tmem + lane_off, r, s.a[0], &ty, n0, static_cast<int>(blockIdx.y * p.ws_rows) + m0, wn);
    } else {
      // Y tile: wn / 64 chunks of [128 rows x 64 bf16] (<= 3 x 16 KB staged)
      for (int c = 0; c < wn / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + c * 32, v);
        tmem_ld_wait();
        const uint32_t chunk = stage + (c >> 1) * (BM * 128);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          sts128(chunk + sw128(r, (c & 1) * 4 + q), w);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
        for (int c = 0; c < wn / 64; ++c)
          tma_store_2d_hint(&ty, s.a[0] + c * (BM * 128), n0 + 64 * c, m0, kEvictFirst);
        bulk_commit();
        bulk_wait_read0();
      }
      if (LN && p.write_d4) {
        // d4 = (d1/K) / sigma * colsum[f]: a rank-1 tile, staged the same way
        named_bar_sync(1, 128);  // staging area free again
        const float mi = mean * inv;
        for (int c = 0; c < wn / 32; ++c) {
          const uint32_t chunk = stage + (c >> 1) * (BM * 128);
          const float* cs = p.colsum + n0 + c * 32;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs + 8 * q));
            const float4 c1 = __ldg(reinterpret_cast<const float4*>(cs + 8 * q + 4));
            uint4 w;
            w.x = pack_bf16x2(mi * c0.x, mi * c0.y);
            w.y = pack_bf16x2(mi * c0.z, mi * c0.w);
            w.z = pack_bf16x2(mi * c1.x, mi * c1.y);
            w.w = pack_bf16x2(mi * c1.z, mi * c1.w);
            sts128(chunk + sw128(r, (c & 1) * 4 + q), w);
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 0) {
          for (int c = 0; c < wn / 64; ++c)
            tma_store_2d_hint(&ty4, s.a[0] + c * (BM * 128), n0 + 64 * c, m0, kEvictFirst);
          bulk_commit();
        }
      }
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
stats_done:
  tc_fence_before();
  cluster_sync();
  if (warp == MMA_WARP) tmem_dealloc_2sm<256>(tmem);
}

}  // namespace rms3
