// FAST fused predictor kernel (included by spx_predictor.cu, namespace spx).
//
// Warp-specialised, persistent, one CTA per SM:
//   * 1 PRODUCER warp: loads the speculative ids of the CTA's rows eight units
//     at a time and streams each row's GROUP LM-head rows (8 KiB each at 7B)
//     into a ring of NS shared-memory stages with 1-D TMA bulk copies
//     (cp.async.bulk, mbarrier complete_tx).  Stage reuse is gated by an
//     "empty" mbarrier the consumer releases.
//   * NTEAM CONSUMER teams of 4 warps: team t owns CTA rows t, t+NTEAM, ...
//     Warp w of a team owns canonical partial group g = w, so each per-row
//     reduction is split four ways.  The hidden row (f32) is loaded straight
//     into registers (one row ahead), so shared memory holds only LM-head
//     rows, the per-CTA constants (W1, b1, w2, final-norm gain) and scratch.
// Fast-path algebra (canonical, shared with K4/K6):
//   mean = CSUM(x)/d ; xc = x - mean ; var = CSUM(xc*xc)/d ; r = 1/sqrt(var+eps)
//   logit_v = r * CDOT(xc*g, W_v) + bw_v      (bw_v = CDOT(b, W_v), per model)
// i.e. the LayerNorm is folded into the head dot (one pass over the row for
// the variance and the K dots), with packed FP32 (FADD2/FMUL2/FFMA2).

constexpr int NTEAM = 4;
constexpr int TEAM = 4;
constexpr int NS_MAX = 8;
constexpr int RED_FLOATS = 32;                 // (GROUP + 2) * 4 used
constexpr int FAST_THREADS = 32 * (TEAM * NTEAM + 1);

struct SmemPlan {
  int ns;          // LM-head stages
  int w1_smem;     // W1 staged in shared memory?
  size_t bytes;
  size_t off_g, off_w2, off_b1, off_w1, off_team, team_bytes, off_stage, stage_bytes, off_bar,
      off_sflag;
};

template <typename TW>
inline SmemPlan plan_smem(int d, int K, int H, int max_bytes, int force_w1 = -1,
                          int max_stages = NS_MAX) {
  SmemPlan best{};
  const size_t stage = ((size_t)GROUP * d * sizeof(TW) + 127) / 128 * 128;
  const size_t team = ((size_t)(RED_FLOATS + 4 + 3 * MAXK + (H > 0 ? H : 4) + 64) * 4 + 127) /
                      128 * 128;
  const size_t w1b = ((size_t)3 * K * H * 4 + 127) / 128 * 128;
  const size_t fixed0 = (((size_t)d + 2 * H) * 4 + 127) / 128 * 128 + NTEAM * team + 256;
  for (int w1 = 0; w1 <= (H > 0 ? 1 : 0); ++w1) {
    if (force_w1 >= 0 && w1 != force_w1) continue;
    const size_t fixed = fixed0 + (w1 ? w1b : 0);
    int ns = 0;
    for (int t = max_stages; t >= 2; --t)
      if (fixed + (size_t)t * stage + (2 * NS_MAX + 1) * 8 + NS_MAX * 4 <= (size_t)max_bytes) {
        ns = t;
        break;
      }
    // prefer W1 in shared memory as long as it keeps >= 4 stages
    const bool better = ns > 0 && (best.ns == 0 || (w1 && ns >= 4) || (!best.w1_smem && ns > best.ns));
    if (better) {
      SmemPlan s{};
      s.ns = ns; s.w1_smem = w1;
      size_t o = 0;
      s.off_g = o; o += (size_t)d * 4;
      s.off_w2 = o; o += (size_t)H * 4;
      s.off_b1 = o; o += (size_t)H * 4;
      o = (o + 127) / 128 * 128;
      s.off_w1 = o; if (w1) o += w1b;
      s.off_team = o; s.team_bytes = team; o += NTEAM * team;
      s.off_stage = o; s.stage_bytes = stage; o += (size_t)ns * stage;
      s.off_bar = o; o += (size_t)(2 * NS_MAX + 1) * 8;
      s.off_sflag = o; o += NS_MAX * 4;
      s.bytes = o;
      best = s;
    }
  }
  return best;
}

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename TW, int CPL, bool FULL>
__global__ void __launch_bounds__(FAST_THREADS, 1)
predictor_fast_kernel(PredParams p, SmemPlan sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = p.d, K = p.K, H = p.H, nchunk = d / CHUNK, ns = sp.ns;
  float *gs = reinterpret_cast<float *>(smem + sp.off_g);
  float *w2s = reinterpret_cast<float *>(smem + sp.off_w2);
  float *b1s = reinterpret_cast<float *>(smem + sp.off_b1);
  float *w1s = reinterpret_cast<float *>(smem + sp.off_w1);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + sp.off_bar);
  uint64_t *empty = full + NS_MAX;
  uint64_t *setup_bar = full + 2 * NS_MAX;
  int *sflag = reinterpret_cast<int *>(smem + sp.off_sflag);
  const TW *head = reinterpret_cast<const TW *>(p.head);
  const bool mlp = p.policy == SPX_POLICY_MLP;
  const bool bulk_consts = (H % 4) == 0;
  const uint32_t wrow_bytes = (uint32_t)((size_t)d * sizeof(TW));
  const int ngroups = (K + GROUP - 1) / GROUP;
  const int rows_cta = p.B > (int)blockIdx.x ? (p.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int units = rows_cta * ngroups;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    mbar_init(setup_bar, 1);
  }
  fence_mbar_init();
  __syncthreads();

  if (warp == TEAM * NTEAM) {
    // =========================== PRODUCER ===========================
    if (lane == 0) {                         // per-CTA constants by TMA
      uint32_t bytes = (uint32_t)d * 4u;
      if (mlp && bulk_consts) bytes += 2u * H * 4u + (sp.w1_smem ? 3u * K * H * 4u : 0u);
      mbar_arrive_expect_tx(setup_bar, bytes);
      bulk_g2s(gs, p.norm_g, (uint32_t)d * 4u, setup_bar);
      if (mlp && bulk_consts) {
        bulk_g2s(w2s, p.w2, (uint32_t)H * 4u, setup_bar);
        bulk_g2s(b1s, p.b1, (uint32_t)H * 4u, setup_bar);
        if (sp.w1_smem) bulk_g2s(w1s, p.w1, 3u * K * H * 4u, setup_bar);
      }
    }
    for (int ub = 0; ub < units; ub += 8) {
      // lane l prefetches id q = l % 4 of unit ub + l / 4
      const int my_unit = ub + (lane >> 2), q = lane & 3;
      int my_id = 0, my_bad = 0, my_skip = 1;
      if (my_unit < units) {
        const int k = my_unit / ngroups, g = my_unit % ngroups, c = g * GROUP + q;
        const int row = (int)blockIdx.x + k * (int)gridDim.x;
        if (q == 0) my_skip = row_skipped(p, row) ? 1 : 0;
        if (c < K) {
          my_id = p.ids[(size_t)row * K + c];
          if (my_id < 0 || my_id >= p.V) { my_bad = 1; my_id = 0; }
        }
      }
      for (int j = 0; j < 8 && ub + j < units; ++j) {
        const int unit = ub + j, s = unit % ns;
        const int skip = __shfl_sync(0xffffffffu, my_skip, 4 * j);
        int ids4[GROUP], bad = 0;
#pragma unroll
        for (int qq = 0; qq < GROUP; ++qq) {
          ids4[qq] = __shfl_sync(0xffffffffu, my_id, 4 * j + qq);
          bad |= __shfl_sync(0xffffffffu, my_bad, 4 * j + qq);
        }
        if (lane == 0) {
          mbar_wait(empty + s, ((unit / ns) & 1) ^ 1);
          const int g = unit % ngroups;
          const int ng = (K - g * GROUP) < GROUP ? (K - g * GROUP) : GROUP;
          sflag[s] = skip ? 1 : (bad ? 2 : 0);
          if (skip) {
            mbar_arrive(full + s);
          } else {
            const int k = unit / ngroups;
            const int row = (int)blockIdx.x + k * (int)gridDim.x;
            if (p.trace && g == 0) p.trace[(size_t)row * 8 + 5] = gtimer();
            TW *dst = reinterpret_cast<TW *>(smem + sp.off_stage + (size_t)s * sp.stage_bytes);
            fence_proxy_async();
            mbar_arrive_expect_tx(full + s, (uint32_t)ng * wrow_bytes);
            for (int qq = 0; qq < ng; ++qq)
              bulk_g2s(dst + (size_t)qq * d, head + (size_t)ids4[qq] * d, wrow_bytes, full + s);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // =========================== CONSUMERS ===========================
  const int team = warp / TEAM, w = warp % TEAM;
  uint8_t *tbase = smem + sp.off_team + (size_t)team * sp.team_bytes;
  float *red = reinterpret_cast<float *>(tbase);            // [GROUP+2][4]
  int *tflag = reinterpret_cast<int *>(red + RED_FLOATS);   // [4]
  float *feats = red + RED_FLOATS + 4;
  float *hs = feats + 3 * MAXK;
  float *as = hs + (H > 0 ? H : 4);
  const bool leader = (w == 0 && lane == 0);

  // one row ahead: hidden chunks (registers), prev + bw of this lane's ids
  float4 xr[CPL];
  float pv0 = 0.f, pv1 = 0.f, bw0 = 0.f, bw1 = 0.f;
  auto prefetch = [&](int k) {
    if (k >= rows_cta) return;
    const int row = (int)blockIdx.x + k * (int)gridDim.x;
    const float *x = p.hidden + (size_t)row * p.hidden_stride;
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int c = 32 * w + lane + NPART * s;
      if (FULL || c < nchunk) xr[s] = __ldg(reinterpret_cast<const float4 *>(x + CHUNK * c));
      else xr[s] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (w == 0) {
      if (lane < K) {
        pv0 = p.prev[(size_t)row * K + lane];
        int id = p.ids[(size_t)row * K + lane];
        id = (id < 0 || id >= p.V) ? 0 : id;
        bw0 = p.head_bw ? __ldg(p.head_bw + id) : 0.f;
      }
      if (lane + 32 < K) {
        pv1 = p.prev[(size_t)row * K + lane + 32];
        int id = p.ids[(size_t)row * K + lane + 32];
        id = (id < 0 || id >= p.V) ? 0 : id;
        bw1 = p.head_bw ? __ldg(p.head_bw + id) : 0.f;
      }
    }
  };

  int k = team;
  prefetch(k);
  mbar_wait(setup_bar, 0);
  while (k < rows_cta) {
    const int row = (int)blockIdx.x + k * (int)gridDim.x;
    const int unit0 = k * ngroups;
    mbar_wait(full + unit0 % ns, (unit0 / ns) & 1);
    const int sf = sflag[unit0 % ns];
    if (sf == 1) {                               // skipped row (exited / not scheduled)
      if (leader && p.fired) p.fired[row] = 0;
      team_sync(team);
      if (leader)
        for (int g = 0; g < ngroups; ++g) {
          const int u = unit0 + g;
          if (g > 0) mbar_wait(full + u % ns, (u / ns) & 1);
          mbar_arrive(empty + u % ns);
        }
      k += NTEAM;
      prefetch(k);
      continue;
    }
    if (p.trace && leader) p.trace[(size_t)row * 8 + 1] = gtimer();
    // ---- pass 1: mean (this warp = canonical group w), from registers
    float part = 0.f;
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int c = 32 * w + lane + NPART * s;
      if (FULL || c < nchunk)
        part = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(part, xr[s].x), xr[s].y), xr[s].z), xr[s].w);
    }
    part = warp_butterfly_sum(part);
    if (lane == 0) red[GROUP * 4 + w] = part;
    team_sync(team);
    const float total = canon_combine(red[GROUP * 4 + 0], red[GROUP * 4 + 1], red[GROUP * 4 + 2],
                                      red[GROUP * 4 + 3]);
    const float mean = __fdiv_rn(total, (float)d);
    bool hbad = false;
    if (!is_finite(total)) {              // rare: exact element scan (model.py:310-311)
      bool fin = true;
#pragma unroll
      for (int s = 0; s < CPL; ++s)
        fin &= is_finite(xr[s].x) & is_finite(xr[s].y) & is_finite(xr[s].z) & is_finite(xr[s].w);
      const bool wbad = __any_sync(0xffffffffu, !fin);
      if (lane == 0) tflag[w] = wbad ? 1 : 0;
      team_sync(team);
      hbad = (tflag[0] | tflag[1] | tflag[2] | tflag[3]) != 0;
      team_sync(team);
    }
    if (p.trace && leader) p.trace[(size_t)row * 8 + 2] = gtimer();
    float r = 0.f;
    int ibad = 0;
    const float2 nmean = make_float2(-mean, -mean);
    for (int g = 0; g < ngroups; ++g) {
      const int unit = unit0 + g, s = unit % ns;
      if (g > 0) mbar_wait(full + s, (unit / ns) & 1);
      ibad |= (sflag[s] == 2);
      const TW *sw = reinterpret_cast<const TW *>(smem + sp.off_stage + (size_t)s * sp.stage_bytes);
      const int c0 = g * GROUP, ng = (K - c0) < GROUP ? (K - c0) : GROUP;
      float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
      float sq = 0.f;
#pragma unroll
      for (int s2 = 0; s2 < CPL; ++s2) {
        const int c = 32 * w + lane + NPART * s2;
        if (FULL || c < nchunk) {
          const float4 xv = xr[s2];
          const float4 gv = *reinterpret_cast<const float4 *>(gs + CHUNK * c);
          const float2 xc01 = fadd2(make_float2(xv.x, xv.y), nmean);
          const float2 xc23 = fadd2(make_float2(xv.z, xv.w), nmean);
          if (g == 0)
            sq = __fmaf_rn(xc23.y, xc23.y, __fmaf_rn(xc23.x, xc23.x,
                           __fmaf_rn(xc01.y, xc01.y, __fmaf_rn(xc01.x, xc01.x, sq))));
          const float2 xg01 = fmul2(xc01, make_float2(gv.x, gv.y));
          const float2 xg23 = fmul2(xc23, make_float2(gv.z, gv.w));
          float wv[GROUP][4];
#pragma unroll
          for (int q = 0; q < GROUP; ++q) {
            Chunk<TW> ch;
            ch.lds(sw + (size_t)q * d + CHUNK * c);
            ch.to_f32(wv[q]);
          }
          const float xe[4] = {xg01.x, xg01.y, xg23.x, xg23.y};
#pragma unroll
          for (int e = 0; e < CHUNK; ++e) {
            const float2 xx = make_float2(xe[e], xe[e]);
            acc01 = ffma2(xx, make_float2(wv[0][e], wv[1][e]), acc01);
            acc23 = ffma2(xx, make_float2(wv[2][e], wv[3][e]), acc23);
          }
        }
      }
      float acc[GROUP] = {acc01.x, acc01.y, acc23.x, acc23.y};
#pragma unroll
      for (int q = 0; q < GROUP; ++q) acc[q] = warp_butterfly_sum(acc[q]);
      if (g == 0) sq = warp_butterfly_sum(sq);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < GROUP; ++q) red[q * 4 + w] = acc[q];
        if (g == 0) red[(GROUP + 1) * 4 + w] = sq;
      }
      team_sync(team);                         // all warps done with stage s and wrote red
      if (leader) mbar_arrive(empty + s);      // release the stage to the producer
      if (g == 0) {
        const float var = __fdiv_rn(canon_combine(red[(GROUP + 1) * 4 + 0], red[(GROUP + 1) * 4 + 1],
                                                  red[(GROUP + 1) * 4 + 2], red[(GROUP + 1) * 4 + 3]),
                                    (float)d);
        r = __frcp_rn(__fsqrt_rn(__fadd_rn(var, 1e-5f)));
      }
      if (w == 0) {
        // lane q (< ng) combines id c0+q; its bw sits in lane (c0+q) % 32
        const float bwa = __shfl_sync(0xffffffffu, bw0, (c0 + lane) & 31);
        const float bwb = __shfl_sync(0xffffffffu, bw1, (c0 + lane) & 31);
        if (lane < ng) {
          const float dot = canon_combine(red[lane * 4 + 0], red[lane * 4 + 1], red[lane * 4 + 2],
                                          red[lane * 4 + 3]);
          feats[c0 + lane] = __fadd_rn(__fmul_rn(r, dot), (c0 + lane) < 32 ? bwa : bwb);
        }
      }
      if (ngroups > 1) team_sync(team);        // red reused by the next group
    }
    if (p.trace && leader) p.trace[(size_t)row * 8 + 3] = gtimer();
    // this row's prev for the softmax; then prefetch the next row (x regs are dead)
    const float cpv0 = pv0, cpv1 = pv1;
    k += NTEAM;
    prefetch(k);
    team_sync(team);                           // feats complete
    // ---- softmax / features (warp 0)
    if (w == 0) {
      int ok = 0;
      const int Kk = K;
      if (ibad || hbad) {
        if (lane == 0) atomicOr(p.err, (ibad ? ERR_ID_RANGE : 0) | (hbad ? ERR_HIDDEN_NONFINITE : 0));
      } else {
        const bool v0 = lane < Kk, v1 = lane + 32 < Kk;
        const float x0 = v0 ? feats[lane] : 0.f, x1 = v1 ? feats[lane + 32] : 0.f;
        bool bad = (v0 && !is_finite(x0)) || (v1 && !is_finite(x1));
        bad = __any_sync(0xffffffffu, bad);
        float m = v0 ? x0 : -INFINITY;
        if (v1) m = fmaxf(m, x1);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float e0 = v0 ? np_expf(__fsub_rn(x0, m)) : 0.f;
        const float e1 = v1 ? np_expf(__fsub_rn(x1, m)) : 0.f;
        float esum = 0.f, psum = 0.f;                 // strict left-to-right (seq_sum)
        for (int c = 0; c < Kk; ++c) {
          esum = __fadd_rn(esum, __shfl_sync(0xffffffffu, c < 32 ? e0 : e1, c & 31));
          psum = __fadd_rn(psum, __shfl_sync(0xffffffffu, c < 32 ? cpv0 : cpv1, c & 31));
        }
        int e = 0;
        if (bad) e |= ERR_LOGIT_NONFINITE;
        if (fabs((double)psum - 1.0) > 1e-5) e |= ERR_PREV_SUM;
        if (e) {
          if (lane == 0) atomicOr(p.err, e);
        } else {
          ok = 1;
          if (v0) {
            const float pr = __fdiv_rn(e0, esum);
            feats[Kk + lane] = pr;
            feats[2 * Kk + lane] = __fsub_rn(pr, cpv0);
            p.prev[(size_t)row * Kk + lane] = pr;                       // engine.py:196
          }
          if (v1) {
            const float pr = __fdiv_rn(e1, esum);
            feats[Kk + lane + 32] = pr;
            feats[2 * Kk + lane + 32] = __fsub_rn(pr, cpv1);
            p.prev[(size_t)row * Kk + lane + 32] = pr;
          }
        }
        if (p.logits_out) {
          if (v0) p.logits_out[(size_t)row * Kk + lane] = x0;
          if (v1) p.logits_out[(size_t)row * Kk + lane + 32] = x1;
        }
      }
      __syncwarp();
      if (ok) {
        if (p.feat_out)
          for (int i = lane; i < 3 * Kk; i += 32) p.feat_out[(size_t)row * 3 * Kk + i] = feats[i];
        if (lane == 0 && p.evals) p.evals[row] += 1;
      } else if (lane == 0 && p.fired) {
        p.fired[row] = 0;
      }
      if (lane == 0) tflag[0] = ok;
    }
    team_sync(team);
    if (tflag[0]) {
      if (mlp) {
        if (sp.w1_smem) mlp_z1<1, false>(feats, w1s, b1s, 3 * K, H, hs, lane, w);
        else mlp_z1<1, true>(feats, p.w1, b1s, 3 * K, H, hs, lane, w);
        team_sync(team);
        if (w < 2) as[32 * w + lane] = z2_partial(hs, w2s, H, 32 * w + lane);
        team_sync(team);
        if (w == 0) {
          const float z2 = z2_tree(as[lane], as[lane + 32], hs, w2s, H, p.b2, lane);
          if (lane == 0) {
            if (p.z_out) p.z_out[row] = z2;
            if (p.prob_out) p.prob_out[row] = sigmoid64(z2);
            if (p.fired) p.fired[row] = (z2 >= p.z_cut) ? 1 : 0;
          }
        }
      } else if (leader) {
        if (p.prob_out) p.prob_out[row] = p.const_prob;
        if (p.z_out) p.z_out[row] = 0.0f;
        if (p.fired) p.fired[row] = (p.const_prob > p.threshold) ? 1 : 0;
      }
    }
    if (p.trace && leader) p.trace[(size_t)row * 8 + 4] = gtimer();
    team_sync(team);                           // feats/hs/as/tflag reused by the next row
  }
}

template <typename TW>
struct FastLaunch {
  const PredParams &p; const SmemPlan &sp; int grid; cudaStream_t stream; int smem_optin;
  template <int CPL> void operator()() const {
    if (p.d == CHUNK * NPART * CPL) launch<CPL, true>();
    else launch<CPL, false>();
  }
  template <int CPL, bool FULL> void launch() const {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(predictor_fast_kernel<TW, CPL, FULL>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
      configured = true;
    }
    predictor_fast_kernel<TW, CPL, FULL><<<grid, FAST_THREADS, sp.bytes, stream>>>(p, sp);
  }
};
