// STREAM fused predictor kernel (included by spx_predictor.cu, namespace spx):
// the FAST-mode K1+K2+K3 launch for K <= 8 at LLM widths.  Same canonical
// arithmetic as predictor_fast_kernel (CDOT order, folded LayerNorm), so its
// logits, features and decisions are bit-identical to it -- only the schedule
// differs.
//
// Persistent CTA per SM, warp-specialised around a ring of S "eval slots":
//   * PRODUCER warp: streams whole evaluations in row order -- the f32 hidden
//     row and the K bf16 LM-head rows of one request land in one slot with
//     1 + K cp.async.bulk copies on one mbarrier (expect_tx = d*4 + K*d*2).
//     Ids are read up front for a window of 32 rows (one per lane), so the
//     copy issue never waits on a dependent load.  With pdl == 2 ("ids
//     ready") the LM-head copies of the first S rows are issued before
//     griddepcontrol.wait.
//   * 4 COMPUTE warps, all on the same slot: warp g owns canonical partial
//     group g of every LM-head row of the slot and of the mean / variance
//     passes.  Two named barriers per row; the slot is released right after
//     the second.
//   * 4 TAIL warps: softmax over the K ids + features, MLP (W1/b1/w2 in
//     shared memory), f32 sigmoid for the reported prob, exact decision
//     z2 >= z_cut.  Each tail warp prefetches its next row's prev / bias-fold
//     / id values from global memory before waiting for the logits.
// With S = 3 slots of 48 KB (7B: d = 4096, K = 4) three evaluations are in
// flight per SM while one is reduced: HBM stays saturated and the per-row
// critical path is one slot's reduction (~0.5 us) plus the tail.

constexpr int SW_COMPUTE = 4;                           // compute warps (one per group)
constexpr int SW_TAIL = 4;
constexpr int SW_THREADS = 32 * (SW_COMPUTE + 1 + SW_TAIL);
constexpr int SKMAX = 8;                                // max K of this kernel
constexpr int SQS = 8;                                  // tail queue slots
constexpr int SWIN = 32;                                // ids window (rows)

struct SQSlot {
  int row, flags, pad0, pad1;
  float logit[SKMAX];                                   // r * CDOT (bias fold added by the tail)
};

struct StreamPlan {
  int S;                                                // eval slots
  int w1_smem;
  size_t slot_bytes, off_slots, off_w1, off_w2, off_b1, off_g, off_red, off_q, off_tail,
      tail_bytes, off_hdr, off_ids, off_bar, bytes;
};

// ldgx: the hidden rows go HBM -> registers (ld.global) instead of through
// the slot, the slots hold only the K LM-head rows, and the plan is sized for
// two CTAs per SM (so the next launch's CTAs can start on half an SM while
// this launch finishes).
template <typename TW>
inline StreamPlan plan_stream(int d, int K, int H, int max_bytes, bool ldgx = false) {
  StreamPlan s{};
  const size_t slot = ((ldgx ? 0 : (size_t)d * 4) + (size_t)K * d * sizeof(TW) + 127) / 128 * 128;
  const size_t w1b = ((size_t)3 * K * H * 4 + 127) / 128 * 128;
  const size_t fixed = ((size_t)2 * H * 4 + 127) / 128 * 128 +
                       /*red*/ 2 * (SKMAX + 2) * 4 * 4 * 2 + /*queue*/ sizeof(SQSlot) * SQS +
                       /*tail*/ SW_TAIL * (((size_t)(3 * SKMAX + H + 32) * 4 + 127) / 128 * 128) +
                       /*hdr*/ 8 * 16 + /*ids*/ SWIN * SKMAX * 4 + /*bars*/ (2 * 8 + 2 * SQS + 2) * 8 +
                       1024;
  // deepest ring with W1 resident first; W1 through L1 only as the last resort
  for (int S = 4; S >= 1; --S) {
    bool w1 = H > 0 && fixed + S * slot + w1b <= (size_t)max_bytes;
    if (!w1 && S > 1 && H > 0) continue;
    if (fixed + S * slot + (w1 ? w1b : 0) > (size_t)max_bytes) continue;
    size_t o = 0;
    s.S = S;
    s.w1_smem = w1;
    s.slot_bytes = slot;
    s.off_slots = o; o += S * slot;
    s.off_w1 = o; if (w1) o += w1b;
    s.off_w2 = o; o += (size_t)H * 4;
    s.off_b1 = o; o += (size_t)H * 4;
    o = (o + 127) / 128 * 128;
    s.off_g = o;
    s.off_red = o; o += 2 * (SKMAX + 2) * 4 * 4 * 2;
    s.off_q = o; o += sizeof(SQSlot) * SQS;
    o = (o + 127) / 128 * 128;
    s.off_tail = o; s.tail_bytes = ((size_t)(3 * SKMAX + H + 32) * 4 + 127) / 128 * 128;
    o += SW_TAIL * s.tail_bytes;
    s.off_hdr = o; o += 8 * 16;
    s.off_ids = o; o += SWIN * SKMAX * 4;
    o = (o + 7) / 8 * 8;
    s.off_bar = o; o += (2 * 8 + 2 * SQS + 2) * 8;
    s.bytes = o;
    return s;
  }
  return s;                                             // bytes == 0: does not fit
}

__device__ __forceinline__ void cbar_sync() {          // the 4 compute warps
  asm volatile("bar.sync 1, %0;" ::"r"(32 * SW_COMPUTE) : "memory");
}

template <typename TW, int CPL, int KC, int HC, bool W1S, bool LDGX>
__global__ void __launch_bounds__(SW_THREADS, 2)
predictor_stream_kernel(PredParams p, StreamPlan sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = p.d, K = KC ? KC : p.K, H = HC ? HC : p.H;
  const int S = sp.S;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + sp.off_bar);     // [S]
  uint64_t *empty = full + 8;                                           // [S]
  uint64_t *qfull = empty + 8;                                          // [SQS]
  uint64_t *qempty = qfull + SQS;                                       // [SQS]
  uint64_t *setup_bar = qempty + SQS;
  int *hdr = reinterpret_cast<int *>(smem + sp.off_hdr);                // [S][4]: row, flags
  float *w2s = reinterpret_cast<float *>(smem + sp.off_w2);
  float *b1s = reinterpret_cast<float *>(smem + sp.off_b1);
  float *w1s = reinterpret_cast<float *>(smem + sp.off_w1);
  SQSlot *queue = reinterpret_cast<SQSlot *>(smem + sp.off_q);
  const bool mlp = p.policy == SPX_POLICY_MLP;
  const uint32_t hid_bytes = LDGX ? 0u : (uint32_t)d * 4u;      // hidden bytes in a slot
  const uint32_t wrow_bytes = (uint32_t)((size_t)d * sizeof(TW));
  const int rows_cta =
      p.B > (int)blockIdx.x ? (p.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto row_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };

  int &s_defer = reinterpret_cast<int *>(smem + sp.off_hdr)[31];   // rows deferred (recheck)
  if (threadIdx.x == 0) {
    s_defer = 0;
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int s = 0; s < SQS; ++s) { mbar_init(qfull + s, 1); mbar_init(qempty + s, 1); }
    mbar_init(setup_bar, 1);
  }
  fence_mbar_init();
  __syncthreads();
  if (threadIdx.x == 0) {                  // per-CTA constants by TMA
    uint32_t bytes = 0;
    if (mlp) bytes += 2u * H * 4u + (W1S ? 3u * K * H * 4u : 0u);
    mbar_arrive_expect_tx(setup_bar, bytes);
    if (mlp) {
      bulk_g2s(w2s, p.w2, (uint32_t)H * 4u, setup_bar);
      bulk_g2s(b1s, p.b1, (uint32_t)H * 4u, setup_bar);
      if (W1S) bulk_g2s(w1s, p.w1, 3u * K * H * 4u, setup_bar);
    }
  }
  const bool early = p.pdl == 2 && !p.row_done && !p.row_layer_mask;
  auto pdl_wait_trigger = [&]() {
    if (p.pdl) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
  };

  if (!early) pdl_wait_trigger();            // every role reads dependent data

  // ============================== PRODUCER ==============================
  if (warp == SW_COMPUTE) {
    int *ids_s = reinterpret_cast<int *>(smem + sp.off_ids);            // [SWIN][SKMAX]
    // rows are skipped (row_done / row_layer_mask) identically by every role
    int j = 0;                              // slot sequence over non-skipped rows
    bool waited = !early;
    for (int w0 = 0; w0 < rows_cta; w0 += SWIN) {
      // ids of rows w0 .. w0+31: lane i loads row w0+i (one dependent load per window)
      int myid[SKMAX];
      int bad = 0;
      const int ri = w0 + lane;
      const bool have = ri < rows_cta;
      const int row_i = row_of(have ? ri : 0);
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) {
        myid[c] = 0;
        if (have && c < K) {
          const int v = p.ids[(size_t)row_i * K + c];
          if (v < 0 || v >= p.V) bad = 1; else myid[c] = v;
        }
      }
      __syncwarp();
      if (have)
#pragma unroll
        for (int c = 0; c < SKMAX; ++c) ids_s[lane * SKMAX + c] = myid[c];
      unsigned badmask = __ballot_sync(0xffffffffu, bad);
      __syncwarp();
      if (lane == 0) {
        const int wn = rows_cta - w0 < SWIN ? rows_cta - w0 : SWIN;
        for (int i = 0; i < wn; ++i) {
          const int row = row_of(w0 + i);
          if (waited && row_skipped(p, row)) continue;
          const int s = j % S;
          if (j >= S) mbar_wait(empty + s, ((j / S) - 1) & 1);
          uint8_t *dst = smem + sp.off_slots + (size_t)s * sp.slot_bytes;
          hdr[s * 4 + 0] = row;
          hdr[s * 4 + 1] = ((badmask >> i) & 1) ? 2 : 0;
          if (p.trace) p.trace[(size_t)row * 16 + 5] = gtimer();
          mbar_arrive_expect_tx(full + s, hid_bytes + (uint32_t)K * wrow_bytes);
          const TW *head = reinterpret_cast<const TW *>(p.head);
          for (int c = 0; c < K; ++c)
            bulk_g2s(dst + hid_bytes + (size_t)c * wrow_bytes,
                     head + (size_t)ids_s[i * SKMAX + c] * d, wrow_bytes, full + s);
          if (waited && !LDGX)
            bulk_g2s(dst, p.hidden + (size_t)row * p.hidden_stride, hid_bytes, full + s);
          ++j;
          if (!waited && (j == S || (w0 + i + 1 == rows_cta))) {
            // the hidden rows of the early slots: after the wait
            pdl_wait_trigger();
            waited = true;
            for (int jj = 0; jj < (LDGX ? 0 : j); ++jj)
              bulk_g2s(smem + sp.off_slots + (size_t)jj * sp.slot_bytes,
                       p.hidden + (size_t)hdr[jj * 4 + 0] * p.hidden_stride, hid_bytes, full + jj);
          }
        }
      }
      __syncwarp();
      waited = __shfl_sync(0xffffffffu, waited ? 1 : 0, 0) != 0;
      j = __shfl_sync(0xffffffffu, j, 0);
    }
    if (!waited) pdl_wait_trigger();
  } else {

  if (early) pdl_wait_trigger();             // compute + tail warps: after the prefetch
  mbar_wait(setup_bar, 0);

  // ============================== TAIL WARPS ==============================
  // Tail warp tw takes rows tw, tw+4, ... of the slot sequence: softmax over
  // the K ids + features, the MLP, the exact decision.  Each prefetches its
  // next row's carried probabilities and bias folds before waiting.
  if (warp > SW_COMPUTE) {
    const int tw = warp - SW_COMPUTE - 1;
    float *feats = reinterpret_cast<float *>(smem + sp.off_tail + (size_t)tw * sp.tail_bytes);
    float *hs = feats + 3 * SKMAX;
    const float *w1 = W1S ? w1s : p.w1;
    int j = 0;                                // same sequence as the producer
    for (int i = 0; i < rows_cta; ++i) {
      const int row = row_of(i);
      if (row_skipped(p, row)) {
        if (lane == 0 && (i % SW_TAIL) == tw && p.fired) p.fired[row] = 0;
        continue;
      }
      const int myj = j++;
      if ((myj % SW_TAIL) != tw) continue;
      float pv[SKMAX], bw[SKMAX], wmx[SKMAX];
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) {
        pv[c] = 0.f; bw[c] = 0.f; wmx[c] = 0.f;
        if (c < K) {
          pv[c] = p.prev[(size_t)row * K + c];
          if (p.head_bw || p.recheck) {
            const int id = p.ids[(size_t)row * K + c];
            const bool ok = id >= 0 && id < p.V;
            if (p.head_bw && ok) bw[c] = __ldg(p.head_bw + id);
            if (p.recheck && ok) wmx[c] = __ldg(p.head_wmax + id);
          }
        }
      }
      const int qs = myj % SQS;
      mbar_wait(qfull + qs, (myj / SQS) & 1);
      if (p.trace && lane == 0) p.trace[(size_t)row * 16 + 0] = gtimer();
      const int flags = queue[qs].flags;
      const int lnf_bits = queue[qs].pad0;        // sqrt(1 + mean^2/var) of the row
      float x[SKMAX];
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) x[c] = c < K ? __fadd_rn(queue[qs].logit[c], bw[c]) : 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty + qs);
      if (flags & 6) {
        if (lane == 0) {
          atomicOr(p.err, ((flags & 2) ? ERR_ID_RANGE : 0) | ((flags & 4) ? ERR_HIDDEN_NONFINITE : 0));
          if (p.fired) p.fired[row] = 0;
        }
        continue;
      }
      // softmax over the K ids (model.py:149-152), features (predictor.py:42-52)
      bool bad = false;
      float m = x[0];
#pragma unroll
      for (int c = 0; c < SKMAX; ++c)
        if (c < K) { bad |= !is_finite(x[c]); m = fmaxf(m, x[c]); }
      float e[SKMAX], esum = 0.f, psum = 0.f;
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) e[c] = c < K ? np_expf(__fsub_rn(x[c], m)) : 0.f;
#pragma unroll
      for (int c = 0; c < SKMAX; ++c)
        if (c < K) esum = __fadd_rn(esum, e[c]);
      psum = np_sum_upto8(pv, K);                        // numpy pairwise (predictor.py:49)
      if (p.logits_out && lane < K) {
#pragma unroll
        for (int c = 0; c < SKMAX; ++c) if (lane == c) p.logits_out[(size_t)row * K + c] = x[c];
      }
      int ecode = 0;
      if (bad) ecode |= ERR_LOGIT_NONFINITE;
      if (fabsf(psum - 1.0f) > 1e-5f && fabs((double)psum - 1.0) > 1e-5) ecode |= ERR_PREV_SUM;
      if (ecode) {
        if (lane == 0) {
          atomicOr(p.err, ecode);
          if (p.fired) p.fired[row] = 0;
        }
        continue;
      }
      float pr[SKMAX];
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) pr[c] = c < K ? div_rn_unit(e[c], esum) : 0.f;
#pragma unroll
      for (int c = 0; c < SKMAX; ++c) {
        if (c < K && lane == c) {
          feats[c] = x[c];
          feats[K + c] = pr[c];
          feats[2 * K + c] = __fsub_rn(pr[c], pv[c]);
        }
      }
      __syncwarp();
      float z2 = 0.f;
      if (mlp) {
        mlp_z1<4, !W1S>(feats, w1, b1s, 3 * K, H, hs, lane, 0);
        __syncwarp();
        z2 = z2_tree(z2_partial(hs, w2s, H, lane), z2_partial(hs, w2s, H, lane + 32), hs, w2s, H,
                     p.b2, lane);
      }
      float perr = 0.f;
      if (p.recheck &&
          !certify_row(p, row, feats, hs + H, hs, w1, b1s, w2s, z2, __int_as_float(lnf_bits), K,
                       H, mlp, lane, perr, [&](int c) {
                         float v = 0.f;
#pragma unroll
                         for (int cc = 0; cc < SKMAX; ++cc) v = cc == c ? wmx[cc] : v;
                         return v;
                       })) {
        if (lane == 0) defer_row(p, row, &s_defer);  // STRICT re-evaluation decides
        __syncwarp();
        continue;
      }
#pragma unroll
      for (int c = 0; c < SKMAX; ++c)
        if (c < K && lane == c) p.prev[(size_t)row * K + c] = pr[c];   // engine.py:196
      if (lane == 0 && p.prev_err) p.prev_err[row] = perr;
      if (p.feat_out)
        for (int q = lane; q < 3 * K; q += 32) p.feat_out[(size_t)row * 3 * K + q] = feats[q];
      if (lane == 0 && p.evals) p.evals[row] += 1;
      if (mlp) {
        if (lane == 0) {
          if (p.z_out) p.z_out[row] = z2;
          if (p.prob_out) p.prob_out[row] = (double)sigmoid32(z2);
          write_fired(p, row, z2 >= p.z_cut);
        }
      } else if (lane == 0) {
        if (p.prob_out) p.prob_out[row] = p.const_prob;
        if (p.z_out) p.z_out[row] = 0.0f;
        write_fired(p, row, p.const_prob > p.threshold);
      }
      if (p.trace && lane == 0) p.trace[(size_t)row * 16 + 4] = gtimer();
      __syncwarp();
    }
  } else {

  // ============================== COMPUTE WARPS ==============================
  // warp g = canonical partial group g, for every LM-head row of the slot;
  // final_norm.g of this lane's chunks lives in registers for the whole kernel
  const int g = warp;
  constexpr int KP = (KC ? (KC + 1) / 2 : SKMAX / 2);       // LM-head row pairs
  float4 gr[CPL];
#pragma unroll
  for (int t = 0; t < CPL; ++t)
    gr[t] = __ldg(reinterpret_cast<const float4 *>(p.norm_g + CHUNK * (32 * g + lane + NPART * t)));
  float *red = reinterpret_cast<float *>(smem + sp.off_red);
  float *red_mean = red;                          // [4]
  float *red_sq = red + 4;                        // [4]
  float *red_dot = red + 8;                       // [SKMAX][4]
  int *red_flag = reinterpret_cast<int *>(red + 8 + SKMAX * 4);   // [4]
  int j = 0;
  for (int i = 0; i < rows_cta; ++i) {
    const int row = row_of(i);
    if (row_skipped(p, row)) continue;
    const int s = j % S;
    float4 xr[CPL];
    if (LDGX) {                                    // hidden row straight to registers
      const float *xg_ = p.hidden + (size_t)row * p.hidden_stride;
#pragma unroll
      for (int t = 0; t < CPL; ++t)
        xr[t] = __ldcs(reinterpret_cast<const float4 *>(xg_ + CHUNK * (32 * g + lane + NPART * t)));
    }
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)row * 16 + 6] = gtimer();
    mbar_wait(full + s, (j / S) & 1);
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)row * 16 + 1] = gtimer();
    const uint8_t *slot = smem + sp.off_slots + (size_t)s * sp.slot_bytes;
    const float *xh = reinterpret_cast<const float *>(slot);
    const TW *wk = reinterpret_cast<const TW *>(slot + hid_bytes);
    const int flags0 = hdr[s * 4 + 1];
    // ---- pass 1: mean (canonical group g)
    if (!LDGX) {
#pragma unroll
      for (int t = 0; t < CPL; ++t)
        xr[t] = *reinterpret_cast<const float4 *>(xh + CHUNK * (32 * g + lane + NPART * t));
    }
    float part = 0.f;
#pragma unroll
    for (int t = 0; t < CPL; ++t)
      part = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(part, xr[t].x), xr[t].y), xr[t].z), xr[t].w);
    part = warp_butterfly_sum(part);
    if (lane == 0) red_mean[g] = part;
    cbar_sync();
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)row * 16 + 2] = gtimer();
    const float total = canon_combine(red_mean[0], red_mean[1], red_mean[2], red_mean[3]);
    const float mean = __fdiv_rn(total, (float)d);
    int hflag = 0;
    if (!is_finite(total)) {                      // rare: exact element scan (model.py:310-311)
      bool fin = true;
#pragma unroll
      for (int t = 0; t < CPL; ++t)
        fin &= is_finite(xr[t].x) & is_finite(xr[t].y) & is_finite(xr[t].z) & is_finite(xr[t].w);
      const bool wbad = __any_sync(0xffffffffu, !fin);
      if (lane == 0) red_flag[g] = wbad ? 1 : 0;
      cbar_sync();
      for (int q = 0; q < 4; ++q) hflag |= red_flag[q];
      cbar_sync();
    }
    // ---- pass 2: variance and the K dots, LM-head rows in pairs (packed FMA)
    const float2 nmean = make_float2(-mean, -mean);
    float sq = 0.f;
    float2 acc[KP];
#pragma unroll
    for (int kp = 0; kp < KP; ++kp) acc[kp] = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = 32 * g + lane + NPART * t;
      const float2 xc01 = fadd2(make_float2(xr[t].x, xr[t].y), nmean);
      const float2 xc23 = fadd2(make_float2(xr[t].z, xr[t].w), nmean);
      sq = __fmaf_rn(xc23.y, xc23.y, __fmaf_rn(xc23.x, xc23.x,
                     __fmaf_rn(xc01.y, xc01.y, __fmaf_rn(xc01.x, xc01.x, sq))));
      const float2 xg01 = fmul2(xc01, make_float2(gr[t].x, gr[t].y));
      const float2 xg23 = fmul2(xc23, make_float2(gr[t].z, gr[t].w));
      const float xe[4] = {xg01.x, xg01.y, xg23.x, xg23.y};
#pragma unroll
      for (int kp = 0; kp < KP; ++kp) {
        if (2 * kp < K) {
          float wa[4], wb[4] = {0.f, 0.f, 0.f, 0.f};
          { Chunk<TW> ch; ch.lds(wk + (size_t)(2 * kp) * d + CHUNK * c); ch.to_f32(wa); }
          if (2 * kp + 1 < K) { Chunk<TW> ch; ch.lds(wk + (size_t)(2 * kp + 1) * d + CHUNK * c); ch.to_f32(wb); }
#pragma unroll
          for (int e = 0; e < CHUNK; ++e)
            acc[kp] = ffma2(make_float2(xe[e], xe[e]), make_float2(wa[e], wb[e]), acc[kp]);
        }
      }
    }
    sq = warp_butterfly_sum(sq);
    float dots[2 * KP];
#pragma unroll
    for (int kp = 0; kp < KP; ++kp) {
      dots[2 * kp] = 2 * kp < K ? warp_butterfly_sum(acc[kp].x) : 0.f;
      dots[2 * kp + 1] = 2 * kp + 1 < K ? warp_butterfly_sum(acc[kp].y) : 0.f;
    }
    if (lane == 0) {
      red_sq[g] = sq;
#pragma unroll
      for (int k = 0; k < 2 * KP; ++k) if (k < K) red_dot[k * 4 + g] = dots[k];
    }
    cbar_sync();                                   // slot fully read; partials visible
    if (threadIdx.x == 0) mbar_arrive(empty + s);  // producer may refill the slot
    if (p.trace && threadIdx.x == 0) p.trace[(size_t)row * 16 + 3] = gtimer();
    if (warp == 0) {
      // logits (bias fold added by the tail) -> tail queue
      const int qs = j % SQS;
      if (lane == 0) mbar_wait(qempty + qs, ((j / SQS) & 1) ^ 1);
      __syncwarp();
      const float var = __fdiv_rn(canon_combine(red_sq[0], red_sq[1], red_sq[2], red_sq[3]),
                                  (float)d);
      const float r = __frcp_rn(__fsqrt_rn(__fadd_rn(var, 1e-5f)));
      if (lane < K) {
        const float dot = canon_combine(red_dot[lane * 4 + 0], red_dot[lane * 4 + 1],
                                        red_dot[lane * 4 + 2], red_dot[lane * 4 + 3]);
        queue[qs].logit[lane] = __fmul_rn(r, dot);
      }
      if (lane == 0) {
        queue[qs].row = row;
        queue[qs].flags = flags0 | (hflag ? 4 : 0);
        queue[qs].pad0 = __float_as_int(sqrtf(1.f + mean * mean / var));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(qfull + qs);
    }
    ++j;
  }
  }  // compute warps
  }  // compute + tail warps
  recheck_epilogue<TW>(p, smem, &s_defer, rows_cta, row_of);   // deferred rows: STRICT
}

template <typename TW>
struct StreamLaunch {
  const PredParams &p; const StreamPlan &sp; int grid; cudaStream_t stream; int smem_optin;
  bool ldgx;
  template <int CPL> void operator()() const {
    if (ldgx) {
      if (p.K == 4 && p.H == 512 && p.policy == SPX_POLICY_MLP) {
        if (sp.w1_smem) launch<CPL, 4, 512, true, true>(); else launch<CPL, 4, 512, false, true>();
      } else {
        if (sp.w1_smem) launch<CPL, 0, 0, true, true>(); else launch<CPL, 0, 0, false, true>();
      }
      return;
    }
    if (p.K == 4 && p.H == 512 && p.policy == SPX_POLICY_MLP) {
      if (sp.w1_smem) launch<CPL, 4, 512, true, false>(); else launch<CPL, 4, 512, false, false>();
    } else {
      if (sp.w1_smem) launch<CPL, 0, 0, true, false>(); else launch<CPL, 0, 0, false, false>();
    }
  }
  template <int CPL, int KC, int HC, bool W1S, bool LDGX> void launch() const {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(predictor_stream_kernel<TW, CPL, KC, HC, W1S, LDGX>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
      configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(SW_THREADS);
    cfg.dynamicSmemBytes = sp.bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, predictor_stream_kernel<TW, CPL, KC, HC, W1S, LDGX>, p, sp);
  }
};
