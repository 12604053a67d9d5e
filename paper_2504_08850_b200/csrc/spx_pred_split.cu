// SPLIT predictor path for large batches (B >= a few hundred rows per launch):
// the fused K1+K2+K3 launch cut at its only cross-layer dependency.
//
//   K1  predictor_gather_kernel  LayerNorm + K-row LM-head gather + the K
//       local logits r * CDOT((x - mean) g, W_id) per row (model.py:298-314)
//       -> inter[row] = {logits[K], lnf, flags}.  Pure HBM streaming: it does
//       not read `prev`, so layer l+1's gather does not depend on layer l's
//       predictor at all and consecutive gathers overlap (programmatic
//       dependent launch without griddepcontrol.wait when the caller says
//       the inputs are ready, pdl == 3).
//   K2+K3  predictor_tail_kernel  softmax over the K ids + features vs the
//       carried probabilities (predictor.py:42-52), MLP + sigmoid + exact
//       threshold (predictor.py:87-109), FAST-decision certification and the
//       STRICT re-evaluation of uncertified rows -- one warp per row, W1 in
//       shared memory.  Chains layer to layer through `prev`; runs
//       concurrently with the next layer's gather on a second stream.
//
// Same arithmetic, bit for bit, as the fused STREAM kernel (spx_pred_stream.cuh):
// canonical CDOT partial groups, folded LayerNorm, the identical tail.  Only
// the schedule differs: the fused kernel's per-launch drain (last row's
// reduction + ~2.5 us MLP/certification tail) and the griddepcontrol.wait
// ramp disappear from the bandwidth-bound kernel.
#include "spx_pred_common.cuh"

namespace spx {

constexpr int GK_MAX = 8;                      // max K of the split path
constexpr int G_TEAMS = 2;                     // compute teams (rows in reduction at once)
constexpr int G_WARPS = 4 * G_TEAMS + 1;       // + producer
constexpr int G_THREADS = 32 * G_WARPS;
constexpr int G_WIN = 32;                      // ids window (rows)
constexpr int HDR = 2 + GK_MAX;                // slot header: row, flags, ids
constexpr int T_WARPS = 4;                     // tail kernel: rows per CTA pass (a 4-warp tail CTA fits beside two gather CTAs: registers)
constexpr int T_THREADS = 32 * T_WARPS;

struct GatherPlan {
  int S;                                       // LM-head slots (K rows each)
  int tail_floats;                             // per tail warp scratch (floats)
  size_t slot_bytes, off_red, off_ids, off_hdr, off_tail, off_w, off_bar, bytes;
};

constexpr int G_TAILW = 4;                     // max tail warps of the pipelined variant

inline GatherPlan plan_gather(int d, int K, int max_bytes, int tail_H = -1, int tail_K = 0) {
  GatherPlan g{};
  const size_t slot = ((size_t)K * d * 2 + 127) / 128 * 128;
  const int tf = tail_H >= 0 ? (6 * GK_MAX + tail_H + 32 + 31) / 32 * 32 : 0;
  const size_t tail = (size_t)G_TAILW * tf * 4;
  // the tail layer's W1 / b1 / w2 staged once per launch
  const size_t wbytes = tail_H > 0 ? ((size_t)3 * tail_K * tail_H + 2 * tail_H) * 4 : 0;
  const size_t fixed = (size_t)G_TEAMS * 2 * (GK_MAX + 3) * 4 * 4 + G_WIN * GK_MAX * 4 + 8 * HDR * 4 +
                       tail + wbytes + (2 * 8) * 8 + 512;
  for (int S = 6; S >= 2; --S) {
    if (fixed + S * slot > (size_t)max_bytes) continue;
    size_t o = (size_t)S * slot;
    g.S = S;
    g.tail_floats = tf;
    g.slot_bytes = slot;
    g.off_red = o; o += (size_t)G_TEAMS * 2 * (GK_MAX + 3) * 4 * 4;
    g.off_ids = o; o += G_WIN * GK_MAX * 4;
    g.off_hdr = o; o += 8 * HDR * 4;
    o = (o + 127) / 128 * 128;
    g.off_tail = o; o += tail;
    o = (o + 127) / 128 * 128;
    g.off_w = o; o += wbytes;
    o = (o + 7) / 8 * 8;
    g.off_bar = o; o += 2 * 8 * 8 + 16;
    g.bytes = o;
    return g;
  }
  return g;
}

__device__ __forceinline__ void split_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void team_bar(int team) {     // the 4 warps of one team
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(128) : "memory");
}

// Tail of one row by one warp from its gathered logits (the fused STREAM
// kernel's tail-warp code; W1 / b1 / w2 read through L1).  q = inter row.
// Returns false when the row was deferred to the STRICT re-evaluation.
template <int KC, int HC>
__device__ void warp_tail_row(const PredParams &p, int row, const float *q, float *feats,
                              float *hs, int *s_defer, int lane, const float *w1, const float *b1,
                              const float *w2) {
  const int K = KC ? KC : p.K, H = HC ? HC : p.H;
  const bool mlp = p.policy == SPX_POLICY_MLP;
  float pv[GK_MAX], x[GK_MAX], wmx[GK_MAX];
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c) {
    pv[c] = c < K ? p.prev[(size_t)row * K + c] : 0.f;
    x[c] = c < K ? q[c] : 0.f;
    wmx[c] = c < K ? q[K + c] : 0.f;
  }
  const float lnf = q[2 * K];
  const int flags = __float_as_int(q[2 * K + 1]);
  if (flags & 6) {
    if (lane == 0) {
      atomicOr(p.err, ((flags & 2) ? ERR_ID_RANGE : 0) | ((flags & 4) ? ERR_HIDDEN_NONFINITE : 0));
      if (p.fired) p.fired[row] = 0;
    }
    return;
  }
  bool bad = false;
  float m = x[0];
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c)
    if (c < K) { bad |= !is_finite(x[c]); m = fmaxf(m, x[c]); }
  float e[GK_MAX], esum = 0.f;
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c) e[c] = c < K ? np_expf(__fsub_rn(x[c], m)) : 0.f;
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c)
    if (c < K) esum = __fadd_rn(esum, e[c]);
  const float psum = np_sum_upto8(pv, K);                   // numpy pairwise (predictor.py:49)
  if (p.logits_out && lane < K) {
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) if (lane == c) p.logits_out[(size_t)row * K + c] = x[c];
  }
  int ecode = 0;
  if (bad) ecode |= ERR_LOGIT_NONFINITE;
  if (fabsf(psum - 1.0f) > 1e-5f && fabs((double)psum - 1.0) > 1e-5) ecode |= ERR_PREV_SUM;
  if (ecode) {
    if (lane == 0) {
      atomicOr(p.err, ecode);
      if (p.fired) p.fired[row] = 0;
    }
    return;
  }
  float pr[GK_MAX];
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c) pr[c] = c < K ? div_rn_unit(e[c], esum) : 0.f;
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c) {
    if (c < K && lane == c) {
      feats[c] = x[c];
      feats[K + c] = pr[c];
      feats[2 * K + c] = __fsub_rn(pr[c], pv[c]);
    }
  }
  __syncwarp();
  float z2 = 0.f;
  if (mlp) {
    mlp_z1<4, false>(feats, w1, b1, 3 * K, H, hs, lane, 0);
    __syncwarp();
    z2 = z2_tree(z2_partial(hs, w2, H, lane), z2_partial(hs, w2, H, lane + 32), hs, w2, H,
                 p.b2, lane);
  }
  float perr = 0.f;
  if (p.recheck &&
      !certify_row(p, row, feats, hs + H, hs, w1, b1, w2, z2, lnf, K, H, mlp, lane, perr,
                   [&](int c) {
                     float v = 0.f;
#pragma unroll
                     for (int cc = 0; cc < GK_MAX; ++cc) v = cc == c ? wmx[cc] : v;
                     return v;
                   })) {
    if (lane == 0) defer_row(p, row, s_defer);      // STRICT re-evaluation decides
    __syncwarp();
    return;
  }
#pragma unroll
  for (int c = 0; c < GK_MAX; ++c)
    if (c < K && lane == c) p.prev[(size_t)row * K + c] = pr[c];   // engine.py:196
  if (lane == 0 && p.prev_err) p.prev_err[row] = perr;
  if (p.feat_out)
    for (int qq = lane; qq < 3 * K; qq += 32) p.feat_out[(size_t)row * 3 * K + qq] = feats[qq];
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
  __syncwarp();
}

// K1 gather of layer l (+ optionally, TW: the K2+K3 tail of layer l-1 by two
// tail warps -- the PIPELINED form: each launch streams layer l's LM-head
// rows while finishing layer l-1's predictor, so neither the per-row tail nor
// the prev chain ever sits on the bandwidth-bound path).
// Per row (stride 2K + 2) inter[c] = r * CDOT + bw[id_c] (the local logits,
// c < K), [K + c] = wmax[id_c] (certification), [2K] = lnf =
// sqrt(1 + mean^2 / var), [2K + 1] = flags (2: id out of range, 4: non-finite
// hidden row) as float bits.
template <int CPL, int KC, int MINB, int NTM, int NTW>
__global__ void __launch_bounds__(32 * (4 * NTM + 1 + NTW), MINB)
predictor_gather_kernel(PredParams p, GatherPlan gp, float *inter, PredParams pt,
                        const float *inter_t) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = p.d, K = KC ? KC : p.K, KS = 2 * K + 2;
  const int S = gp.S;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + gp.off_bar);
  uint64_t *empty = full + 8;
  int *s_defer = reinterpret_cast<int *>(empty + 8);
  int *hdr = reinterpret_cast<int *>(smem + gp.off_hdr);      // [S][HDR]: row, flags, ids
  const uint32_t wrow = (uint32_t)d * 2u;
  const int rows_cta =
      p.B > (int)blockIdx.x ? (p.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  auto row_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    *s_defer = 0;
  }
  fence_mbar_init();
  __syncthreads();
  // pdl 3: inputs (hidden rows, ids) are not produced by the preceding
  // kernel -- no wait, let the next launch start as soon as SMs free up
  if (p.pdl == 3) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (p.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  if (warp == 4 * NTM) {
    // ============================ PRODUCER ============================
    int *ids_s = reinterpret_cast<int *>(smem + gp.off_ids);
    int j = 0;
    for (int w0 = 0; w0 < rows_cta; w0 += G_WIN) {
      int myid[GK_MAX];
      int bad = 0;
      const int ri = w0 + lane;
      const bool have = ri < rows_cta;
      const int row_i = row_of(have ? ri : 0);
      const bool skip_i = have && row_skipped(p, row_i);
#pragma unroll
      for (int c = 0; c < GK_MAX; ++c) {
        myid[c] = 0;
        if (have && !skip_i && c < K) {
          const int v = p.ids[(size_t)row_i * K + c];
          if (v < 0 || v >= p.V) bad = 1; else myid[c] = v;
        }
      }
      if (have)
#pragma unroll
        for (int c = 0; c < GK_MAX; ++c) ids_s[lane * GK_MAX + c] = myid[c];
      const unsigned badmask = __ballot_sync(0xffffffffu, bad);
      const unsigned skipmask = __ballot_sync(0xffffffffu, skip_i);
      __syncwarp();
      if (lane == 0) {
        const int wn = rows_cta - w0 < G_WIN ? rows_cta - w0 : G_WIN;
        for (int i = 0; i < wn; ++i) {
          if ((skipmask >> i) & 1) continue;
          const int s = j % S;
          if (j >= S) mbar_wait(empty + s, ((j / S) - 1) & 1);
          hdr[s * HDR + 0] = row_of(w0 + i);
          hdr[s * HDR + 1] = ((badmask >> i) & 1) ? 2 : 0;
          for (int c = 0; c < K; ++c) hdr[s * HDR + 2 + c] = ids_s[i * GK_MAX + c];
          mbar_arrive_expect_tx(full + s, (uint32_t)K * wrow);
          uint8_t *dst = smem + (size_t)s * gp.slot_bytes;
          const __nv_bfloat16 *head = reinterpret_cast<const __nv_bfloat16 *>(p.head);
          for (int c = 0; c < K; ++c)
            bulk_g2s(dst + (size_t)c * wrow, head + (size_t)ids_s[i * GK_MAX + c] * d, wrow,
                     full + s);
          ++j;
        }
      }
      __syncwarp();
      j = __shfl_sync(0xffffffffu, j, 0);
    }
  } else if (warp > 4 * NTM) {
    // ============================ TAIL WARPS (layer l-1) ============================
    if (NTW > 0 && pt.B > 0) {
      // the tail layer's MLP weights do not depend on the preceding launch:
      // staged before the wait (the two tail warps split the copy)
      const int tw = warp - 4 * NTM - 1;
      const bool tmlp = pt.policy == SPX_POLICY_MLP;
      float *w1s = reinterpret_cast<float *>(smem + gp.off_w);
      float *b1s = w1s + (tmlp ? 3 * pt.K * pt.H : 0), *w2s = b1s + pt.H;
      if (tmlp) {
        const int nw = 3 * pt.K * pt.H / 4;
        for (int i = tw * 32 + lane; i < nw; i += 32 * NTW)
          reinterpret_cast<float4 *>(w1s)[i] = __ldg(reinterpret_cast<const float4 *>(pt.w1) + i);
        for (int i = tw * 32 + lane; i < pt.H; i += 32 * NTW) { b1s[i] = pt.b1[i]; w2s[i] = pt.w2[i]; }
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + NTM), "r"(32 * NTW) : "memory");
      asm volatile("griddepcontrol.wait;" ::: "memory");   // layer l-1's launch is complete
      float *feats = reinterpret_cast<float *>(smem + gp.off_tail) + (size_t)tw * gp.tail_floats;
      float *hs = feats + 3 * GK_MAX;
      const int KT = pt.K, KST = 2 * KT + 2;
      for (int r = blockIdx.x * NTW + tw; r < pt.B; r += gridDim.x * NTW) {
        if (row_skipped(pt, r)) {
          if (lane == 0 && pt.fired) pt.fired[r] = 0;
          continue;
        }
        if (KT == 4 && pt.H == 512 && pt.policy == SPX_POLICY_MLP)
          warp_tail_row<4, 512>(pt, r, inter_t + (size_t)r * KST, feats, hs, s_defer, lane, w1s,
                                b1s, w2s);
        else
          warp_tail_row<0, 0>(pt, r, inter_t + (size_t)r * KST, feats, hs, s_defer, lane, w1s, b1s,
                              w2s);
      }
    }
  } else {

  // ============================ COMPUTE TEAMS ============================
  // team t reduces slots j = t, t + 2, ...; warp g of a team owns canonical
  // partial group g of every row (mean, variance, the K dots)
  const int team = warp >> 2, g = warp & 3;
  constexpr int KP = (KC ? (KC + 1) / 2 : GK_MAX / 2);
  float4 gr[CPL];
#pragma unroll
  for (int t = 0; t < CPL; ++t)
    gr[t] = __ldg(reinterpret_cast<const float4 *>(p.norm_g + CHUNK * (32 * g + lane + NPART * t)));
  float *red = reinterpret_cast<float *>(smem + gp.off_red) + team * 2 * (GK_MAX + 3) * 4;
  int j = 0;                                    // slot sequence (non-skipped rows)
  for (int i = 0; i < rows_cta; ++i) {
    const int row = row_of(i);
    if (row_skipped(p, row)) continue;
    const int myj = j++;
    if ((myj % NTM) != team) continue;
    const int s = myj % S;
    float *rb = red + (myj / NTM & 1) * (GK_MAX + 3) * 4;     // double-buffered partials
    float4 xr[CPL];
    const float *xg_ = p.hidden + (size_t)row * p.hidden_stride;
#pragma unroll
    for (int t = 0; t < CPL; ++t)
      xr[t] = __ldcs(reinterpret_cast<const float4 *>(xg_ + CHUNK * (32 * g + lane + NPART * t)));
    mbar_wait(full + s, (myj / S) & 1);
    const __nv_bfloat16 *wk =
        reinterpret_cast<const __nv_bfloat16 *>(smem + (size_t)s * gp.slot_bytes);
    const int flags0 = hdr[s * HDR + 1];
    // the bias fold and certification statistic of this row's ids, loaded
    // now and consumed after the reduction
    float bwv = 0.f, wmv = 0.f;
    if (g == 0 && lane < K) {
      const int id = hdr[s * HDR + 2 + lane];
      if (p.head_bw) bwv = __ldg(p.head_bw + id);
      if (p.recheck) wmv = __ldg(p.head_wmax + id);
    }
    // ---- pass 1: mean
    float part = 0.f;
#pragma unroll
    for (int t = 0; t < CPL; ++t)
      part = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(part, xr[t].x), xr[t].y), xr[t].z), xr[t].w);
    part = warp_butterfly_sum(part);
    if (lane == 0) rb[g] = part;
    team_bar(team);
    const float total = canon_combine(rb[0], rb[1], rb[2], rb[3]);
    const float mean = __fdiv_rn(total, (float)d);
    int hflag = 0;
    if (!is_finite(total)) {                      // rare: exact element scan (model.py:310-311)
      bool fin = true;
#pragma unroll
      for (int t = 0; t < CPL; ++t)
        fin &= is_finite(xr[t].x) & is_finite(xr[t].y) & is_finite(xr[t].z) & is_finite(xr[t].w);
      hflag = __any_sync(0xffffffffu, !fin) ? 1 : 0;
      int *fl = reinterpret_cast<int *>(rb + 8 + GK_MAX * 4);
      if (lane == 0) fl[g] = hflag;
      team_bar(team);
      hflag = fl[0] | fl[1] | fl[2] | fl[3];
      team_bar(team);
    }
    // ---- pass 2: variance and the K dots (LM-head rows in pairs, packed FMA)
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
          { Chunk<__nv_bfloat16> ch; ch.lds(wk + (size_t)(2 * kp) * d + CHUNK * c); ch.to_f32(wa); }
          if (2 * kp + 1 < K) {
            Chunk<__nv_bfloat16> ch; ch.lds(wk + (size_t)(2 * kp + 1) * d + CHUNK * c); ch.to_f32(wb);
          }
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
      rb[4 + g] = sq;
#pragma unroll
      for (int k = 0; k < 2 * KP; ++k) if (k < K) rb[8 + k * 4 + g] = dots[k];
    }
    team_bar(team);                               // slot fully read; partials visible
    if (g == 0) {
      if (lane == 0) split_mbar_arrive(empty + s);       // producer may refill the slot
      const float var = __fdiv_rn(canon_combine(rb[4], rb[5], rb[6], rb[7]), (float)d);
      const float r = __frcp_rn(__fsqrt_rn(__fadd_rn(var, 1e-5f)));
      float *q = inter + (size_t)row * KS;
      if (lane < K) {
        const float dot = canon_combine(rb[8 + lane * 4 + 0], rb[8 + lane * 4 + 1],
                                        rb[8 + lane * 4 + 2], rb[8 + lane * 4 + 3]);
        q[lane] = __fadd_rn(__fmul_rn(r, dot), bwv);
        q[K + lane] = wmv;
      }
      if (lane == 0) {
        q[2 * K] = sqrtf(1.f + mean * mean / var);
        q[2 * K + 1] = __int_as_float(flags0 | (hflag ? 4 : 0));
      }
    }
  }

  }  // compute teams
  // deferred tail rows of this CTA (layer l-1): the STRICT chain, scratch in
  // the (now idle) LM-head slots
  if (NTW > 0 && pt.recheck) {
    __syncthreads();
    if (*(volatile int *)s_defer) {
      float *scr = reinterpret_cast<float *>(smem);
      for (int tw = 0; tw < NTW; ++tw)
        for (int r = blockIdx.x * NTW + tw; r < pt.B; r += gridDim.x * NTW)
          if (*(volatile int *)(pt.recheck + 5 + r)) {
            __syncthreads();
            if (threadIdx.x == 0) pt.recheck[5 + r] = 0;
            recheck_row<__nv_bfloat16>(pt, r, scr);
          }
    }
  }
}

// K2+K3 from the gathered logits, ONE LANE PER ROW: a warp evaluates 32
// rows at once.  Per row the arithmetic is the fused STREAM kernel's tail
// warp's, operation for operation -- the warp-cooperative sums (the z1 units
// owned by lanes, the OpenBLAS sdot tree of z2, the butterfly sums of the
// certification bound) are replayed serially in the same association order
// (tree32 / z2 fold below), so fired / prob / prev / prev_err are bit-identical
// to spx_predictor_eval's.  The MLP weights are read as shared-memory
// broadcasts (every lane reads the same W1 element), so a 1024-row layer costs
// 32 warps -- small enough to run beside the next layer's gathers.
constexpr int TL_WARPS = 2;
constexpr int TL_THREADS = 32 * TL_WARPS;

// lane 0's result of a 32-lane xor-butterfly sum (warp_butterfly_sum)
__device__ __forceinline__ float tree32(const float *v) {
  float a[16];
#pragma unroll
  for (int l = 0; l < 16; ++l) a[l] = __fadd_rn(v[l], v[l + 16]);
#pragma unroll
  for (int l = 0; l < 8; ++l) a[l] = __fadd_rn(a[l], a[l + 8]);
#pragma unroll
  for (int l = 0; l < 4; ++l) a[l] = __fadd_rn(a[l], a[l + 4]);
#pragma unroll
  for (int l = 0; l < 2; ++l) a[l] = __fadd_rn(a[l], a[l + 2]);
  return __fadd_rn(a[0], a[1]);
}

// relu(z1_j + b1_j) of one unit (mlp_z1 order: ascending FMA chain from 0)
__device__ __forceinline__ float unit_h(const float *f, const float *w1, const float *b1, int n,
                                        int H, int j) {
  float t = 0.f;
  for (int i = 0; i < n; ++i) t = __fmaf_rn(f[i], w1[(size_t)i * H + j], t);
  return fmaxf(__fadd_rn(t, b1[j]), 0.f);
}

// The certification of one row (certify_row + mlp_margin_ok of
// spx_pred_common.cuh, replayed serially in their association order).
// hws: an upper bound of sum_j h_j |w2_j| (see the caller).  Returns whether
// the FAST decision is certified; perr = the new probabilities' error bound.
template <int KC, int HC>
__device__ __forceinline__ bool cert_lane(const PredParams &p, const float *x, const float *wm,
                                          const float *pr, const float *f, float lnf, float dprev,
                                          float z2, float hws, const float *w1s, const float *b1s,
                                          const float *w2s, float &perr) {
  const int K = KC ? KC : p.K, H = HC ? HC : p.H, n = 3 * K;
  const bool mlp = p.policy == SPX_POLICY_MLP;
  bool ok = true;
  perr = 0.f;
  {
  if (p.recheck) {
    float ev[GK_MAX], emax = 0.f, v[32];
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c)
      ev[c] = c < K ? p.cert_kappa * fmaf(p.cert_hnorm * wm[c], 1.f + lnf, fabsf(x[c])) : 0.f;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) emax = fmaxf(emax, ev[c]);
#pragma unroll
    for (int l = 0; l < 32; ++l) v[l] = 0.f;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) if (c < K) v[c] = pr[c] * ev[c] + 0.f;
    const float spe = tree32(v);
    const float slackp = 8.f * U24 * (float)(K + 4);
    float df[3 * GK_MAX];
#pragma unroll
    for (int c = 0; c < 3 * GK_MAX; ++c) df[c] = 0.f;
    float pe = 0.f;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) {
      if (c < K) {
        const float dp = fmaf(pr[c], ev[c] + spe + slackp, 2.f * emax * emax);
        df[c] = ev[c];
        df[K + c] = dp;
        df[2 * K + c] = dp + dprev + 2.f * U24 * fabsf(f[2 * K + c]);
        pe = fmaxf(pe, dp);
      }
    }
    perr = pe;
    if (mlp && fabsf(p.z_cut) <= 3.0e38f) {
      const float *M = p.cert;
      float vs[32], vf[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) { vs[l] = 0.f; vf[l] = 0.f; }
#pragma unroll
      for (int i = 0; i < 3 * GK_MAX; ++i)
        if (i < n) { vs[i] = fmaf(M[i], df[i], 0.f); vf[i] = fmaf(fabsf(f[i]), M[i], 0.f); }
      const float sm = tree32(vs), sfm = tree32(vf);
      const float lu = CERT_LAMBDA * U24;
      const float rz1 = lu * sqrtf((float)(n + 1));
      auto eps_of = [&](float shw) {
        return 2.f * (rz1 * (sfm + M[n]) + lu * sqrtf((float)H / 64.f + 8.f) * shw) +
               4.f * U24 * (fabsf(z2) + fabsf(p.b2));
      };
      const float gap = fabsf(z2 - p.z_cut);
      float eps_r = eps_of(hws * 1.001f);
      bool loose = gap > (sm + eps_r) * 1.0001f;
      if (!loose) {                            // exact shw: residue classes of 32
        float hw[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) hw[l] = 0.f;
        for (int j = 0; j < H; ++j)
          hw[j & 31] = fmaf(unit_h(f, w1s, b1s, n, H, j), fabsf(w2s[j]), hw[j & 31]);
        eps_r = eps_of(tree32(hw));
        loose = gap > (sm + eps_r) * 1.0001f;
      }
      if (!loose) {
        // tight pass (rare): classify units, gradient of the surely-active part
        // (the active set as a bit mask, so the per-input gradient sums can
        // run input by input in mlp_margin_ok's residue-class order)
        float bs[32];
        uint32_t act[MAXH / 32];
#pragma unroll
        for (int l = 0; l < 32; ++l) bs[l] = 0.f;
        for (int w = 0; w < MAXH / 32; ++w) act[w] = 0u;
        for (int j = 0; j < H; ++j) {
          float z1 = 0.f, dz = 0.f, fa = 0.f;
          for (int i = 0; i < n; ++i) {
            const float w = w1s[(size_t)i * H + j];
            z1 = fmaf(f[i], w, z1);
            dz = fmaf(fabsf(w), df[i], dz);
            fa = fmaf(fabsf(f[i]), fabsf(w), fa);
          }
          z1 += b1s[j];
          dz = dz * 1.0001f + 2.f * rz1 * (fa + fabsf(b1s[j])) + 4.f * U24 * fabsf(z1);
          if (z1 > dz) act[j >> 5] |= 1u << (j & 31);
          else if (z1 >= -dz) bs[j & 31] = fmaf(fabsf(w2s[j]), dz, bs[j & 31]);
        }
        const float bsum = tree32(bs);
        float gs = 0.f;
        for (int i = 0; i < n; ++i) {
          float g[32];
#pragma unroll
          for (int l = 0; l < 32; ++l) g[l] = 0.f;
          for (int j = 0; j < H; ++j) {
            const float coef = ((act[j >> 5] >> (j & 31)) & 1u) ? w2s[j] : 0.f;
            g[j & 31] = fmaf(coef, w1s[(size_t)i * H + j], g[j & 31]);
          }
          gs = fmaf(fabsf(tree32(g)), df[i], gs);
        }
        ok = gap > (gs + bsum + eps_r) * 1.0001f;
      }
    }
  }
  }
  return ok;
}

template <int KC, int HC, int LPR>
__global__ void __launch_bounds__(TL_THREADS, 7)
predictor_tail_lanes_kernel(PredParams p, const float *inter) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = KC ? KC : p.K, H = HC ? HC : p.H, n = 3 * K, KS = 2 * K + 2;
  const bool mlp = p.policy == SPX_POLICY_MLP;
  float *w1s = reinterpret_cast<float *>(smem);
  float *b1s = w1s + (mlp ? n * H : 0);
  float *w2s = b1s + H;
  __shared__ int s_defer;
  if (threadIdx.x == 0) s_defer = 0;
  if (mlp) {
    for (int i = threadIdx.x; i < n * H / 4; i += TL_THREADS)
      reinterpret_cast<float4 *>(w1s)[i] = __ldg(reinterpret_cast<const float4 *>(p.w1) + i);
    for (int i = threadIdx.x; i < H; i += TL_THREADS) { b1s[i] = p.b1[i]; w2s[i] = p.w2[i]; }
  }
  const int row = (blockIdx.x * TL_THREADS + threadIdx.x) / LPR;
  bool live = row < p.B && !row_skipped(p, row);
  float x[GK_MAX], wm[GK_MAX], pv[GK_MAX];
  float lnf = 0.f, dprev = 0.f;
  int flags = 0;
  if (row < p.B && !live && p.fired && (lane & (LPR - 1)) == 0) p.fired[row] = 0;
  if (live) {                                   // one round trip for every input of the row
    const float *q = inter + (size_t)row * KS;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) {
      x[c] = c < K ? q[c] : 0.f;
      wm[c] = c < K ? q[K + c] : 0.f;
      pv[c] = c < K ? p.prev[(size_t)row * K + c] : 0.f;
    }
    lnf = q[2 * K];
    flags = __float_as_int(q[2 * K + 1]);
    if (p.prev_err) dprev = p.prev_err[row];
  }
  __syncthreads();                              // weights staged
  if (live && (flags & 6)) {
    atomicOr(p.err, ((flags & 2) ? ERR_ID_RANGE : 0) | ((flags & 4) ? ERR_HIDDEN_NONFINITE : 0));
    if (p.fired) p.fired[row] = 0;
    live = false;
  }
  float pr[GK_MAX], f[3 * GK_MAX];
  if (live) {
    // softmax over the K ids (model.py:149-152), features (predictor.py:42-52)
    bool bad = false;
    float m = x[0];
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c)
      if (c < K) { bad |= !is_finite(x[c]); m = fmaxf(m, x[c]); }
    float e[GK_MAX], esum = 0.f;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) e[c] = c < K ? np_expf(__fsub_rn(x[c], m)) : 0.f;
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c)
      if (c < K) esum = __fadd_rn(esum, e[c]);
    const float psum = np_sum_upto8(pv, K);                 // numpy pairwise (predictor.py:49)
    if (p.logits_out)
      for (int c = 0; c < K; ++c) p.logits_out[(size_t)row * K + c] = x[c];
    int ecode = 0;
    if (bad) ecode |= ERR_LOGIT_NONFINITE;
    if (fabsf(psum - 1.0f) > 1e-5f && fabs((double)psum - 1.0) > 1e-5) ecode |= ERR_PREV_SUM;
    if (ecode) {
      atomicOr(p.err, ecode);
      if (p.fired) p.fired[row] = 0;
      live = false;
    }
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c) {
      pr[c] = c < K ? div_rn_unit(e[c], esum) : 0.f;
      f[c] = 0.f; f[GK_MAX + c] = 0.f; f[2 * GK_MAX + c] = 0.f;
    }
#pragma unroll
    for (int c = 0; c < GK_MAX; ++c)
      if (c < K) { f[c] = x[c]; f[K + c] = pr[c]; f[2 * K + c] = __fsub_rn(pr[c], pv[c]); }
  }
  float z2 = 0.f, hws = 0.f;
  if constexpr (LPR == 1) {
    if (live && mlp) {
      // ---- MLP: z1 units, the z2 sdot accumulators A[c] and the certification's
      // sum |w2_j| h_j in residue classes of 32 (warp_mlp / mlp_margin_ok order)
      // shw_ub: an upper bound of the certification's sum_j h_j |w2_j| (any
      // order, +0.1%); the exact residue-class sum is computed only for rows
      // the bound does not certify at once, so the outcome equals the warp
      // version's (the check is monotone in shw)
      const int n1 = H & ~31, n64 = n1 & ~63;
      {
        float A[64];
  #pragma unroll
        for (int c = 0; c < 64; ++c) A[c] = 0.f;
        for (int b0 = 0; b0 < n64; b0 += 64) {
  #pragma unroll
          for (int c4 = 0; c4 < 64; c4 += 4) {
            const int j = b0 + c4;
            float t[4] = {0.f, 0.f, 0.f, 0.f};
  #pragma unroll
            for (int i = 0; i < 3 * GK_MAX; ++i) {
              if (i < n) {
                const float4 w = *reinterpret_cast<const float4 *>(w1s + (size_t)i * H + j);
                t[0] = __fmaf_rn(f[i], w.x, t[0]); t[1] = __fmaf_rn(f[i], w.y, t[1]);
                t[2] = __fmaf_rn(f[i], w.z, t[2]); t[3] = __fmaf_rn(f[i], w.w, t[3]);
              }
            }
            const float4 bb = *reinterpret_cast<const float4 *>(b1s + j);
            const float4 ww = *reinterpret_cast<const float4 *>(w2s + j);
            const float h0 = fmaxf(__fadd_rn(t[0], bb.x), 0.f), h1 = fmaxf(__fadd_rn(t[1], bb.y), 0.f);
            const float h2 = fmaxf(__fadd_rn(t[2], bb.z), 0.f), h3 = fmaxf(__fadd_rn(t[3], bb.w), 0.f);
            A[c4 + 0] = __fmaf_rn(h0, ww.x, A[c4 + 0]); A[c4 + 1] = __fmaf_rn(h1, ww.y, A[c4 + 1]);
            A[c4 + 2] = __fmaf_rn(h2, ww.z, A[c4 + 2]); A[c4 + 3] = __fmaf_rn(h3, ww.w, A[c4 + 3]);
            hws = fmaf(h0, fabsf(ww.x), fmaf(h1, fabsf(ww.y),
                       fmaf(h2, fabsf(ww.z), fmaf(h3, fabsf(ww.w), hws))));
          }
        }
        // z2_tree (spx_pred_common.cuh) replayed: fold 16 -> 8, the optional
        // 32-element step, lane-wise ((a0 + a1) + a2) + a3, 8 -> 4, quad sum
        float blo[32], bhi[32];
  #pragma unroll
        for (int l = 0; l < 24; ++l) { blo[l] = __fadd_rn(A[l], A[l + 8]); bhi[l] = __fadd_rn(A[l + 32], A[l + 40]); }
        if (n1 > n64) {
  #pragma unroll
          for (int l = 0; l < 24; ++l) {
            const int mm = l & 15;
            if (mm < 8) {
              const int a2 = l >> 4;
              const int ja = n64 + 8 * a2 + mm, jb = n64 + 8 * (a2 + 2) + mm;
              const float ha = unit_h(f, w1s, b1s, n, H, ja), hb = unit_h(f, w1s, b1s, n, H, jb);
              blo[l] = __fmaf_rn(ha, w2s[ja], blo[l]);
              bhi[l] = __fmaf_rn(hb, w2s[jb], bhi[l]);
            }
          }
          for (int j = n64; j < n1; ++j)
            hws = fmaf(unit_h(f, w1s, b1s, n, H, j), fabsf(w2s[j]), hws);
        }
        float sv[8];
  #pragma unroll
        for (int l = 0; l < 8; ++l)
          sv[l] = __fadd_rn(__fadd_rn(__fadd_rn(blo[l], blo[l + 16]), bhi[l]), bhi[l + 16]);
        float qv[4];
  #pragma unroll
        for (int l = 0; l < 4; ++l) qv[l] = __fadd_rn(sv[l], sv[l + 4]);
        float dot = n1 ? __fadd_rn(__fadd_rn(qv[0], qv[1]), __fadd_rn(qv[2], qv[3])) : 0.f;
        for (int j = n1; j < H; ++j) {
          const float h = unit_h(f, w1s, b1s, n, H, j);
          dot = __fadd_rn(dot, __fmul_rn(h, w2s[j]));
          hws = fmaf(h, fabsf(w2s[j]), hws);
        }
        z2 = __fadd_rn(dot, p.b2);
      }

    }
  } else {
    // LPR lanes per row: lane q of a row owns the z2 accumulators A[c],
    // c in [16q, 16q + 16) (H % 64 == 0, K == 4): the 16 -> 8 fold is local
    // (blo / bhi of the warp version), the lane-wise ((a0 + a1) + a2) + a3 is
    // a 4-lane gather.  Executed by every lane (shuffles); dead rows compute
    // on zeros and write nothing.
    static_assert(LPR == 4, "LPR");
    const int qd = lane & (LPR - 1), base = lane & ~(LPR - 1);
    if (mlp) {
      float A[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) A[c] = 0.f;
      for (int b0 = 0; b0 < H; b0 += 64) {
#pragma unroll
        for (int c4 = 0; c4 < 16; c4 += 4) {
          const int j = b0 + 16 * qd + c4;
          float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < 3 * GK_MAX; ++i) {
            if (i < n) {
              const float4 w = *reinterpret_cast<const float4 *>(w1s + (size_t)i * H + j);
              t[0] = __fmaf_rn(f[i], w.x, t[0]); t[1] = __fmaf_rn(f[i], w.y, t[1]);
              t[2] = __fmaf_rn(f[i], w.z, t[2]); t[3] = __fmaf_rn(f[i], w.w, t[3]);
            }
          }
          const float4 bb = *reinterpret_cast<const float4 *>(b1s + j);
          const float4 ww = *reinterpret_cast<const float4 *>(w2s + j);
          const float h0 = fmaxf(__fadd_rn(t[0], bb.x), 0.f), h1 = fmaxf(__fadd_rn(t[1], bb.y), 0.f);
          const float h2 = fmaxf(__fadd_rn(t[2], bb.z), 0.f), h3 = fmaxf(__fadd_rn(t[3], bb.w), 0.f);
          A[c4 + 0] = __fmaf_rn(h0, ww.x, A[c4 + 0]); A[c4 + 1] = __fmaf_rn(h1, ww.y, A[c4 + 1]);
          A[c4 + 2] = __fmaf_rn(h2, ww.z, A[c4 + 2]); A[c4 + 3] = __fmaf_rn(h3, ww.w, A[c4 + 3]);
          hws = fmaf(h0, fabsf(ww.x), fmaf(h1, fabsf(ww.y),
                     fmaf(h2, fabsf(ww.z), fmaf(h3, fabsf(ww.w), hws))));
        }
      }
      float sv[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float bq = __fadd_rn(A[l], A[l + 8]);
        const float b1 = __shfl_sync(0xffffffffu, bq, base + 1);
        const float b2 = __shfl_sync(0xffffffffu, bq, base + 2);
        const float b3 = __shfl_sync(0xffffffffu, bq, base + 3);
        sv[l] = __fadd_rn(__fadd_rn(__fadd_rn(bq, b1), b2), b3);
      }
      float qv[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) qv[l] = __fadd_rn(sv[l], sv[l + 4]);
      z2 = __fadd_rn(__fadd_rn(__fadd_rn(qv[0], qv[1]), __fadd_rn(qv[2], qv[3])), p.b2);
      z2 = __shfl_sync(0xffffffffu, z2, base);
      hws += __shfl_xor_sync(0xffffffffu, hws, 1);
      hws += __shfl_xor_sync(0xffffffffu, hws, 2);
    }
  }
  if (live) {
    float perr = 0.f;
    const bool ok = cert_lane<KC, HC>(p, x, wm, pr, f, lnf, dprev, z2, hws, w1s, b1s, w2s, perr);
    const bool writer = LPR == 1 || (lane & (LPR - 1)) == 0;
    if (writer) {
      if (!ok) {
        p.recheck[5 + row] = 1;                  // STRICT re-evaluation decides
        atomicAdd(&s_defer, 1);
      } else {
        for (int c = 0; c < K; ++c) p.prev[(size_t)row * K + c] = pr[c];   // engine.py:196
        if (p.prev_err) p.prev_err[row] = perr;
        if (p.feat_out)
          for (int qq = 0; qq < n; ++qq) p.feat_out[(size_t)row * n + qq] = f[qq];
        if (p.evals) p.evals[row] += 1;
        if (mlp) {
          if (p.z_out) p.z_out[row] = z2;
          if (p.prob_out) p.prob_out[row] = (double)sigmoid32(z2);
          write_fired(p, row, z2 >= p.z_cut);
        } else {
          if (p.prob_out) p.prob_out[row] = p.const_prob;
          if (p.z_out) p.z_out[row] = 0.0f;
          write_fired(p, row, p.const_prob > p.threshold);
        }
      }
    }
  }
  // deferred rows of this CTA: the STRICT chain (scratch aliases the weights)
  __syncthreads();
  if (!p.recheck || s_defer == 0) return;
  float *scr = reinterpret_cast<float *>(smem);
  const int r0 = blockIdx.x * (TL_THREADS / LPR);
  for (int r = r0; r < r0 + TL_THREADS / LPR && r < p.B; ++r)
    if (*(volatile int *)(p.recheck + 5 + r)) {
      __syncthreads();
      if (threadIdx.x == 0) p.recheck[5 + r] = 0;
      recheck_row<__nv_bfloat16>(p, r, scr);
    }
}

static int g_split_sms = 0, g_split_optin = 0;
static void split_limits() {
  if (g_split_sms) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_split_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&g_split_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (g_split_sms <= 0) g_split_sms = 148;
}

template <int CPL, int KC, int MINB, int NTM, int NTW>
static int launch_gather_t(const PredParams &p, const GatherPlan &gp, int grid, float *inter,
                           const PredParams &pt, const float *inter_t, cudaStream_t s) {
  auto kern = predictor_gather_kernel<CPL, KC, MINB, NTM, NTW>;
  static size_t configured = 48 * 1024;
  if (gp.bytes > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gp.bytes) !=
        cudaSuccess)
      return SPX_EINVAL;
    configured = gp.bytes;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * (4 * NTM + 1 + NTW));
  cfg.dynamicSmemBytes = gp.bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, p, gp, inter, pt, inter_t);
  return 0;
}

// Which shapes the split path takes (the caller falls back to the fused kernel).
bool split_supported(const PredParams &p, int head_dtype) {
  return head_dtype == SPX_DTYPE_BF16 && p.K <= GK_MAX &&
         (p.d == 2048 || p.d == 4096 || p.d == 8192) &&
         (p.policy != SPX_POLICY_MLP || (p.H <= MAXH && p.H % 4 == 0));
}

// pt == nullptr: the plain gather; else the pipelined form (tail warps finish
// layer pt->layer, whose gathered logits are inter_t, after the preceding
// launch completes).
int launch_split_gather(const PredParams &p, float *inter, const PredParams *pt,
                        const float *inter_t, cudaStream_t s) {
  split_limits();
  // two CTAs per SM (the next launch's CTAs take an SM's slot as soon as one
  // of this launch's CTAs retires) unless the row width needs the registers
  const int per_sm = p.d <= 4096 ? 2 : 1;
  // SPX_SPLIT_GATHER_KB (sweeps): shared-memory budget of one gather CTA
  static const int env_kb = getenv("SPX_SPLIT_GATHER_KB") ? atoi(getenv("SPX_SPLIT_GATHER_KB")) : 0;
  const int tH = pt ? (pt->policy == SPX_POLICY_MLP ? pt->H : 0) : -1;
  const int budget = (env_kb > 0 ? env_kb * 1024 : per_sm == 2 ? 70 * 1024 : 180 * 1024) +
                     (pt ? 10 * 1024 + (tH > 0 ? (3 * pt->K * tH + 2 * tH) * 4 : 0) : 0);
  const GatherPlan gp = plan_gather(p.d, p.K, budget, tH, pt ? pt->K : 0);
  if (!gp.bytes) return SPX_EINVAL;
  if (pt && pt->recheck && recheck_scratch_bytes(pt->d, pt->K) > (size_t)gp.S * gp.slot_bytes)
    return SPX_EINVAL;
  const long long cap = (long long)per_sm * g_split_sms;
  const int rows = p.B > 0 ? p.B : pt ? pt->B : 0;      // B = 0: tail warps only
  const int grid = (int)(rows < cap ? rows : cap);
  PredParams none{};
  const PredParams &q = pt ? *pt : none;
  // SPX_SPLIT_PIPE (A/B): 1 = one compute team + 4 tail warps (default:
  // 10.8 vs 12.2 us per layer at the bench shape), 2 = two teams + 2 tail warps
  static const int env_pipe = getenv("SPX_SPLIT_PIPE") ? atoi(getenv("SPX_SPLIT_PIPE")) : 1;
#define SPX_G(CPL, KC, MB)                                                                     \
  return !pt ? launch_gather_t<CPL, KC, MB, 2, 0>(p, gp, grid, inter, q, inter_t, s)           \
       : env_pipe == 1 ? launch_gather_t<CPL, KC, MB, 1, 4>(p, gp, grid, inter, q, inter_t, s) \
                       : launch_gather_t<CPL, KC, MB, 2, 2>(p, gp, grid, inter, q, inter_t, s)
  if (p.d == 2048) {
    if (p.K == 4) SPX_G(4, 4, 2);
    SPX_G(4, 0, 2);
  }
  if (p.d == 4096) {
    if (p.K == 4) SPX_G(8, 4, 2);
    SPX_G(8, 0, 2);
  }
  if (p.K == 4) SPX_G(16, 4, 1);
  SPX_G(16, 0, 1);
#undef SPX_G
}

template <int KC, int HC, int LPR>
static int launch_tail_t(const PredParams &p, const float *inter, size_t smem, cudaStream_t s) {
  static size_t configured = 48 * 1024;
  static bool carved = false;
  if (!carved) {
    cudaFuncSetAttribute(predictor_tail_lanes_kernel<KC, HC, LPR>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carved = true;
  }
  if (smem > configured) {
    if (cudaFuncSetAttribute(predictor_tail_lanes_kernel<KC, HC, LPR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SPX_EINVAL;
    configured = smem;
  }
  const int rows_cta = TL_THREADS / LPR;
  const int grid = (p.B + rows_cta - 1) / rows_cta;
  predictor_tail_lanes_kernel<KC, HC, LPR><<<grid, TL_THREADS, smem, s>>>(p, inter);
  return 0;
}

int launch_split_tail(const PredParams &p, const float *inter, cudaStream_t s) {
  split_limits();
  const bool mlp = p.policy == SPX_POLICY_MLP;
  size_t smem = (size_t)(mlp ? 3 * p.K * p.H + 2 * p.H : 0) * 4;
  if (p.recheck) {
    const size_t rscr = recheck_scratch_bytes(p.d, p.K);
    if (rscr > smem) smem = rscr;
  }
  if (smem < 16) smem = 16;
  if (smem > (size_t)g_split_optin) return SPX_EINVAL;
  // 4 lanes per row for the paper's K = 4, H = 512 predictor (shorter per-row
  // chains, 4x the warps); 1 lane per row otherwise.  SPX_SPLIT_LPR=1 forces
  // the latter (A/B runs).
  static const int env_lpr = getenv("SPX_SPLIT_LPR") ? atoi(getenv("SPX_SPLIT_LPR")) : 4;
  if (mlp && p.K == 4 && p.H == 512) {
    if (env_lpr == 4) return launch_tail_t<4, 512, 4>(p, inter, smem, s);
    return launch_tail_t<4, 512, 1>(p, inter, smem, s);
  }
  return launch_tail_t<0, 0, 1>(p, inter, smem, s);
}

}  // namespace spx
