// FAST fused predictor kernel (included by spx_predictor.cu, namespace spx).
//
// Persistent, one CTA per SM, warp-specialised into a two-stage pipeline:
//   * NTEAM DOT teams of 4 warps.  Team t owns CTA rows t, t+NTEAM, ...  Warp
//     w of a team owns canonical partial group g = w, so every per-row
//     reduction is split four ways.  Each team streams its own LM-head rows
//     through a private double-buffered shared-memory ring: one "unit" is
//     HALF = 2 vocab rows (16 KiB at 7B) fetched with 1-D TMA bulk copies
//     (cp.async.bulk, mbarrier complete_tx).  The team leader re-arms a slot
//     as soon as the team has consumed it, so the next row's LM-head rows are
//     in flight while the current row is being reduced.  The hidden row (f32)
//     is loaded straight into registers one row ahead.  A team computes the
//     LayerNorm statistics and the K local logits and hands them to a tail
//     warp through a shared-memory queue.
//   * NTAIL TAIL warps: softmax over the K ids + features, the MLP (W1, b1,
//     w2 resident in shared memory), f64 sigmoid, strict threshold, outputs.
//     The tail of row k overlaps the streaming of later rows.
// Fast-path algebra (canonical, shared with K4/K6):
//   mean = CSUM(x)/d ; xc = x - mean ; var = CSUM(xc*xc)/d ; r = 1/sqrt(var+eps)
//   logit_v = r * CDOT(xc*g, W_v) + bw_v      (bw_v = CDOT(b, W_v), per model)
// i.e. the LayerNorm is folded into the head dot (one pass over the row for
// the variance and the K dots), with packed FP32 (FADD2/FMUL2/FFMA2).

#include <type_traits>

#ifndef SPX_FAST_NTEAM
#define SPX_FAST_NTEAM 4
#endif
constexpr int NTEAM = SPX_FAST_NTEAM;           // DOT teams (2 in the wide-row variant)
constexpr int TEAM = 4;
constexpr int NTAIL = 4;
constexpr int HALF = 2;                        // LM-head rows per TMA unit
constexpr int MAX_RING = 3;                    // units in flight per team (2 or 3)
constexpr int QS = 8;                          // tail queue slots (multiple of NTEAM, NTAIL)
constexpr int RED_FLOATS = 32;
constexpr int FAST_THREADS = 32 * (TEAM * NTEAM + NTAIL);

struct QSlot {                                 // dot team -> tail warp hand-off
  int row, flags, pad0, pad1;                  // flags: 1 skip, 2 bad id, 4 bad hidden
  float logits[MAXK];
  float prev[MAXK];
};

struct SmemPlan {
  int w1_smem;     // W1 staged in shared memory?
  int ring;        // TMA units in flight per team
  int g_smem;      // final_norm.g staged in shared memory (else read through L1)
  size_t bytes;
  size_t off_g, off_w2, off_b1, off_w1, off_team, team_bytes, off_ring, unit_bytes, off_tail,
      tail_bytes, off_q, off_bar;
};

template <typename TW>
inline SmemPlan plan_smem_ring(int d, int K, int H, int max_bytes, int force_w1, int ring,
                               bool g_smem = true) {
  SmemPlan s{};
  const size_t gb = g_smem ? (size_t)d * 4 : 0;
  const size_t unit = ((size_t)HALF * d * sizeof(TW) + 127) / 128 * 128;
  const size_t team = ((size_t)(RED_FLOATS + 4 + MAXK) * 4 + 127) / 128 * 128;
  const size_t tail = ((size_t)(6 * MAXK + (H > 0 ? H : 4) + 64) * 4 + 127) / 128 * 128;
  const size_t qbytes = (sizeof(QSlot) * QS + 127) / 128 * 128;
  const size_t w1b = ((size_t)3 * K * H * 4 + 127) / 128 * 128;
  const size_t bars = (NTEAM * MAX_RING + 2 * QS + 2) * 8;    // + the deferred-row count
  const size_t base = (gb + (size_t)2 * H * 4 + 127) / 128 * 128 + NTEAM * team +
                      (size_t)NTEAM * ring * unit + NTAIL * tail + qbytes + bars + 128;
  const bool w1 = H > 0 && force_w1 != 0 && base + w1b <= (size_t)max_bytes;
  if (base > (size_t)max_bytes) return s;          // does not fit: bytes == 0
  size_t o = 0;
  s.w1_smem = w1;
  s.ring = ring;
  s.g_smem = g_smem;
  s.off_g = o; o += gb;
  s.off_w2 = o; o += (size_t)H * 4;
  s.off_b1 = o; o += (size_t)H * 4;
  o = (o + 127) / 128 * 128;
  s.off_w1 = o; if (w1) o += w1b;
  s.off_team = o; s.team_bytes = team; o += NTEAM * team;
  s.off_ring = o; s.unit_bytes = unit; o += (size_t)NTEAM * ring * unit;
  s.off_tail = o; s.tail_bytes = tail; o += NTAIL * tail;
  s.off_q = o; o += qbytes;
  s.off_bar = o; o += bars;
  s.bytes = o;
  return s;
}

// Ring depth 2 (one row's LM-head rows per team in flight); force_ring = 3
// (sweeps) trades W1/g shared-memory residency for a third unit.
template <typename TW>
inline SmemPlan plan_smem(int d, int K, int H, int max_bytes, int force_w1 = -1,
                          int force_ring = -1) {
  if (force_ring == 3) {     // measured slower at 7B (W1 and g then come from L1)
    SmemPlan s = plan_smem_ring<TW>(d, K, H, max_bytes, force_w1, 3);
    if (!s.bytes) s = plan_smem_ring<TW>(d, K, H, max_bytes, force_w1, 3, false);
    if (s.bytes) return s;
  }
  return plan_smem_ring<TW>(d, K, H, max_bytes, force_w1, 2);
}

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// KC / HC: compile-time K / H (0 = runtime) -- the K=4, H=512 configuration
// of the paper gets fully unrolled softmax, MLP and dot loops.
template <typename TW, int CPL, bool FULL, bool W1S, int KC, int HC, int RING>
__global__ void __launch_bounds__(FAST_THREADS, 1)
predictor_fast_kernel(PredParams p, SmemPlan sp) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = p.d, K = KC ? KC : p.K, H = HC ? HC : p.H, nchunk = d / CHUNK;
  const float *gs = sp.g_smem ? reinterpret_cast<const float *>(smem + sp.off_g) : p.norm_g;
  float *w2s = reinterpret_cast<float *>(smem + sp.off_w2);
  float *b1s = reinterpret_cast<float *>(smem + sp.off_b1);
  float *w1s = reinterpret_cast<float *>(smem + sp.off_w1);
  QSlot *queue = reinterpret_cast<QSlot *>(smem + sp.off_q);
  uint64_t *ringbar = reinterpret_cast<uint64_t *>(smem + sp.off_bar);   // [NTEAM][RING]
  uint64_t *qfull = ringbar + NTEAM * MAX_RING;
  uint64_t *qempty = qfull + QS;
  uint64_t *setup_bar = qempty + QS;
  const TW *head = reinterpret_cast<const TW *>(p.head);
  const bool mlp = p.policy == SPX_POLICY_MLP;
  const bool bulk_consts = (H % 4) == 0;
  const uint32_t wrow_bytes = (uint32_t)((size_t)d * sizeof(TW));
  const int nhalf = (K + HALF - 1) / HALF;          // units per row
  const int rows_cta =
      p.B > (int)blockIdx.x ? (p.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;

  int &s_defer = *reinterpret_cast<int *>(setup_bar + 1);   // rows deferred (recheck)
  if (threadIdx.x == 0) {
    s_defer = 0;
    for (int s = 0; s < NTEAM * RING; ++s) mbar_init(ringbar + s, 1);
    for (int s = 0; s < QS; ++s) { mbar_init(qfull + s, 1); mbar_init(qempty + s, 1); }
    mbar_init(setup_bar, 1);
  }
  fence_mbar_init();
  __syncthreads();
  if (threadIdx.x == 0) {                  // per-CTA constants (weights) by TMA
    uint32_t bytes = sp.g_smem ? (uint32_t)d * 4u : 0u;
    if (mlp && bulk_consts) bytes += 2u * H * 4u + (sp.w1_smem ? 3u * K * H * 4u : 0u);
    mbar_arrive_expect_tx(setup_bar, bytes);
    if (sp.g_smem) bulk_g2s(smem + sp.off_g, p.norm_g, (uint32_t)d * 4u, setup_bar);
    if (mlp && bulk_consts) {
      bulk_g2s(w2s, p.w2, (uint32_t)H * 4u, setup_bar);
      bulk_g2s(b1s, p.b1, (uint32_t)H * 4u, setup_bar);
      if (sp.w1_smem) bulk_g2s(w1s, p.w1, 3u * K * H * 4u, setup_bar);
    }
  }
  if (mlp && !bulk_consts) {               // ragged H: plain copies
    for (int i = threadIdx.x; i < H; i += blockDim.x) { w2s[i] = p.w2[i]; b1s[i] = p.b1[i]; }
    if (sp.w1_smem)
      for (int i = threadIdx.x; i < 3 * K * H; i += blockDim.x) w1s[i] = p.w1[i];
    __syncthreads();
  }
  // Programmatic dependent launch: everything above touches only weights;
  // per-request inputs (hidden rows, ids, prev, engine flags) may be written
  // by the previous kernel in the stream, so wait for it here, then let the
  // next kernel's CTAs start their own prologue as SMs free up.
  // pdl == 2 ("ids ready"): the dot teams first issue the LM-head prefetch of
  // their first rows -- it depends only on ids and the head -- and wait after.
  const bool early = p.pdl == 2 && !p.row_done && !p.row_layer_mask;
  if (p.pdl && !early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (early && warp >= TEAM * NTEAM) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  if (warp >= TEAM * NTEAM) {
    // =========================== TAIL WARPS ===========================
    const int tw = warp - TEAM * NTEAM;
    float *feats = reinterpret_cast<float *>(smem + sp.off_tail + (size_t)tw * sp.tail_bytes);
    float *hs = feats + 3 * MAXK;
    mbar_wait(setup_bar, 0);
    if (mlp && !bulk_consts) __syncwarp();
    for (int k = tw; k < rows_cta; k += NTAIL) {
      const int slot = k % QS;
      mbar_wait(qfull + slot, (k / QS) & 1);
      const QSlot &q = queue[slot];
      const int row = q.row, flags = q.flags, q_lnf = q.pad0;
      if (p.trace && lane == 0 && !(flags & 1)) {
        p.trace[(size_t)row * 16 + 0] = gtimer();
        p.trace[(size_t)row * 16 + 8] = clock64();
      }
      if constexpr (KC > 0 && KC <= 8) {
        // every lane holds all K logits: no shuffles on the critical path
        float x[KC], pv[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) { x[c] = q.logits[c]; pv[c] = q.prev[c]; }
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty + slot);             // slot consumed
        if (flags & 1) {                                        // skipped row
          if (lane == 0 && p.fired) p.fired[row] = 0;
          continue;
        }
        if (flags & 6) {
          if (lane == 0) {
            atomicOr(p.err, ((flags & 2) ? ERR_ID_RANGE : 0) | ((flags & 4) ? ERR_HIDDEN_NONFINITE : 0));
            if (p.fired) p.fired[row] = 0;
          }
          continue;
        }
        bool bad = false;
        float m = x[0];
#pragma unroll
        for (int c = 0; c < KC; ++c) { bad |= !is_finite(x[c]); m = fmaxf(m, x[c]); }
        float e[KC], esum = 0.f, psum = 0.f;
#pragma unroll
        for (int c = 0; c < KC; ++c) e[c] = np_expf(__fsub_rn(x[c], m));
#pragma unroll
        for (int c = 0; c < KC; ++c) esum = __fadd_rn(esum, e[c]);
        {
          float pv8[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) pv8[c] = c < KC ? pv[c] : 0.f;
          psum = np_sum_upto8(pv8, KC);                     // numpy pairwise (predictor.py:49)
        }
        if (p.logits_out && lane < KC) {
#pragma unroll
          for (int c = 0; c < KC; ++c) if (lane == c) p.logits_out[(size_t)row * KC + c] = x[c];
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
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          if (lane == c) {
            const float pr = __fdiv_rn(e[c], esum);
            feats[c] = x[c];
            feats[KC + c] = pr;
            feats[2 * KC + c] = __fsub_rn(pr, pv[c]);
          }
        }
      } else {
        const bool v0 = lane < K, v1 = lane + 32 < K;
        const float x0 = v0 ? q.logits[lane] : 0.f, x1 = v1 ? q.logits[lane + 32] : 0.f;
        const float pv0 = v0 ? q.prev[lane] : 0.f, pv1 = v1 ? q.prev[lane + 32] : 0.f;
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty + slot);               // slot consumed
        if (flags & 1) {                                          // skipped row
          if (lane == 0 && p.fired) p.fired[row] = 0;
          continue;
        }
        if (flags & 6) {
          if (lane == 0) {
            atomicOr(p.err, ((flags & 2) ? ERR_ID_RANGE : 0) | ((flags & 4) ? ERR_HIDDEN_NONFINITE : 0));
            if (p.fired) p.fired[row] = 0;
          }
          continue;
        }
        // ---- softmax over the K ids (model.py:149-152), features (predictor.py:42-52)
        bool bad = (v0 && !is_finite(x0)) || (v1 && !is_finite(x1));
        bad = __any_sync(0xffffffffu, bad);
        float m = v0 ? x0 : -INFINITY;
        if (v1) m = fmaxf(m, x1);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float e0 = 0.f, e1 = 0.f;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {                          // one np_expf copy
          if (hh ? v1 : v0) {
            const float ev = np_expf(__fsub_rn(hh ? x1 : x0, m));
            if (hh) e1 = ev; else e0 = ev;
          }
        }
        float esum = 0.f;                                         // strict left-to-right
        for (int c = 0; c < K; ++c)
          esum = __fadd_rn(esum, __shfl_sync(0xffffffffu, c < 32 ? e0 : e1, c & 31));
        const float psum = np_pairwise_block(                     // numpy pairwise (predictor.py:49)
            0, K, [&](int c) { return __shfl_sync(0xffffffffu, c < 32 ? pv0 : pv1, c & 31); });
        if (p.logits_out) {
          if (v0) p.logits_out[(size_t)row * K + lane] = x0;
          if (v1) p.logits_out[(size_t)row * K + lane + 32] = x1;
        }
        int e = 0;
        if (bad) e |= ERR_LOGIT_NONFINITE;
        if (fabs((double)psum - 1.0) > 1e-5) e |= ERR_PREV_SUM;
        if (e) {
          if (lane == 0) {
            atomicOr(p.err, e);
            if (p.fired) p.fired[row] = 0;
          }
          continue;
        }
        if (v0) {
          const float pr = __fdiv_rn(e0, esum);
          feats[lane] = x0;
          feats[K + lane] = pr;
          feats[2 * K + lane] = __fsub_rn(pr, pv0);
        }
        if (v1) {
          const float pr = __fdiv_rn(e1, esum);
          feats[lane + 32] = x1;
          feats[K + lane + 32] = pr;
          feats[2 * K + lane + 32] = __fsub_rn(pr, pv1);
        }
      }
      __syncwarp();
      if (p.trace && lane == 0) p.trace[(size_t)row * 16 + 10] = clock64();
      float z2 = 0.f;
      if (mlp) {
        if (p.trace) {
          mlp_z1<4, !W1S>(feats, W1S ? w1s : p.w1, b1s, 3 * K, H, hs, lane, 0);
          __syncwarp();
          if (lane == 0) p.trace[(size_t)row * 16 + 11] = clock64();
          const float a0 = z2_partial(hs, w2s, H, lane), a1 = z2_partial(hs, w2s, H, lane + 32);
          if (lane == 0) p.trace[(size_t)row * 16 + 12] = clock64();
          z2 = z2_tree(a0, a1, hs, w2s, H, p.b2, lane);
          if (lane == 0) p.trace[(size_t)row * 16 + 13] = clock64();
        } else {
          z2 = W1S ? warp_mlp(feats, w1s, b1s, w2s, p.b2, K, H, hs, lane)
                   : warp_mlp_g(feats, p.w1, b1s, w2s, p.b2, K, H, hs, lane);
        }
      }
      float perr = 0.f;
      if (p.recheck &&
          !certify_row(p, row, feats, hs + (H > 0 ? H : 4), hs, W1S ? w1s : p.w1, b1s, w2s, z2,
                       __int_as_float(q_lnf), K, H, mlp, lane, perr, [&](int c) {
                         return __ldg(p.head_wmax + p.ids[(size_t)row * K + c]);
                       })) {
        if (lane == 0) defer_row(p, row, &s_defer);  // STRICT re-evaluation decides
        __syncwarp();
        continue;
      }
      for (int c = lane; c < K; c += 32) p.prev[(size_t)row * K + c] = feats[K + c];  // engine.py:196
      if (lane == 0 && p.prev_err) p.prev_err[row] = perr;
      if (p.feat_out)
        for (int i = lane; i < 3 * K; i += 32) p.feat_out[(size_t)row * 3 * K + i] = feats[i];
      if (lane == 0 && p.evals) p.evals[row] += 1;
      if (mlp) {
        if (lane == 0) {
          if (p.z_out) p.z_out[row] = z2;
          // the decision is exact (z2 >= z_cut); the reported probability is
          // the f32 sigmoid (|err| ~1e-7, tolerance 1e-3)
          if (p.prob_out) p.prob_out[row] = (double)sigmoid32(z2);
          write_fired(p, row, z2 >= p.z_cut);
        }
      } else if (lane == 0) {
        if (p.prob_out) p.prob_out[row] = p.const_prob;
        if (p.z_out) p.z_out[row] = 0.0f;
        write_fired(p, row, p.const_prob > p.threshold);
      }
      if (p.trace && lane == 0) {
        p.trace[(size_t)row * 16 + 4] = gtimer();
        p.trace[(size_t)row * 16 + 9] = clock64();
      }
    }
  } else {

  // =========================== DOT TEAMS ===========================
  const int team = warp / TEAM, w = warp % TEAM;
  uint8_t *tbase = smem + sp.off_team + (size_t)team * sp.team_bytes;
  float *red = reinterpret_cast<float *>(tbase);            // [(HALF+2) slots][4]
  int *tflag = reinterpret_cast<int *>(red + RED_FLOATS);   // [4]
  float *logit = red + RED_FLOATS + 4;                      // [MAXK]
  uint64_t *tbar = ringbar + team * RING;
  uint8_t *tring = smem + sp.off_ring + (size_t)team * RING * sp.unit_bytes;
  const bool leader = (w == 0 && lane == 0);
  auto row_of = [&](int kk) { return (int)blockIdx.x + kk * (int)gridDim.x; };

  // Warp 0 keeps the ids of the CURRENT row (cid*) and of the team's NEXT row
  // (nid*), lane c / c+32 holding id c / c+32, so the ring can be refilled
  // with the next row's LM-head rows while the current row is reduced.
  int cid0 = 0, cid1 = 0, nid0 = 0, nid1 = 0, cbad = 0, nbad = 0;
  bool cskip = true, nskip = true;
  auto load_ids = [&](int kk, int &i0, int &i1, int &bad, bool &skip) {
    skip = true; bad = 0; i0 = i1 = 0;
    if (kk >= rows_cta) return;
    const int row = row_of(kk);
    skip = row_skipped(p, row);
    if (skip) return;
    int b = 0;
    if (lane < K) {
      i0 = p.ids[(size_t)row * K + lane];
      if (i0 < 0 || i0 >= p.V) { b = 1; i0 = 0; }
    }
    if (lane + 32 < K) {
      i1 = p.ids[(size_t)row * K + lane + 32];
      if (i1 < 0 || i1 >= p.V) { b = 1; i1 = 0; }
    }
    bad = __any_sync(0xffffffffu, b) ? 1 : 0;
  };
  // Row data of the current row: hidden chunks of this warp's partial group
  // (registers, all warps); warp 0 lanes: prev[c], bw[id[c]].
  float4 xr[CPL];
  float pv0 = 0.f, pv1 = 0.f, bw0 = 0.f, bw1 = 0.f;
  auto load_row = [&](int kk) {
    if (kk >= rows_cta) return;
    const int row = row_of(kk);
    if (row_skipped(p, row)) return;
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
        bw0 = p.head_bw ? __ldg(p.head_bw + cid0) : 0.f;
      }
      if (lane + 32 < K) {
        pv1 = p.prev[(size_t)row * K + lane + 32];
        bw1 = p.head_bw ? __ldg(p.head_bw + cid1) : 0.f;
      }
    }
  };

  // ---- the team's TMA ring (warp 0 issues; all warps consume in order)
  uint32_t n_issue = 0, n_wait = 0;
  int ik = team, ih = 0;            // next unit to issue: (row index, half)
  int k = team;                     // current row index
  auto issue_unit = [&](int kk, int h, int i0, int i1) {
    const int c0 = h * HALF, nr = (K - c0) < HALF ? (K - c0) : HALF;
    int idv[HALF];
#pragma unroll
    for (int q = 0; q < HALF; ++q) {
      const int c = (c0 + q) < K ? (c0 + q) : 0;
      const int a = __shfl_sync(0xffffffffu, i0, c & 31), b = __shfl_sync(0xffffffffu, i1, c & 31);
      idv[q] = c < 32 ? a : b;
    }
    if (lane == 0) {
      const int slot = n_issue % RING;
      TW *dst = reinterpret_cast<TW *>(tring + (size_t)slot * sp.unit_bytes);
      fence_proxy_async();
      mbar_arrive_expect_tx(tbar + slot, (uint32_t)nr * wrow_bytes);
      for (int q = 0; q < nr; ++q)
        bulk_g2s(dst + (size_t)q * d, head + (size_t)idv[q] * d, wrow_bytes, tbar + slot);
      if (p.trace && h == 0) p.trace[(size_t)row_of(kk) * 16 + 5] = gtimer();
    }
    ++n_issue;
  };
  // keep RING units in flight, in (row, half) order over non-skipped rows
  auto pump = [&]() {
    while (n_issue < n_wait + RING && ik < rows_cta) {
      const bool cur = ik == k, nxt = ik == k + NTEAM;
      if (!cur && !nxt) return;                 // ids of that row not loaded yet
      if (cur ? cskip : nskip) { ik += NTEAM; ih = 0; continue; }
      issue_unit(ik, ih, cur ? cid0 : nid0, cur ? cid1 : nid1);
      if (++ih == nhalf) { ik += NTEAM; ih = 0; }
    }
  };
  // hand a row to its tail warp (warp 0 of the team)
  auto handoff = [&](int kk, int row, int flags, float cpv0, float cpv1, float lnf) {
    const int slot = kk % QS;
    if (lane == 0) mbar_wait(qempty + slot, ((kk / QS) & 1) ^ 1);
    __syncwarp();
    QSlot &q = queue[slot];
    if (lane == 0) { q.row = row; q.flags = flags; q.pad0 = __float_as_int(lnf); }
    if (lane < K) { q.logits[lane] = logit[lane]; q.prev[lane] = cpv0; }
    if (lane + 32 < K) { q.logits[lane + 32] = logit[lane + 32]; q.prev[lane + 32] = cpv1; }
    __syncwarp();
    if (lane == 0) mbar_arrive(qfull + slot);
  };

  if (w == 0) {
    load_ids(k, cid0, cid1, cbad, cskip);
    load_ids(k + NTEAM, nid0, nid1, nbad, nskip);
    pump();
  }
  if (early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  {  // every warp needs the skip status of its current row
    const int row = row_of(k);
    cskip = k >= rows_cta || row_skipped(p, row);
  }
  load_row(k);
  mbar_wait(setup_bar, 0);

  while (k < rows_cta) {
    const int row = row_of(k);
    if (cskip) {
      if (w == 0) handoff(k, row, 1, 0.f, 0.f, 0.f);
    } else {
      if (p.trace && leader) p.trace[(size_t)row * 16 + 1] = gtimer();
      // ---- pass 1: mean (this warp = canonical group w), from registers
      float part = 0.f;
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int c = 32 * w + lane + NPART * s;
        if (FULL || c < nchunk)
          part = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(part, xr[s].x), xr[s].y), xr[s].z), xr[s].w);
      }
      part = warp_butterfly_sum(part);
      if (lane == 0) red[HALF * 4 + w] = part;
      team_sync(team);
      const float total = canon_combine(red[HALF * 4 + 0], red[HALF * 4 + 1], red[HALF * 4 + 2],
                                        red[HALF * 4 + 3]);
      const float mean = __fdiv_rn(total, (float)d);
      bool hbad = false;
      if (!is_finite(total)) {            // rare: exact element scan (model.py:310-311)
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
      if (p.trace && leader) p.trace[(size_t)row * 16 + 2] = gtimer();
      float r = 0.f, lnf = 0.f;
      const float2 nmean = make_float2(-mean, -mean);
      for (int h = 0; h < nhalf; ++h) {
        const int slot = n_wait % RING;
        mbar_wait(tbar + slot, (n_wait / RING) & 1);
        if (p.trace && leader && h < 2) p.trace[(size_t)row * 16 + 6 + h] = gtimer();
        const TW *sw = reinterpret_cast<const TW *>(tring + (size_t)slot * sp.unit_bytes);
        const int c0 = h * HALF, nr = (K - c0) < HALF ? (K - c0) : HALF;
        float2 acc = make_float2(0.f, 0.f);
        float sq = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < CPL; ++s2) {
          const int c = 32 * w + lane + NPART * s2;
          if (FULL || c < nchunk) {
            const float4 xv = xr[s2];
            const float4 gv = *reinterpret_cast<const float4 *>(gs + CHUNK * c);
            const float2 xc01 = fadd2(make_float2(xv.x, xv.y), nmean);
            const float2 xc23 = fadd2(make_float2(xv.z, xv.w), nmean);
            if (h == 0)
              sq = __fmaf_rn(xc23.y, xc23.y, __fmaf_rn(xc23.x, xc23.x,
                             __fmaf_rn(xc01.y, xc01.y, __fmaf_rn(xc01.x, xc01.x, sq))));
            const float2 xg01 = fmul2(xc01, make_float2(gv.x, gv.y));
            const float2 xg23 = fmul2(xc23, make_float2(gv.z, gv.w));
            float wv[HALF][4];
#pragma unroll
            for (int q = 0; q < HALF; ++q) {
              Chunk<TW> ch;
              ch.lds(sw + (size_t)q * d + CHUNK * c);
              ch.to_f32(wv[q]);
            }
            const float xe[4] = {xg01.x, xg01.y, xg23.x, xg23.y};
#pragma unroll
            for (int e = 0; e < CHUNK; ++e)
              acc = ffma2(make_float2(xe[e], xe[e]), make_float2(wv[0][e], wv[1][e]), acc);
          }
        }
        const float a0 = warp_butterfly_sum(acc.x), a1 = warp_butterfly_sum(acc.y);
        if (h == 0) sq = warp_butterfly_sum(sq);
        if (lane == 0) {
          red[0 * 4 + w] = a0;
          red[1 * 4 + w] = a1;
          if (h == 0) red[(HALF + 1) * 4 + w] = sq;
        }
        team_sync(team);                       // all warps done with the slot; red written
        ++n_wait;
        if (w == 0) pump();                    // re-arm the freed slot
        if (h == 0) {
          const float var = __fdiv_rn(canon_combine(red[(HALF + 1) * 4 + 0], red[(HALF + 1) * 4 + 1],
                                                    red[(HALF + 1) * 4 + 2], red[(HALF + 1) * 4 + 3]),
                                      (float)d);
          r = __frcp_rn(__fsqrt_rn(__fadd_rn(var, 1e-5f)));
          lnf = sqrtf(1.f + mean * mean / var);
        }
        if (w == 0) {
          const float bwa = __shfl_sync(0xffffffffu, bw0, (c0 + lane) & 31);
          const float bwb = __shfl_sync(0xffffffffu, bw1, (c0 + lane) & 31);
          if (lane < nr) {
            const float dot = canon_combine(red[lane * 4 + 0], red[lane * 4 + 1], red[lane * 4 + 2],
                                            red[lane * 4 + 3]);
            logit[c0 + lane] = __fadd_rn(__fmul_rn(r, dot), (c0 + lane) < 32 ? bwa : bwb);
          }
        }
        if (h + 1 < nhalf) team_sync(team);    // red reused by the next half
      }
      if (p.trace && leader) p.trace[(size_t)row * 16 + 3] = gtimer();
      if (w == 0) {
        __syncwarp();
        handoff(k, row, (cbad ? 2 : 0) | (hbad ? 4 : 0), pv0, pv1, lnf);
      }
    }
    // ---- advance: next row becomes current; load its data; fetch the ids of
    // the row after it and keep the ring full
    k += NTEAM;
    if (w == 0) {
      cid0 = nid0; cid1 = nid1; cbad = nbad; cskip = nskip;
    }
    cskip = __shfl_sync(0xffffffffu, cskip ? 1 : 0, 0) != 0;   // warp 0 value (others below)
    if (w != 0) cskip = k >= rows_cta || row_skipped(p, row_of(k));
    load_row(k);
    if (w == 0) {
      load_ids(k + NTEAM, nid0, nid1, nbad, nskip);
      pump();
    }
  }
  }  // dot teams
  recheck_epilogue<TW>(p, smem, &s_defer, rows_cta,
                       [&](int kk) { return (int)blockIdx.x + kk * (int)gridDim.x; });
}

template <typename TW>
struct FastLaunch {
  const PredParams &p; const SmemPlan &sp; int grid; cudaStream_t stream; int smem_optin;
  template <int CPL> void operator()() const {
    const bool full = p.d == CHUNK * NPART * CPL;
    // the 3-deep ring only for the bf16 full-width kernels (LLM shapes); the
    // smem plan of a 3-ring also holds a 2-ring
    if constexpr (std::is_same<TW, __nv_bfloat16>::value) {
      if (sp.ring == 3 && full) { go<CPL, 3>(); return; }
    }
    go<CPL, 2>();
  }
  template <int CPL, int RG> void go() const {
    const bool full = p.d == CHUNK * NPART * CPL;
    if constexpr (RG == 3) {
      if (p.K == 4 && p.H == 512 && p.policy == SPX_POLICY_MLP) {
        if (sp.w1_smem) launch<CPL, true, true, 4, 512, 3>(); else launch<CPL, true, false, 4, 512, 3>();
      } else {
        if (sp.w1_smem) launch<CPL, true, true, 0, 0, 3>(); else launch<CPL, true, false, 0, 0, 3>();
      }
      return;
    }
    if (full && p.K == 4 && p.H == 512 && p.policy == SPX_POLICY_MLP) {
      if (sp.w1_smem) launch<CPL, true, true, 4, 512, RG>(); else launch<CPL, true, false, 4, 512, RG>();
      return;
    }
    if (sp.w1_smem) { if (full) launch<CPL, true, true, 0, 0, RG>(); else launch<CPL, false, true, 0, 0, RG>(); }
    else { if (full) launch<CPL, true, false, 0, 0, RG>(); else launch<CPL, false, false, 0, 0, RG>(); }
  }
  template <int CPL, bool FULL, bool W1S, int KC, int HC, int RG> void launch() const {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(predictor_fast_kernel<TW, CPL, FULL, W1S, KC, HC, RG>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
      configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FAST_THREADS);
    cfg.dynamicSmemBytes = sp.bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, predictor_fast_kernel<TW, CPL, FULL, W1S, KC, HC, RG>, p, sp);
  }
};
