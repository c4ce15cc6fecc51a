// Stage scheduler keyed on the rank profile and the
// super-core contraction of merged stages.  Pure host code: no CUDA calls, so
// the planner is testable without a GPU through qtt_plan_stages (include/qtt.h).
//
// PAPER.md Alg. 2 runs the levels k = 1..d strictly in order;
// each level reads the N*r_{k-1} intermediate and writes the N*r_k one.  A
// stage of L consecutive levels k0..k1 is applied here as ONE GEMM with the
// super-core
//   W[a][ii][jj][b] = sum_{bonds} G_k0[a,i_1,j_1,:] G_k0+1[:,i_2,j_2,:] ... G_k1[:,i_L,j_L,b]
//   ii = sum_l i_l 2^{l-1},  jj = sum_l j_l 2^{l-1}
// (the definition of the QTT matrix, Eq. TTdeccores P:519-523 with the
// operator pairing P:953-962, restricted to the stage's digits), so the
// intermediates inside the stage never exist.  Per element of N the GEMM does
// 2^(L+1) r_in r_out flops (a multiply-add counted as 2) against Alg. 2's
// 4 * sum_l r_{l-1} r_l: cheaper at the tapered ends of a rank
// profile (r_0 = r_d = 1), equal for L = 2 at constant rank, dearer for L >= 3
// at constant rank -- the planner weighs exactly that against the HBM bytes
// the merge removes.
#include "../../include/qtt.h"
#include "qtt_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <limits>
#include <vector>

namespace qtt {

namespace {

// Cost model of one B200 (148 SMs, 1965 MHz): DMMA 148*64 FMA/clk, HBM copy
// bandwidth as measured in MEASURED_PEAKS.json (~6.5 TB/s), launch ~3 us.
constexpr double kFp64 = 37.2e12 * 0.955;     // DMMA rate of the resident kernel with 12 consumer warps
constexpr double kHbm = 6.45e12 * 0.90;
// most warp tiles per SM a stage may have and still run on the small (L2-fed warp-tile) kernel
#ifndef QTT_SMALL_MAX_WT_PER_SM
#define QTT_SMALL_MAX_WT_PER_SM 24
#endif
#ifndef QTT_PLAN_KLAUNCH
#define QTT_PLAN_KLAUNCH 5.0e-6
#endif
constexpr double kLaunch = QTT_PLAN_KLAUNCH;   // per-launch cost in the stage DP (build knob for calibration)
// measured (profiles/, c3-c5 stages): 8 consumer warps (NB <= 8) reach ~0.84
// of nominal against 12 warps' ~0.955; a wide tile pays a fixed epilogue
// against its k-chunks, ~nch / (nch + 0.15) (c3's K = 64 stage [1-6]: 0.93,
// K = 128 pairs: 0.97 of the resident rate; 0.3 made the planner keep c3's
// r = 32 single level, 0.4% slower, profiles/r02zl_ab_c3*.json)
double fp64_rate(int NB, double nchunks) {
  const double warps = dmma_col_groups(NB) >= 3 ? 1.0 : 0.88;
  return kFp64 * warps * (nchunks / (nchunks + 0.15));
}
constexpr double kL2 = 7.0e12;                   // L2 -> SM bytes the wide kernel may pull
constexpr double kTileLatency = 1.5e-6;          // one tile: TMA round trip + epilogue
constexpr double kChunkLatency = 0.4e-6;         // one more k-chunk of a wide tile
constexpr double kSmBw = 100e9;                  // bytes/s one SM's TMA pulls when few SMs are busy
constexpr double kSms = 148;
constexpr double kSplitLatency = 2.5e-6;        // split-K: partial store, arrival atomics, S-way sum
constexpr double kSmallLatencyDefault = 2.0e-6; // small variant: operand round trips + epilogue of one warp tile
// calibration knob (diagnostic): QTT_PLAN_SMALL_LAT=<seconds>
double small_latency() {
  static const double v = [] {
    const char* e = std::getenv("QTT_PLAN_SMALL_LAT");
    return e ? std::atof(e) : kSmallLatencyDefault;
  }();
  return v;
}
constexpr double kSmallStep = 0.05e-6;          // small variant: one k-step of 8 (16 dependent MMAs + loads)
constexpr size_t kTwoCtaSmem = 113 * 1024;      // two resident-kernel CTAs per SM

uint32_t round_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// Fraction of the SM-waves a stage keeps busy: its tiles fill ceil(tiles / slots)
// waves of `slots` CTAs (the last one partly), e.g. 256 tiles on 148 SMs -> 86%.
double wave_efficiency(double tiles, double slots) {
  return tiles / (std::ceil(tiles / slots) * slots);
}

}  // namespace

bool split_enabled() {
  static const bool on = std::getenv("QTT_NO_SPLIT") == nullptr;
  return on;
}

int wide_ksplit(int64_t tiles, int nchunks, int sms) {
  if (tiles <= 0 || nchunks < 4 || !split_enabled()) return 1;
  // small stages are latency-bound: the partial round trip costs more than the
  // idle SMs (c1, c2: 20 -> 23 us, 35 -> 45 us split); split from ~28 chunk-times per SM
  if (double(tiles) * nchunks < 28.0 * sms) return 1;
  // time in k-chunk units: waves x (chunks per tile + epilogue); a split tile's
  // epilogue also stores its partial and (last arrival) sums S of them
  auto cost = [&](int S) {
    const int cps = (nchunks + S - 1) / S;
    const double waves = std::ceil(double(tiles) * S / sms);
    return waves * (cps + (S > 1 ? 1.0 : 0.3));
  };
  int best = 1;
  double bc = cost(1);
  for (int S = 2; S <= 64 && (nchunks + S - 1) / S >= 2; ++S) {
    const double c = cost(S);
    if (c < 0.95 * bc) {   // only for a clear win
      bc = c;
      best = S;
    }
  }
  const int cps = (nchunks + best - 1) / best;
  return (nchunks + cps - 1) / cps;   // no empty split
}

size_t dmma_smem_bytes(int KB, int NB, int K, int rep, int stages) {
  const size_t stage = round_up(uint32_t(kDmmaRowsPerSubtile * rep) * uint32_t(K) * 8u, 128u);
  return kBarBytes + size_t(KB) * NB * 32 * 32 + stage * stages;
}

bool dmma_tiling(int K, int KB, int NB, size_t smem_optin, int* rep_out, int* stages_out, size_t* smem_out) {
  if (!dmma_instantiated(KB, NB)) return false;

  // TMA stage: >= 16 KiB per stage (HBM bytes in flight), <= 64 KiB.
  const size_t sub_bytes = size_t(kDmmaRowsPerSubtile) * K * 8;
  int rep = int(std::max<size_t>(1, (16384 + sub_bytes - 1) / sub_bytes));
  while (rep > 1 && sub_bytes * rep > 65536) --rep;
  for (int stages = kMaxStages; stages >= 2; --stages) {
    const size_t smem = dmma_smem_bytes(KB, NB, K, rep, stages);
    if (smem <= smem_optin) {
      *rep_out = rep;
      *stages_out = stages;
      *smem_out = smem;
      return true;
    }
  }
  return false;
}

// Shape and estimated time of a stage k0..k1 (1-based), or false if no kernel
// instance covers it.  Estimates are at N = n, nrhs = 1.
static bool stage_shape(const int64_t* ranks, int k0, int k1, int64_t n, size_t smem_optin, StagePlan* sp) {
  const int L = k1 - k0 + 1;
  const int n_i = 1 << L;
  const int r_in = int(ranks[k0 - 1]), r_out = int(ranks[k1]);
  sp->k0 = k0;
  sp->k1 = k1;
  sp->r_in = r_in;
  sp->r_out = r_out;
  sp->n_i = n_i;
  sp->K = n_i * r_in;
  sp->RP = (r_out + 1) / 2 * 2;
  sp->KB = (sp->K + 15) / 16;
  sp->NB = (n_i * sp->RP + 7) / 8;
  const double M = double(n) / n_i;
  const double bytes = 8.0 * double(n) * (r_in + r_out);
  bool ok = false;
  if (dmma_tiling(sp->K, sp->KB, sp->NB, smem_optin, &sp->rep, &sp->stages, &sp->smem)) {
    sp->variant = L == 1 ? kDmma : kMerged;
    const double tiles = std::ceil(M / (kDmmaRowsPerSubtile * sp->rep));
    // padded tensor-pipe work: whole tiles of 64 * rep rows, K and N to fragment blocks
    const double flops = 2.0 * tiles * kDmmaRowsPerSubtile * sp->rep * 16.0 * sp->KB * 8.0 * sp->NB;
    const double u = wave_efficiency(tiles, kSms);                   // busy fraction of the SM-waves
    // latency floor of tiny problems: each CTA's tiles run one after another,
    // each at least one TMA round trip
    const double tile_bytes = kDmmaRowsPerSubtile * sp->rep * 8.0 * sp->K;
    const double lat = std::ceil(tiles / kSms) * (kTileLatency + tile_bytes / kSmBw) + sp->KB * sp->NB * 1024.0 / kSmBw;
    sp->est_seconds = std::max({flops / (fp64_rate(sp->NB, 1e9) * u), bytes / (kHbm * u), lat}) + kLaunch;
    ok = true;
    // Near the ridge (HBM time >= 0.85 x FP64 time) two CTAs per SM with a
    // shallower ring keep more bytes in flight than one CTA with a deep one
    // (c5's single r = 24 level: 11.5 -> 9.2 ms); compute-bound levels keep
    // one CTA and the deepest ring (c3's r = 32 levels lose 3% with two).
    if (bytes / kHbm >= 0.85 * flops / kFp64) {
      int rep2 = 0, st2 = 0;
      size_t sm2 = 0;
      if (dmma_tiling(sp->K, sp->KB, sp->NB, kTwoCtaSmem, &rep2, &st2, &sm2) && st2 >= 2) {
        sp->rep = rep2;
        sp->stages = st2;
        sp->smem = sm2;
      }
    }
  }
  // Wide variant: super-core streamed from L2 in k-chunks (qtt_wide_kernel.cu).
  const int nout = n_i * r_out;
  const double wbytes = 8.0 * sp->K * nout;
  // (K need not be a multiple of the k-chunk: the TMA unit zero-fills the A
  // columns past K and the packed W rows past K are zero.)
  if (wbytes <= double(kWideMaxCoreBytes)) {
    // widest column block that the output needs (NB = 16 runs 16 consumer warps;
    // it beats 96-column blocks of whole ii blocks too: c4 levels 1-7 5.96 vs 6.04 ms)
    // For nout > 96 also try 96-column blocks: less padding when nout mod 128 is
    // small or just below 96 (r = 95: 2 x 96 = 192 computed columns instead of 256).
    const int NBfit = nout <= 32 ? 4 : nout <= 64 ? 8 : nout <= 96 ? 12 : 16;
    const int NBdef = NBfit < QTT_WIDE_NB_CAP ? NBfit : QTT_WIDE_NB_CAP;
    const bool try96 = QTT_WIDE_NB_CAP >= 12 && nout > 96 && (nout + 95) / 96 * 96 < (nout + 127) / 128 * 128;
    for (const int NBw : {NBdef, try96 ? 12 : 0}) {
    if (NBw == 0) continue;
    const size_t smem = wide_smem_bytes(NBw);
    if (smem <= smem_optin) {
      const int ncb = (nout + 8 * NBw - 1) / (8 * NBw);
      const double tiles_out = std::ceil(M / kDmmaRowsPerSubtile) * ncb;
      const double nch_all = std::ceil(sp->K / double(kWideBK));
      // split-K when the output tiles alone leave SMs idle (small M, huge K)
      const int S = wide_ksplit(int64_t(tiles_out), int(nch_all), int(kSms));
      const double nch = std::ceil(nch_all / S);                  // k-chunks per tile
      const double tiles = tiles_out * S;
      const double flops = 2.0 * tiles_out * kDmmaRowsPerSubtile * nch_all * kWideBK * 8.0 * NBw;
      const double u = wave_efficiency(tiles, kSms);
      const double l2 = tiles_out * (kDmmaRowsPerSubtile * 8.0 * sp->K + 8.0 * sp->K * 8.0 * NBw) +
                        (S > 1 ? 2.0 * tiles * kDmmaRowsPerSubtile * 8.0 * NBw * 8.0 : 0.0);
      // a wide tile streams its k-chunks one after another
      const double tile_bytes = nch * kWideBK * 8.0 * (kDmmaRowsPerSubtile + 8.0 * NBw);
      const double lat = std::ceil(tiles / kSms) * (kTileLatency + nch * kChunkLatency + tile_bytes / kSmBw) +
                         (S > 1 ? kSplitLatency : 0.0);
      const double rate = S > 1 ? fp64_rate(NBw, 1e9) * nch / (nch + 1.0) : fp64_rate(NBw, nch);
      const double t = std::max({flops / (rate * u), (bytes + wbytes) / (kHbm * u), l2 / kL2, lat}) + kLaunch;
      if (!ok || t < sp->est_seconds) {
        sp->variant = kWide;
        sp->NB = NBw;
        sp->KB = kWideKBC;
        sp->RP = r_out;
        sp->ncb = ncb;
        sp->nchunks = (sp->K + kWideBK - 1) / kWideBK;
        sp->ksplit = S;
        sp->rep = 1;
        sp->stages = kWideStages;
        sp->smem = smem;
        sp->est_seconds = t;
        ok = true;
      }
    }
    }
  }
  // Small variant: one warp per 16 x 32 output block straight from L2, for
  // stages too small to fill the GPU with 64-row TMA tiles (latency-bound).
  static const bool no_small = std::getenv("QTT_PLAN_NO_SMALL") != nullptr;   // diagnostic
  if (!no_small && wbytes <= double(kWideMaxCoreBytes) && sp->K % 2 == 0) {
    const int ncb = (nout + kSmallCols - 1) / kSmallCols;
    const double wt = std::ceil(M / kSmallRows) * ncb;        // warp tiles
    if (wt <= kSms * QTT_SMALL_MAX_WT_PER_SM) {
      const double nq = std::ceil(sp->K / double(kSmallK));
      const double flops = 2.0 * wt * kSmallRows * kSmallCols * nq * kSmallK;
      const double blocks = std::ceil(wt / kSmallWarps);
      const double sm_used = std::min(1.0, blocks / kSms);
      const double warps_per_sm = wt / std::min(blocks, kSms);
      const double rate = kFp64 * sm_used * std::min(1.0, warps_per_sm / 12.0) * 0.8;
      const double lat = small_latency() + nq * kSmallStep * std::max(1.0, warps_per_sm / 12.0);
      static const bool force = std::getenv("QTT_PLAN_FORCE_SMALL") != nullptr;   // diagnostic
      const double t = std::max({flops / rate, (bytes + wbytes) / kHbm, lat}) + kLaunch;
      if (!ok || t < sp->est_seconds || force) {
        sp->variant = kSmall;
        sp->NB = 4;
        sp->KB = 0;
        sp->RP = r_out;
        sp->ncb = ncb;
        sp->nchunks = int(nq);
        sp->ksplit = 1;
        sp->rep = 1;
        sp->stages = 0;
        sp->smem = 0;
        sp->est_seconds = t;
        ok = true;
      }
    }
  }
  if (ok) return true;
  if (L != 1) return false;
  sp->variant = kGeneric;   // any rank, one thread per output element
  const double flops = 4.0 * double(r_in) * r_out * double(n);
  sp->est_seconds = std::max(flops / (kFp64 * 0.05), bytes / (kHbm * 0.5)) + kLaunch;
  return true;
}

// Dynamic programme over the level sequence: best[k] = min over the last
// stage [k0, k] of best[k0-1] + est(k0..k).  The estimate scales with N; for
// the plan only the relative cost of flops, bytes and launches matters, and
// the launch term is what keeps small-N problems (c1, c2) from being cut
// into many launches, so N is the real N.
// A stage of diagonal levels k0..k1: out[(m, ii)][b] = sum_a in[(m, ii)][a] D[ii][a][b]
// streams the input once (HBM-bound batched GEMV on CUDA cores).
static bool diag_shape(const int64_t* ranks, int k0, int k1, int64_t n, StagePlan* sp) {
  const int L = k1 - k0 + 1;
  const int64_t r_in = ranks[k0 - 1], r_out = ranks[k1];
  if (r_out > kDiagMaxRank || r_in > kDiagMaxRank ||
      double(r_in) * std::ldexp(1.0, L) * double(r_out) > double(kDiagMaxCoreDoubles))
    return false;
  *sp = StagePlan{};
  sp->k0 = k0;
  sp->k1 = k1;
  sp->variant = kDiag;
  sp->r_in = int(r_in);
  sp->r_out = int(r_out);
  sp->n_i = 1 << L;
  sp->K = sp->n_i * sp->r_in;
  sp->RP = sp->r_out;
  const double bytes = 8.0 * double(n) * double(r_in + r_out) + 8.0 * r_in * std::ldexp(1.0, L) * r_out;
  const double flops = 2.0 * double(n) * double(r_in) * double(r_out);
  sp->est_seconds = std::max(bytes / (kHbm * 0.7), flops / (kFp64 * 0.25)) + kLaunch;
  return true;
}

// Diagnostic (A/B of stage splits): QTT_PLAN_FORCE_STAGES="1-7,8-9,...,18-24"
// ("k" alone = the one-level stage k-k)
// forces the partition of levels 1..d into stages (each gets its cheapest
// kernel instance); ignored unless it covers exactly 1..d with coverable stages.
static bool forced_stages(int d, const int64_t* ranks, size_t smem_optin, int64_t n, std::vector<StagePlan>* out) {
  static const char* spec = std::getenv("QTT_PLAN_FORCE_STAGES");
  if (!spec) return false;
  std::vector<StagePlan> p;
  int next = 1;
  const char* c = spec;
  while (*c) {
    char* e = nullptr;
    const long a = std::strtol(c, &e, 10);
    if (e == c) return false;
    long b = a;                    // "k" alone is the one-level stage k-k
    if (*e == '-') {
      c = e + 1;
      b = std::strtol(c, &e, 10);
      if (e == c) return false;
    }
    if (a != next || b < a || b > d || b - a + 1 > kMaxStageLevels) return false;
    StagePlan sp;
    if (!stage_shape(ranks, int(a), int(b), n, smem_optin, &sp)) return false;
    p.push_back(sp);
    next = int(b) + 1;
    c = e;
    if (*c == ',') ++c;
  }
  if (next != d + 1) return false;
  *out = p;
  return true;
}

std::vector<StagePlan> plan_stages(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                   const unsigned char* diag, int64_t rows) {
  const int64_t n = rows > 0 ? rows : int64_t(1) << d;
  {
    std::vector<StagePlan> forced;
    if (forced_stages(d, ranks, smem_optin, n, &forced)) return forced;
  }
  const int maxL = std::max(1, std::min(max_stage_levels, kMaxStageLevels));
  // diagonal stages cost the same whatever L: allow long ones unless the caller capped L
  const int maxLd = max_stage_levels >= kMaxStageLevels ? kDiagMaxLevels : maxL;
  std::vector<double> best(d + 1, std::numeric_limits<double>::infinity());
  std::vector<StagePlan> choice(d + 1);
  best[0] = 0;
  for (int k = 1; k <= d; ++k) {
    for (int L = 1; L <= std::min(maxL, k); ++L) {
      StagePlan sp;
      if (!stage_shape(ranks, k - L + 1, k, n, smem_optin, &sp)) continue;
      const double c = best[k - L] + sp.est_seconds;
      if (c < best[k]) {
        best[k] = c;
        choice[k] = sp;
      }
    }
    if (!diag) continue;
    for (int L = 1; L <= std::min(maxLd, k) && diag[k - L]; ++L) {
      StagePlan sp;
      if (!diag_shape(ranks, k - L + 1, k, n, &sp)) continue;
      const double c = best[k - L] + sp.est_seconds;
      if (c < best[k]) {
        best[k] = c;
        choice[k] = sp;
      }
    }
  }
  std::vector<StagePlan> out;
  for (int k = d; k > 0; k = choice[k].k0 - 1) out.push_back(choice[k]);
  std::reverse(out.begin(), out.end());
  return out;
}

// ---- fused apply (variant kFused): the whole apply as ONE persistent launch.
// Every stage is a small-variant stage (16 x 32 warp tiles from L2) run by all
// warps of the grid, stages separated by grid barriers (fused_small_kernel).
// Cost of a stage: its warp tiles spread over the SM sub-partitions, each tile
// a chain of nq k-steps of 16 DMMA.8x8x4 (16 clk each on one sub-partition's
// FP64 tensor pipe: 0.13 us per step at 1.965 GHz), plus one L2 round trip
// and the barrier.  Calibrated on the box; QTT_FUSED_STEP /
// _LAT / _BAR / _LAUNCH override the constants (diagnostics).
namespace {
double env_or(const char* name, double v) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : v;
}
}  // namespace

double fused_stage_seconds(const int64_t* ranks, int k0, int k1, double rows, StagePlan* sp) {
  // calibrated on c1 / c2 (round 2, QTT_FUSED_PROFILE): a k-step of a warp
  // tile with two warps per sub-partition ~0.16 us; per stage ~2 us of
  // operand latency + epilogue, ~1 us more for the split-K reduction, ~1.5 us
  // for the grid barrier (store drain, release, polling)
  static const double kStep = env_or("QTT_FUSED_STEP", 0.16e-6);
  static const double kLat = env_or("QTT_FUSED_LAT", 2.0e-6);
  static const double kRed = env_or("QTT_FUSED_RED", 1.0e-6);
  static const double kBar = env_or("QTT_FUSED_BAR", 1.5e-6);
  const int L = k1 - k0 + 1;
  const int n_i = 1 << L;
  const int r_in = int(ranks[k0 - 1]), r_out = int(ranks[k1]);
  const int K = n_i * r_in, nout = n_i * r_out;
  if (double(K) * nout * 8.0 > double(kFusedMaxCoreBytes)) return -1.0;
  if (size_t((K + kSmallK - 1) / kSmallK) * 128 * 16 > kFusedMaxBBytes) return -1.0;   // the smem block
  *sp = StagePlan{};
  sp->k0 = k0;
  sp->k1 = k1;
  sp->variant = kFused;
  sp->r_in = r_in;
  sp->r_out = r_out;
  sp->n_i = n_i;
  sp->K = K;
  sp->RP = r_out;
  sp->NB = 4;
  sp->ncb = (nout + kSmallCols - 1) / kSmallCols;
  sp->nchunks = (K + kSmallK - 1) / kSmallK;
  const double tiles = std::ceil(rows / n_i / kSmallRows) * sp->ncb;
  // warps per tile: split the k-steps over up to all warps of a CTA while the
  // grid's warps outnumber the tiles (fixed here, at plan time, for every nrhs)
  const double warps = kSms * kFusedWarps;
  int ks = 1;
  while (ks * 2 <= kFusedWarps && ks * 2 <= sp->nchunks && tiles * ks * 2 <= warps) ks *= 2;
  sp->ksplit = ks;
  const double per_smsp = std::ceil(tiles * ks / (kSms * 4));   // warp tiles one sub-partition runs
  const double steps = std::ceil(double(sp->nchunks) / ks);
  // + a tenth of the stage's executed flops at the FP64 peak: breaks the
  // model's ties toward the cheaper super-cores (c1: [1-7] [8-12], 10.5
  // MFLOP, measured 7.5 us against 7.8 us for [1-8] [9-12], 18.9 MFLOP)
  const double flops = 2.0 * (rows / n_i) * double(K) * double(nout);
  sp->est_seconds = per_smsp * steps * kStep + kLat + (ks > 1 ? kRed : 0.0) + kBar + 0.1 * flops / kFp64;
  return sp->est_seconds;
}

double fused_launch_seconds() {
  static const double v = env_or("QTT_FUSED_LAUNCH", 3.0e-6);   // cooperative launch
  return v;
}

// Diagnostic (A/B): QTT_FUSED_FORCE_STAGES="1-7,8-10,11-15" forces the fused
// plan's split (ignored unless it covers 1..d with stages a fused launch can run).
static bool forced_fused(int d, const int64_t* ranks, int64_t rows, std::vector<StagePlan>* out, double* est) {
  static const char* spec = std::getenv("QTT_FUSED_FORCE_STAGES");
  if (!spec) return false;
  std::vector<StagePlan> p;
  double t = fused_launch_seconds();
  int next = 1;
  const char* c = spec;
  while (*c) {
    char* e = nullptr;
    const long a = std::strtol(c, &e, 10);
    if (e == c) return false;
    long b = a;
    if (*e == '-') {
      c = e + 1;
      b = std::strtol(c, &e, 10);
      if (e == c) return false;
    }
    if (a != next || b < a || b > d || int(p.size()) >= kFusedMaxStages) return false;
    StagePlan sp;
    const double ts = fused_stage_seconds(ranks, int(a), int(b), double(rows), &sp);
    if (ts < 0) return false;
    t += ts;
    p.push_back(sp);
    next = int(b) + 1;
    c = e;
    if (*c == ',') ++c;
  }
  if (next != d + 1) return false;
  *out = p;
  if (est) *est = t;
  return true;
}

std::vector<StagePlan> plan_stages_fused(int d, const int64_t* ranks, int max_stage_levels, int64_t rows,
                                         double* est) {
  {
    std::vector<StagePlan> forced;
    if (forced_fused(d, ranks, rows, &forced, est)) return forced;
  }
  const double kLaunchF = fused_launch_seconds();
  const int maxL = std::max(1, std::min(max_stage_levels, kMaxStageLevels));
  std::vector<double> best(d + 1, std::numeric_limits<double>::infinity());
  std::vector<int> cnt(d + 1, 0);
  std::vector<StagePlan> choice(d + 1);
  best[0] = 0;
  for (int k = 1; k <= d; ++k)
    for (int L = 1; L <= std::min(maxL, k); ++L) {
      StagePlan sp;
      const double t = fused_stage_seconds(ranks, k - L + 1, k, double(rows), &sp);
      if (t < 0 || cnt[k - L] + 1 > kFusedMaxStages) continue;
      if (best[k - L] + t < best[k]) {
        best[k] = best[k - L] + t;
        cnt[k] = cnt[k - L] + 1;
        choice[k] = sp;
      }
    }
  std::vector<StagePlan> out;
  if (!std::isfinite(best[d])) {
    if (est) *est = std::numeric_limits<double>::infinity();
    return out;
  }
  for (int k = d; k > 0; k = choice[k].k0 - 1) out.push_back(choice[k]);
  std::reverse(out.begin(), out.end());
  if (est) *est = best[d] + kLaunchF;
  return out;
}

double plan_seconds(const std::vector<StagePlan>& p) {
  double t = 0;
  for (const auto& sp : p) t += sp.est_seconds;
  return t;
}

// Projection stage of a shard (top-bit sharding): T[m][alpha]
// (n rows, K = r) times Wp[alpha][h] (P = 2^s columns), out row m + n (s' (P-1) + h).
bool projection_plan_wide(int r, int s, size_t smem_optin, StagePlan* sp) {
  const int P = 1 << s;
  if (r % 2) return false;                      // TMA tensor map row stride must be 16-byte aligned
  sp->k0 = sp->k1 = 0;
  sp->r_in = r;
  sp->r_out = 1;
  sp->n_i = P;
  sp->K = r;
  sp->variant = kWide;
  sp->RP = 1;
  sp->NB = P <= 32 ? 4 : P <= 64 ? 8 : P <= 96 ? 12 : 16;
  sp->KB = kWideKBC;
  sp->ncb = (P + 8 * sp->NB - 1) / (8 * sp->NB);
  sp->nchunks = (r + kWideBK - 1) / kWideBK;
  sp->rep = 1;
  sp->stages = kWideStages;
  sp->smem = wide_smem_bytes(sp->NB);
  return sp->smem <= smem_optin;
}

bool projection_plan(int r, int s, size_t smem_optin, StagePlan* sp) {
  const int P = 1 << s;
  sp->k0 = sp->k1 = 0;
  sp->r_in = r;
  sp->r_out = 1;
  sp->n_i = P;
  sp->K = r;
  sp->KB = (r + 15) / 16;
  sp->RP = 2;
  sp->NB = (2 * P + 7) / 8;
  if (dmma_tiling(sp->K, sp->KB, sp->NB, smem_optin, &sp->rep, &sp->stages, &sp->smem)) {
    sp->variant = kMerged;
    return true;
  }
  if (r % 2) return false;                      // TMA tensor map row stride must be 16-byte aligned
  sp->variant = kWide;
  sp->RP = 1;
  sp->NB = P <= 32 ? 4 : P <= 64 ? 8 : P <= 96 ? 12 : 16;
  sp->KB = kWideKBC;
  sp->ncb = (P + 8 * sp->NB - 1) / (8 * sp->NB);
  sp->nchunks = (r + kWideBK - 1) / kWideBK;
  sp->rep = 1;
  sp->stages = kWideStages;
  sp->smem = wide_smem_bytes(sp->NB);
  return sp->smem <= smem_optin;
}

}  // namespace qtt

extern "C" qtt_status_t qtt_plan_stages_split(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                              int* n_stages, int* k_first, int* k_last, int* variant, int* ksplit);

extern "C" qtt_status_t qtt_plan_stages(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                        int* n_stages, int* k_first, int* k_last, int* variant) {
  return qtt_plan_stages_split(d, ranks, smem_optin, max_stage_levels, n_stages, k_first, k_last, variant, nullptr);
}

extern "C" qtt_status_t qtt_plan_stages_split(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                              int* n_stages, int* k_first, int* k_last, int* variant, int* ksplit) {
  if (d < 1 || d > 30 || !ranks || !n_stages || max_stage_levels < 1) return QTT_ERROR_INVALID_VALUE;
  if (ranks[0] != 1 || ranks[d] != 1) return QTT_ERROR_INVALID_VALUE;
  for (int k = 0; k <= d; ++k)
    if (ranks[k] < 1 || ranks[k] > 4096) return QTT_ERROR_INVALID_VALUE;
  if (smem_optin == 0) smem_optin = 232448;   // B200 cudaDevAttrMaxSharedMemoryPerBlockOptin
  try {
    const std::vector<qtt::StagePlan> p = qtt::plan_stages(d, ranks, smem_optin, max_stage_levels);
    *n_stages = int(p.size());
    for (size_t s = 0; s < p.size(); ++s) {
      if (k_first) k_first[s] = p[s].k0;
      if (k_last) k_last[s] = p[s].k1;
      if (variant) variant[s] = p[s].variant;
      if (ksplit) ksplit[s] = p[s].variant == qtt::kWide ? p[s].ksplit : 1;
    }
  } catch (...) {
    return QTT_ERROR_OUT_OF_MEMORY;
  }
  return QTT_SUCCESS;
}
