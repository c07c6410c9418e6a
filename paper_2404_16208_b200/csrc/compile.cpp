// compile.cpp -- validation and network compiler (host side of
// ranc_load_network).
//
// Validation follows SPEC load_network ("fully validated in-memory
// tables; any violation reported with record coordinates") with the ranges
// of include/ranc.h.  The compiler lays the network out for the popcount
// tick kernel:
//   * per-core axon type-sort: axons are renumbered a' so that each axon type
//     occupies a contiguous range.  Integration (Alg. 1 l.12-13) is
//     then sum_k w[n][k] * popcount(column & spikes & segment_k), evaluated
//     over "pieces" = (32-axon word, type present in it): at most
//     ceil(A/32) + K - 1 pieces per neuron instead of K*ceil(A/32).
//     Relabeling axons does not change the result (pinned, P9).
//   * route words with the destination core and the PERMUTED destination axon,
//     so the router writes straight into the destination's sorted ring row
//     ("a spike bit is written directly into the scheduler SRAM array").
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "internal.h"

namespace ranc {

namespace {

std::string core_str(const ranc_network_desc* d, int c) {
  char b[64];
  snprintf(b, sizeof b, "core (%d,%d)", c % d->grid_w, c / d->grid_w);
  return b;
}

bool fits(int64_t v, int bits) {
  int64_t hi = (int64_t(1) << (bits - 1)) - 1, lo = -(int64_t(1) << (bits - 1));
  return v >= lo && v <= hi;
}

// canonical K-major core-matrix layout of a tensor-core operand with R rows (tc.h)
inline uint32_t tc_operand_offset(uint32_t r, uint32_t k, uint32_t R) {
  return (k >> 4) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15);
}

ranc_status fail(std::string* err, ranc_status s, const std::string& m) {
  *err = m;
  return s;
}

}  // namespace

ranc_status validate_and_compile(const ranc_network_desc* d, Compiled* out, std::string* err) {
  char b[256];
  if (!d) return fail(err, RANC_E_ARG, "network descriptor is NULL");
  if (d->abi_version != RANC_ABI_VERSION) {
    snprintf(b, sizeof b, "abi_version=%d, library expects %d", d->abi_version, RANC_ABI_VERSION);
    return fail(err, RANC_E_CONFIG, b);
  }
  if (d->grid_w < 1 || d->grid_h < 1 || (int64_t)d->grid_w * d->grid_h > 65536) {
    snprintf(b, sizeof b, "grid %dx%d: need grid_w, grid_h >= 1 and G <= 65536", d->grid_w, d->grid_h);
    return fail(err, RANC_E_CONFIG, b);
  }
  if (d->axons < 1 || d->axons > 1024 || d->neurons < 1 || d->neurons > 1024) {
    snprintf(b, sizeof b, "axons=%d neurons=%d: each must be in [1,1024]", d->axons, d->neurons);
    return fail(err, RANC_E_CONFIG, b);
  }
  if (d->num_types < 1 || d->num_types > 4) {
    snprintf(b, sizeof b, "num_types=%d: must be in [1,4]", d->num_types);
    return fail(err, RANC_E_CONFIG, b);
  }
  if (d->max_delay < 1 || d->max_delay > 15) {
    snprintf(b, sizeof b, "max_delay=%d: must be in [1,15]", d->max_delay);
    return fail(err, RANC_E_CONFIG, b);
  }
  if (d->num_classes < 0 || d->num_lines < 0 || d->num_classes > 65536) {
    snprintf(b, sizeof b, "num_classes=%d num_lines=%d: must be >= 0", d->num_classes, d->num_lines);
    return fail(err, RANC_E_CONFIG, b);
  }
  const int bits[5] = {d->potential_bits, d->weight_bits, d->leak_bits, d->threshold_bits, d->reset_bits};
  const char* bname[5] = {"potential_bits", "weight_bits", "leak_bits", "threshold_bits", "reset_bits"};
  for (int i = 0; i < 5; ++i)
    if (bits[i] < 2 || bits[i] > 16) {
      snprintf(b, sizeof b, "%s=%d: supported range is [2,16] (int16 storage)", bname[i], bits[i]);
      return fail(err, RANC_E_CONFIG, b);
    }
  if (!d->axon_type || !d->input_line || !d->crossbar || !d->weight || !d->leak || !d->pos_threshold ||
      !d->neg_threshold || !d->reset_potential || !d->initial_potential || !d->reset_mode ||
      !d->dest_kind || !d->dest_dx || !d->dest_dy || !d->dest_axon || !d->dest_delay || !d->out_class)
    return fail(err, RANC_E_ARG, "a network array pointer is NULL");

  const int G = d->grid_w * d->grid_h, A = d->axons, N = d->neurons, K = d->num_types;
  const int D = d->max_delay, C = d->num_classes, I = d->num_lines;
  const int W = (A + 31) / 32;
  // G3: int32 accumulator bound  A*2^(wb-1) + 2^(pb-1) + 2^(lb-1) + 2^(tb-1) + 2^(rb-1) < 2^31
  {
    int64_t bound = (int64_t)A * (int64_t(1) << (d->weight_bits - 1)) + (int64_t(1) << (d->potential_bits - 1)) +
                    (int64_t(1) << (d->leak_bits - 1)) + (int64_t(1) << (d->threshold_bits - 1)) +
                    (int64_t(1) << (d->reset_bits - 1));
    if (bound >= (int64_t(1) << 31)) return fail(err, RANC_E_BOUND, "int32 accumulator could overflow");
  }

  for (int c = 0; c < G; ++c) {
    for (int a = 0; a < A; ++a) {
      int ty = d->axon_type[(size_t)c * A + a];
      if (ty >= K) {
        snprintf(b, sizeof b, "%s axon %d: axon_type=%d >= num_types=%d", core_str(d, c).c_str(), a, ty, K);
        return fail(err, RANC_E_RANGE, b);
      }
      int32_t ln = d->input_line[(size_t)c * A + a];
      if (ln < -1 || ln >= I) {
        snprintf(b, sizeof b, "%s axon %d: input_line=%d not in [-1,%d)", core_str(d, c).c_str(), a, ln, I);
        return fail(err, RANC_E_RANGE, b);
      }
    }
    for (int n = 0; n < N; ++n) {
      size_t cn = (size_t)c * N + n;
      std::string where = core_str(d, c) + " neuron " + std::to_string(n);
      if (A % 32) {
        uint32_t pad = d->crossbar[cn * W + W - 1] >> (A % 32);
        if (pad) return fail(err, RANC_E_RANGE, where + ": crossbar bits beyond axons are set");
      }
      for (int k = 0; k < K; ++k) {
        int v = d->weight[cn * K + k];
        if (!fits(v, d->weight_bits)) {
          snprintf(b, sizeof b, "%s: weight[%d]=%d exceeds weight_bits=%d", where.c_str(), k, v, d->weight_bits);
          return fail(err, RANC_E_BITWIDTH, b);
        }
      }
      struct { const char* nm; int v; int bits; } chk[5] = {
          {"leak", d->leak[cn], d->leak_bits},
          {"pos_threshold", d->pos_threshold[cn], d->threshold_bits},
          {"neg_threshold", d->neg_threshold[cn], d->threshold_bits},
          {"reset_potential", d->reset_potential[cn], d->reset_bits},
          {"initial_potential", d->initial_potential[cn], d->potential_bits}};
      for (auto& q : chk)
        if (!fits(q.v, q.bits)) {
          snprintf(b, sizeof b, "%s: %s=%d exceeds %d bits", where.c_str(), q.nm, q.v, q.bits);
          return fail(err, RANC_E_BITWIDTH, b);
        }
      if (d->reset_mode[cn] > 1) {
        snprintf(b, sizeof b, "%s: reset_mode=%d not in {0,1}", where.c_str(), d->reset_mode[cn]);
        return fail(err, RANC_E_RANGE, b);
      }
      int kind = d->dest_kind[cn];
      if (kind > 2) {
        snprintf(b, sizeof b, "%s: dest_kind=%d not in {0,1,2}", where.c_str(), kind);
        return fail(err, RANC_E_RANGE, b);
      }
      if (kind == 1) {
        int x = c % d->grid_w + d->dest_dx[cn], y = c / d->grid_w + d->dest_dy[cn];
        if (x < 0 || y < 0 || x >= d->grid_w || y >= d->grid_h) {
          snprintf(b, sizeof b, "%s: route (dx=%d,dy=%d) leaves the %dx%d grid", where.c_str(), d->dest_dx[cn],
                   d->dest_dy[cn], d->grid_w, d->grid_h);
          return fail(err, RANC_E_OFFGRID, b);
        }
        if (d->dest_axon[cn] < 0 || d->dest_axon[cn] >= A) {
          snprintf(b, sizeof b, "%s: dest_axon=%d not in [0,%d)", where.c_str(), d->dest_axon[cn], A);
          return fail(err, RANC_E_RANGE, b);
        }
        if (d->dest_delay[cn] < 1 || d->dest_delay[cn] > D) {
          snprintf(b, sizeof b, "%s: dest_delay=%d not in [1,%d]", where.c_str(), d->dest_delay[cn], D);
          return fail(err, RANC_E_RANGE, b);
        }
      } else if (kind == 2) {
        if (d->out_class[cn] >= C) {
          snprintf(b, sizeof b, "%s: out_class=%d >= num_classes=%d", where.c_str(), d->out_class[cn], C);
          return fail(err, RANC_E_RANGE, b);
        }
      }
    }
  }

  // ---------------------------------------------------------------- compile
  Compiled& o = *out;
  o.G = G; o.A = A; o.N = N; o.K = K; o.D = D; o.C = C; o.I = I; o.W = W;
  o.grid_w = d->grid_w; o.grid_h = d->grid_h; o.pb = d->potential_bits;
  o.Npad = (N + 127) / 128 * 128;   // whole 128-lane TMEM halves for the tensor-core path
  o.Kp = W * 32;
  o.Wn = (N + 31) / 32;
  o.WI = (I + 31) / 32;
  o.WIp = (o.WI + 3) / 4 * 4;
  o.Rp = 1;
  while (o.Rp < D + 1) o.Rp <<= 1;
  o.perm.assign((size_t)G * A, 0);
  o.inv.assign((size_t)G * A, 0);
  // per-core stable type-sort
  std::vector<std::vector<uint8_t>> piece_word(G), piece_type(G);
  std::vector<std::vector<uint32_t>> piece_mask(G);
  int E = 1;
  for (int c = 0; c < G; ++c) {
    const uint8_t* ty = d->axon_type + (size_t)c * A;
    int32_t* perm = &o.perm[(size_t)c * A];
    for (int a = 0; a < A; ++a) perm[a] = a;
    std::stable_sort(perm, perm + A, [&](int x, int y) { return ty[x] < ty[y]; });
    for (int ap = 0; ap < A; ++ap) o.inv[(size_t)c * A + perm[ap]] = ap;
    for (int w = 0; w < W; ++w) {
      for (int k = 0; k < K; ++k) {
        uint32_t m = 0;
        for (int j = 0; j < 32; ++j) {
          int ap = w * 32 + j;
          if (ap < A && ty[perm[ap]] == k) m |= 1u << j;
        }
        if (m) {
          piece_word[c].push_back((uint8_t)w);
          piece_type[c].push_back((uint8_t)k);
          piece_mask[c].push_back(m);
        }
      }
    }
    E = std::max<int>(E, (int)piece_word[c].size());
  }
  o.E = pieces_template(E);
  const int Np = o.Npad, Ep = o.E;
  o.xp.assign((size_t)G * Ep * Np, 0u);
  o.wp.assign((size_t)G * Ep * Np, 0);
  o.pword.assign((size_t)G * Ep, 0);
  o.prm.assign((size_t)G * Np, short4{0, 0x7FFF, (short)-0x8000, 0});
  o.route.assign((size_t)G * Np, uint2{0u, 0u});
  o.inl.assign((size_t)G * A, -1);
  o.has_in.assign(G, 0);
  o.init.assign((size_t)G * Np, 0);
  o.kind.assign((size_t)G * N, 0);
  std::vector<uint32_t> col(W);
  for (int c = 0; c < G; ++c) {
    const int32_t* perm = &o.perm[(size_t)c * A];
    const int32_t* inv = &o.inv[(size_t)c * A];
    const int ne = (int)piece_word[c].size();
    for (int e = 0; e < ne; ++e) o.pword[(size_t)c * Ep + e] = piece_word[c][e];
    for (int ap = 0; ap < A; ++ap) {
      int32_t ln = d->input_line[(size_t)c * A + perm[ap]];
      o.inl[(size_t)c * A + ap] = ln;
      if (ln >= 0) o.has_in[c] = 1;
    }
    for (int n = 0; n < N; ++n) {
      size_t cn = (size_t)c * N + n;
      // permuted crossbar column
      std::fill(col.begin(), col.end(), 0u);
      const uint32_t* src = d->crossbar + cn * W;
      for (int a = 0; a < A; ++a)
        if ((src[a >> 5] >> (a & 31)) & 1u) {
          int ap = inv[a];
          col[ap >> 5] |= 1u << (ap & 31);
        }
      for (int e = 0; e < ne; ++e) {
        o.xp[((size_t)c * Ep + e) * Np + n] = col[piece_word[c][e]] & piece_mask[c][e];
        o.wp[((size_t)c * Ep + e) * Np + n] = d->weight[cn * K + piece_type[c][e]];
      }
      size_t cp = (size_t)c * Np + n;
      o.prm[cp] = short4{d->leak[cn], d->pos_threshold[cn], d->neg_threshold[cn], d->reset_potential[cn]};
      o.init[cp] = d->initial_potential[cn];
      uint32_t kind = d->dest_kind[cn];
      o.kind[cn] = (uint8_t)kind;
      uint32_t x = kind | ((uint32_t)d->reset_mode[cn] << 2);
      uint32_t y = 0;
      if (kind == RK_ROUTE) {
        int dx = c % d->grid_w + d->dest_dx[cn], dy = c / d->grid_w + d->dest_dy[cn];
        int dc = dy * d->grid_w + dx;
        int dap = o.inv[(size_t)dc * A + d->dest_axon[cn]];
        x |= ((uint32_t)d->dest_delay[cn] << 3) | ((uint32_t)dap << 8);
        y = (uint32_t)dc;
      } else if (kind == RK_OUTPUT) {
        y = d->out_class[cn];
      }
      o.route[cp] = uint2{x, y};
    }
  }
  // tensor-core eligibility: Wfold of one core fits the 64 KB shared-memory
  // operand budget (<= 256 neurons); the folded weights fit int8, or, split as
  // w = 256*hi + lo (lo the unsigned low byte, hi in [-128,127]), any 16-bit
  // weight (the validated range); the kernel's shared-memory layout is
  // checked against 227 KB when the path is chosen
  // Larger cores (N <= 1024, A <= 1024) run as neuron groups of grp_rows rows
  // (256 when the axons fit 256 and the padded neurons are whole groups of
  // 256, else 128), one 64 KB operand per group.
  {
    const bool single = o.Npad <= 256 && (size_t)o.Npad * o.Kp <= 65536;
    bool ok = single || o.Kp <= 1024;   // beyond 512 axons: K chunks of 512 within a group
    o.tc_grp = !single;
    o.grp_rows = single ? o.Npad : ((o.Kp <= 256 && o.Npad % 256 == 0) ? 256 : 128);
    bool wide = false;
    for (size_t i = 0; ok && i < (size_t)G * N * K; ++i)
      if (d->weight[i] < -128 || d->weight[i] > 127) wide = true;
    o.tc_ok = ok;
    o.tc_wide = ok && wide;
  }
  if (o.tc_ok) {
    // Axon order of the tensor-core path: the types are folded into the
    // weights, so instead of a type-sort the axons are sorted by input line
    // (axons without a line keep their order, after the others).  External
    // inputs then arrive as a few contiguous bit runs per core (a 16x16 image
    // patch is 16 runs of 16) instead of one bit per axon.
    o.perm_tc.assign((size_t)G * A, 0);
    o.inv_tc.assign((size_t)G * A, 0);
    std::vector<std::vector<int2>> runs(G);
    int rmax = 1;
    for (int c = 0; c < G; ++c) {
      const int32_t* il = d->input_line + (size_t)c * A;
      int32_t* perm = &o.perm_tc[(size_t)c * A];
      for (int a = 0; a < A; ++a) perm[a] = a;
      std::stable_sort(perm, perm + A, [&](int x, int y) {
        const bool hx = il[x] >= 0, hy = il[y] >= 0;
        if (hx != hy) return hx;
        return hx && il[x] < il[y];
      });
      for (int ap = 0; ap < A; ++ap) o.inv_tc[(size_t)c * A + perm[ap]] = ap;
      for (int ap = 0; ap < A && il[perm[ap]] >= 0;) {
        int len = 1;
        while (ap + len < A && len < 32 && il[perm[ap + len]] == il[perm[ap]] + len) ++len;
        runs[c].push_back(int2{ap | (len << 16), il[perm[ap]]});
        ap += len;
      }
      rmax = std::max<int>(rmax, (int)runs[c].size());
    }
    o.rmax = rmax;
    o.runs.assign((size_t)G * rmax, int2{0, 0});
    o.nruns.assign(G, 0);
    o.word_runs.assign((size_t)G * W, 0);
    for (int c = 0; c < G; ++c) {
      o.nruns[c] = (int32_t)runs[c].size();
      for (size_t r = 0; r < runs[c].size(); ++r) o.runs[(size_t)c * rmax + r] = runs[c][r];
      // runs are sorted by start axon, so the runs overlapping word w are contiguous
      for (int w = 0; w < W; ++w) {
        int first = -1, cnt = 0;
        for (size_t r = 0; r < runs[c].size(); ++r) {
          const int ap = runs[c][r].x & 0xFFFF, len = runs[c][r].x >> 16;
          if (ap < 32 * (w + 1) && ap + len > 32 * w) {
            if (first < 0) first = (int)r;
            ++cnt;
          }
        }
        o.word_runs[(size_t)c * W + w] = first < 0 ? 0 : (first | (cnt << 16));
      }
    }
    // route words with destination axons in the tensor-core order
    o.route_tc = o.route;
    for (int c = 0; c < G; ++c)
      for (int n = 0; n < N; ++n) {
        const size_t cn = (size_t)c * N + n;
        if (d->dest_kind[cn] != RK_ROUTE) continue;
        uint2& r = o.route_tc[(size_t)c * Np + n];
        const int dc = (int)r.y;
        const int dap = o.inv_tc[(size_t)dc * A + d->dest_axon[cn]];
        r.x = (r.x & 0xFFu) | ((uint32_t)dap << 8);
      }
    // cores that no neuron routes to keep an all-zero scheduler ring: the
    // tensor-core tick neither loads nor clears their rows
    o.incoming.assign(G, 0);
    o.any_route = false;
    for (int c = 0; c < G; ++c)
      for (int n = 0; n < N; ++n) {
        o.any_route |= d->dest_kind[(size_t)c * N + n] == RK_ROUTE;
        o.any_output |= d->dest_kind[(size_t)c * N + n] == RK_OUTPUT;
      }
    for (int c = 0; c < G; ++c)
      for (int n = 0; n < N; ++n)
        if (route_kind(o.route_tc[(size_t)c * Np + n].x) == RK_ROUTE) o.incoming[o.route_tc[(size_t)c * Np + n].y] = 1;
    // warps whose routing neurons all deposit into one ring word ("block
    // routes", e.g. the 32 neurons of an MNIST-layer core feeding 32 axons
    // of the next layer): the epilogue OR-reduces them into one deposit
    o.wflags_tc.assign((size_t)G * (Np / 32), 0);
    for (int c = 0; c < G; ++c)
      for (int w = 0; w < Np / 32; ++w) {
        bool any = false, same = true, ident = true;
        uint32_t key0 = 0, dc0 = 0;
        for (int l = 0; l < 32; ++l) {
          const int n = w * 32 + l;
          if (n >= N) break;
          const uint2 r = o.route_tc[(size_t)c * Np + n];
          if (route_kind(r.x) != RK_ROUTE) continue;
          if ((route_axon(r.x) & 31u) != (uint32_t)l) ident = false;
          const uint32_t key = (route_axon(r.x) >> 5) | (route_delay(r.x) << 16);
          if (!any) {
            any = true;
            key0 = key;
            dc0 = r.y;
          } else if (key != key0 || r.y != dc0) {
            same = false;
          }
        }
        // bit 0: block route; bit 1: lane l deposits bit l (bit transpose)
        if (any && same) o.wflags_tc[(size_t)c * (Np / 32) + w] = ident ? 3 : 1;
      }
    // ring layout: per-neuron routes deposit one bit per (neuron, sample);
    // word-major rows make a warp's 32 samples of one deposit one 128-byte
    // line.  Block routes already deposit one whole word per sample and keep
    // the sample-major rows (one bulk copy per tile).  Word-major pays off
    // when most neurons are such scattered routers (config 5: 94 %); with
    // half of them routing sparsely (VMM counting cores) sample-major is
    // measured ~3 % faster.
    {
      int64_t scattered = 0;
      for (int c = 0; c < G; ++c)
        for (int n = 0; n < N; ++n)
          if (route_kind(o.route_tc[(size_t)c * Np + n].x) == RK_ROUTE && !o.wflags_tc[(size_t)c * (Np / 32) + n / 32])
            ++scattered;
      o.tc_wmajor = 3 * scattered > 2 * (int64_t)G * N;
      // the history scheduler pays off from a third of scattered routers on
      // (VMM-1024: 743 -> 711 ms per step, config 5: 126 -> 97 us per tick)
      o.tc_hist = 3 * scattered > (int64_t)G * N;
    }
    // History scheduler (RANC_OPT_RING_LAYOUT 3): every routing neuron owns
    // one POSITION in a destination-ordered list; each tick it stores its
    // fired bits (one word per 32 samples, zero or not) at its position in the
    // history slot of its ARRIVAL tick t + delay, and the destination core
    // reads its contiguous positions of slot t with one bulk copy (Alg. 1
    // l.15-20 / l.3-5).  No atomics, no clears: the slot
    // of tick t holds, at position i, the word written at tick t - d_i.
    //   hbase [G+1]      first position of destination core c (multiple of 8:
    //                    16-byte aligned bulk copies; padding positions have no
    //                    writer and stay zero)
    //   hpos  [G][Npad]  position of routing neuron (c, n), ~0u otherwise
    //   hax   [P] u16    destination axon a' (tensor-core order) of a position
    //   hdel  [P] u8     delay of a position (host: ranc_read_pending), 0 = padding
    // Positions of one destination are sorted by (delay, source core, source
    // neuron): the words that share a 32-byte sector are mostly written by
    // one source warp in one tick (whole sectors reach DRAM).
    {
      struct Src { uint32_t d, sc, sn, ap; };
      std::vector<std::vector<Src>> in(G);
      for (int c = 0; c < G; ++c)
        for (int n = 0; n < N; ++n) {
          const uint2 r = o.route_tc[(size_t)c * Np + n];
          if (route_kind(r.x) != RK_ROUTE) continue;
          in[r.y].push_back({route_delay(r.x), (uint32_t)c, (uint32_t)n, route_axon(r.x)});
        }
      o.hbase.assign(G + 1, 0);
      o.hpos.assign((size_t)G * Np, ~0u);
      o.hax.clear();
      o.hdel.clear();
      o.hist_emax = 0;
      for (int c = 0; c < G; ++c) {
        std::sort(in[c].begin(), in[c].end(), [](const Src& x, const Src& y) {
          return x.d != y.d ? x.d < y.d : x.sc != y.sc ? x.sc < y.sc : x.sn < y.sn;
        });
        o.hbase[c] = (uint32_t)o.hax.size();
        for (const Src& s : in[c]) {
          o.hpos[(size_t)s.sc * Np + s.sn] = (uint32_t)o.hax.size();
          o.hax.push_back((uint16_t)s.ap);
          o.hdel.push_back((uint8_t)s.d);
        }
        while (o.hax.size() & 7) {
          o.hax.push_back(0);
          o.hdel.push_back(0);
        }
        o.hist_emax = std::max<int32_t>(o.hist_emax, (int32_t)(o.hax.size() - o.hbase[c]));
      }
      o.hbase[G] = (uint32_t)o.hax.size();
      if (o.hax.empty())   // (valid device buffers)
        for (int i = 0; i < 8; ++i) {
          o.hax.push_back(0);
          o.hdel.push_back(0);
        }
    }
    // Compact operand (RANC_OPT_OPERAND, per-tick launches with few sample
    // tiles per core): instead of the 64 KB folded Wfold, the crossbar bits,
    // the neuron's K type weights and the axon types (9.3 KB per core at
    // A = N = 256); the spike warps expand it on chip, one core
    // ahead.  Bit layout for the expansion (tick_tc.cu): word w of neuron n
    // holds the ABSENT connections (1 = no synapse; padding axons and rows
    // are all ones) of axons a' = 32w + 4m + j (m = 0..7, j = 0..3) at bit
    // 16 * (m / 4) + 4j + m % 4, so that one shift puts the four of group m
    // at bits 2, 6, 10, 14 -- bit 2 of each byte selector of a prmt, which
    // then picks a zero byte instead of the axon type's weight.
    //   xbits u32 [G][W][Npad]   wq u32 [G][Npad] (byte k = int8 w[n][k])
    //   tsel  u32 [G][Kp/4]      prmt selector: nibble j = type of axon 4g + j
    o.tc_comp_ok = o.tc_ok && !o.tc_wide && !o.tc_grp && o.Npad <= 256 && W <= 8;
    o.xbits.clear();
    o.wq.clear();
    o.tsel.clear();
    if (o.tc_comp_ok) {
      o.xbits.assign((size_t)G * W * Np, ~0u);
      o.wq.assign((size_t)G * Np, 0u);
      o.tsel.assign((size_t)G * (o.Kp / 4), 0u);
      for (int c = 0; c < G; ++c) {
        const int32_t* inv = &o.inv_tc[(size_t)c * A];
        const int32_t* perm = &o.perm_tc[(size_t)c * A];
        for (int ap = 0; ap < A; ++ap)
          o.tsel[(size_t)c * (o.Kp / 4) + ap / 4] |= (uint32_t)d->axon_type[(size_t)c * A + perm[ap]] << (4 * (ap & 3));
        for (int n = 0; n < N; ++n) {
          const size_t cn = (size_t)c * N + n;
          uint32_t q = 0;
          for (int t = 0; t < K; ++t) q |= (uint32_t)(uint8_t)(int8_t)d->weight[cn * K + t] << (8 * t);
          o.wq[(size_t)c * Np + n] = q;
          const uint32_t* src = d->crossbar + cn * W;
          for (int a = 0; a < A; ++a)
            if ((src[a >> 5] >> (a & 31)) & 1u) {
              const int ap = inv[a], w = ap >> 5, m = (ap >> 2) & 7, j = ap & 3;
              o.xbits[((size_t)c * W + w) * Np + n] &= ~(1u << (16 * (m >> 2) + 4 * j + (m & 3)));
            }
        }
      }
    }
    // folded weights in the canonical operand layout (tc.h)
    // (wide weights: [lo | hi] per core, w = 256*hi + lo, lo unsigned)
    // per core: Npad / grp_rows groups, each [parts][grp_rows * Kp] in the
    // canonical layout of grp_rows rows (one group = the whole core unless tc_grp)
    const size_t GS = (size_t)o.grp_rows, per = GS * o.Kp, parts = o.tc_wide ? 2 : 1;
    o.wfold.assign((size_t)G * parts * o.Npad * o.Kp, 0);
    // a 128-row core whose wide spike stages (512 axons) do not fit four deep
    // runs as one neuron group (the grouped launch keeps 2 stages); its
    // operand layout is the same
    if (!o.tc_grp && tc_smem_bytes(o) > 227 * 1024 && o.Npad == 128) o.tc_grp = true;
    for (int c = 0; c < G; ++c) {
      const int32_t* inv = &o.inv_tc[(size_t)c * A];
      const uint8_t* ty = d->axon_type + (size_t)c * A;
      int8_t* const core_dst = &o.wfold[(size_t)c * parts * o.Npad * o.Kp];
      for (int n = 0; n < N; ++n) {
        const size_t cn = (size_t)c * N + n;
        const uint32_t* src = d->crossbar + cn * W;
        for (int a = 0; a < A; ++a)
          if ((src[a >> 5] >> (a & 31)) & 1u) {
            const int w = d->weight[cn * K + ty[a]];
            // K chunk kc of 512 axons (one chunk unless Kp > 512): its own
            // canonical block of KSc columns, [lo | hi] parts
            const int ap = inv[a], kc = ap / 512, ksc = std::min(512, o.Kp - kc * 512);
            int8_t* const dst = core_dst + (size_t)(n / GS) * parts * per + (size_t)kc * 512 * GS * parts;
            const size_t off = tc_operand_offset((uint32_t)(n % GS), (uint32_t)(ap - kc * 512), (uint32_t)GS);
            if (!o.tc_wide) {
              dst[off] = (int8_t)w;
            } else {
              const int hi = w >> 8;   // floor(w / 256): arithmetic shift, in [-128, 127]
              dst[off] = (int8_t)(uint8_t)(w - 256 * hi);   // low byte, read as u8 by the MMA
              dst[(size_t)GS * ksc + off] = (int8_t)hi;
            }
          }
      }
    }
  }
  return RANC_OK;
}

}  // namespace ranc
