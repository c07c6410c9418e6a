/*
 * oracle.c -- plain serial CPU oracle of the RANC tick (Alg. 1 of GPU-RANC,
 * arXiv 2404.16208).  TEST INFRASTRUCTURE: see oracle.h for who may use it.
 *
 * This is deliberately the obvious program: bool arrays, int64 arithmetic,
 * the loops of Algorithm 1 in the paper's order, one sample at a
 * time.  No blocking, no bit tricks, no reordering.  Every function cites the
 * passage it follows.  Readings of points the paper leaves open are the
 * G-numbers of SURVEY.md 8(c) (restated in DESIGN.md section 3).
 *
 * Pinned by tests/test_oracle_*.py (closed forms, SPEC examples, brute force,
 * invariants, VMM closed form) -- see DESIGN.md section 4.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* single-neuron datapath                                              */
/* ------------------------------------------------------------------ */

/* Configurable bitwidths realised as clamping to the signed
 * range.  G3: applied once, to the value being stored. */
int64_t oracle_saturate(int64_t v, int bits) {
  int64_t hi = ((int64_t)1 << (bits - 1)) - 1;
  int64_t lo = -((int64_t)1 << (bits - 1));
  if (v > hi) return hi;
  if (v < lo) return lo;
  return v;
}

/* Alg. 1 l.12-13: "for axon in num_axons: accumulate neuron
 * potential"; "Input received by an axon is considered in a neuron's
 * computation only if there is a synaptic connection"; "associated
 * weight determined by the axon type".  Wide arithmetic, no intermediate
 * clamp (G3). */
int64_t oracle_integrate(int64_t pot, int A, const uint8_t* spikes,
                         const uint8_t* conn, const uint8_t* type, const int64_t* w) {
  int64_t v = pot;
  for (int a = 0; a < A; ++a)
    if (spikes[a] && conn[a]) v += w[type[a]];
  return v;
}

/* Alg. 1 l.14, "applying leak value, comparing threshold to
 * generate spike and resetting neuron potential", "checks if the
 * current neuron potential exceeds the threshold".
 *   G2: leak is added after integration, every tick.
 *   G1: fire iff v >= positive threshold.
 *   G4: negative threshold: v < neg threshold resets to -R (absolute) or
 *       v - neg_th (linear); reset_mode governs both sides.
 *   G3/G5: thresholds compare the unclamped v; only the stored value is
 *       saturated to pb bits. */
int64_t oracle_lif(int64_t integrated, int64_t leak, int64_t pos_th, int64_t neg_th,
                   int64_t reset, int mode, int pb, int* fired) {
  int64_t v = integrated + leak;
  int64_t nv;
  if (v >= pos_th) {
    *fired = 1;
    nv = (mode == 0) ? reset : v - pos_th;
  } else if (v < neg_th) {
    *fired = 0;
    nv = (mode == 0) ? -reset : v - neg_th;
  } else {
    *fired = 0;
    nv = v;
  }
  return oracle_saturate(nv, pb);
}

/* ------------------------------------------------------------------ */
/* simulator state                                                     */
/* ------------------------------------------------------------------ */

typedef struct { int64_t* rec; int64_t n, cap; } event_list;

struct oracle_state {
  oracle_net net;
  int32_t S, T_in, G, R;       /* R = D+1 scheduler rows (G6) */
  const uint32_t* line_bits;
  int64_t now;                 /* next tick to execute */
  int64_t* pot;                /* [S][G][N] */
  uint8_t* pend;               /* [S][G][R][A]: row r holds spikes due at ticks == r mod R */
  uint8_t* fired;              /* [S][G][N] of the last executed tick */
  int64_t* counts;             /* [S][C] */
  event_list* events;          /* per sample */
  /* scratch */
  uint8_t* conn;               /* [A] */
  int64_t* w;                  /* [K] */
};

static int words_of(int bits) { return (bits + 31) / 32; }

static void push_event(event_list* L, int64_t s, int64_t t, int64_t x, int64_t y, int64_t n) {
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 64;
    L->rec = (int64_t*)realloc(L->rec, (size_t)L->cap * 5 * sizeof(int64_t));
  }
  int64_t* r = L->rec + 5 * L->n++;
  r[0] = s; r[1] = t; r[2] = x; r[3] = y; r[4] = n;
}

/* Alg. 1 l.1 "Initial setup and input decode"; G15: potentials
 * start at initial_potential, scheduler empty, counts zero. */
oracle_state* oracle_create(const oracle_net* net, int32_t S, int32_t T_in,
                            const uint32_t* line_bits) {
  if (!net || S < 0 || T_in < 0 || net->max_delay < 1) return NULL;
  oracle_state* st = (oracle_state*)calloc(1, sizeof(oracle_state));
  st->net = *net;
  st->S = S;
  st->T_in = T_in;
  st->G = net->grid_w * net->grid_h;
  st->R = net->max_delay + 1;
  st->line_bits = line_bits;
  st->now = 0;
  size_t GN = (size_t)st->G * net->neurons;
  st->pot = (int64_t*)calloc((size_t)S * GN + 1, sizeof(int64_t));
  st->pend = (uint8_t*)calloc((size_t)S * st->G * st->R * net->axons + 1, 1);
  st->fired = (uint8_t*)calloc((size_t)S * GN + 1, 1);
  st->counts = (int64_t*)calloc((size_t)S * net->num_classes + 1, sizeof(int64_t));
  st->events = (event_list*)calloc((size_t)S + 1, sizeof(event_list));
  st->conn = (uint8_t*)calloc((size_t)net->axons, 1);
  st->w = (int64_t*)calloc(4, sizeof(int64_t));
  for (int32_t s = 0; s < S; ++s)
    for (size_t i = 0; i < GN; ++i) st->pot[(size_t)s * GN + i] = net->initial_potential[i];
  return st;
}

void oracle_destroy(oracle_state* st) {
  if (!st) return;
  for (int32_t s = 0; s < st->S; ++s) free(st->events[s].rec);
  free(st->events); free(st->pot); free(st->pend); free(st->fired);
  free(st->counts); free(st->conn); free(st->w); free(st);
}

int64_t oracle_now(const oracle_state* st) { return st->now; }

/* One tick of one sample: the body of Alg. 1's tick loop. */
static void tick_one_sample(oracle_state* st, int32_t s, int64_t t) {
  const oracle_net* n = &st->net;
  const int G = st->G, A = n->axons, N = n->neurons, K = n->num_types, R = st->R;
  const int WA = words_of(A), WI = words_of(n->num_lines);
  uint8_t* pend = st->pend + (size_t)s * G * R * A;
  int64_t* pot = st->pot + (size_t)s * G * N;
  uint8_t* fired = st->fired + (size_t)s * G * N;
  const int cur = (int)(t % R);

  /* Alg. 1 l.3-5: for each core, "clear old contents of scheduler
   * SRAM" -- the row of the previous tick, now obsolete -- and
   * "shift in current tick input".  G6: the ring has R = D+1 rows so a
   * delay-D spike never lands in the row being cleared. */
  if (t > 0) {
    const int old = (int)((t - 1) % R);
    for (int c = 0; c < G; ++c)
      memset(pend + ((size_t)c * R + old) * A, 0, (size_t)A);
  }
  /* Alg. 1 l.6-9: input packets for this tick are written into the
   * scheduler SRAM of their destination axons.  G8: inputs are given by
   * ARRIVAL tick; line i fans out to every (core, axon) with input_line == i. */
  if (t < st->T_in && n->num_lines > 0) {
    const uint32_t* row = st->line_bits + ((size_t)s * st->T_in + (size_t)t) * WI;
    for (int c = 0; c < G; ++c)
      for (int a = 0; a < A; ++a) {
        int32_t line = n->input_line[(size_t)c * A + a];
        if (line >= 0 && ((row[line >> 5] >> (line & 31)) & 1u))
          pend[((size_t)c * R + cur) * A + a] = 1;
      }
  }

  /* Alg. 1 l.10-14: for core, for neuron, for axon: accumulate;
   * then leak / threshold / reset. */
  for (int c = 0; c < G; ++c) {
    const uint8_t* spikes = pend + ((size_t)c * R + cur) * A;
    const uint8_t* type = n->axon_type + (size_t)c * A;
    for (int j = 0; j < N; ++j) {
      size_t cj = (size_t)c * N + j;
      const uint32_t* col = n->crossbar + cj * WA;
      for (int a = 0; a < A; ++a) st->conn[a] = (uint8_t)((col[a >> 5] >> (a & 31)) & 1u);
      for (int k = 0; k < K; ++k) st->w[k] = n->weight[cj * K + k];
      int64_t integ = oracle_integrate(pot[cj], A, spikes, st->conn, type, st->w);
      int f = 0;
      pot[cj] = oracle_lif(integ, n->leak[cj], n->pos_threshold[cj], n->neg_threshold[cj],
                           n->reset_potential[cj], n->reset_mode[cj], n->potential_bits, &f);
      fired[cj] = (uint8_t)f;
    }
  }

  /* Alg. 1 l.15-20: for core, for neuron, if spike: calculate
   * destination / offset, route, write into SRAM.  Direct routing (P:156,
   * G18): destination = (x+dx, y+dy); the spike bit is written into the
   * destination scheduler row of tick t+delay (idempotent,
   * G11).  Output-bus spikes (G13) are counted per class and logged. */
  for (int c = 0; c < G; ++c) {
    const int x = c % n->grid_w, y = c / n->grid_w;
    for (int j = 0; j < N; ++j) {
      size_t cj = (size_t)c * N + j;
      if (!fired[cj]) continue;
      int kind = n->dest_kind[cj];
      if (kind == 1) {
        int dx = x + n->dest_dx[cj], dy = y + n->dest_dy[cj];
        if (dx < 0 || dy < 0 || dx >= n->grid_w || dy >= n->grid_h) abort(); /* G17 */
        int dc = dy * n->grid_w + dx;
        int64_t due = t + n->dest_delay[cj];
        pend[((size_t)dc * R + (size_t)(due % R)) * A + n->dest_axon[cj]] = 1;
      } else if (kind == 2) {
        st->counts[(size_t)s * n->num_classes + n->out_class[cj]] += 1;
        push_event(&st->events[s], s, t, x, y, j);
      }
    }
  }
}

/* Alg. 1 l.2: "for tick in num_ticks"; all components finish a
 * tick before the next begins.  Samples are independent simulations (G14). */
void oracle_run(oracle_state* st, int64_t num_ticks) {
  for (int64_t i = 0; i < num_ticks; ++i) {
    for (int32_t s = 0; s < st->S; ++s) tick_one_sample(st, s, st->now);
    st->now += 1;
  }
}

void oracle_get_potentials(const oracle_state* st, int64_t* out) {
  memcpy(out, st->pot, (size_t)st->S * st->G * st->net.neurons * sizeof(int64_t));
}

/* Logical pending rows: row j = spikes due at tick now+j, j = 0..D-1. */
void oracle_get_pending(const oracle_state* st, uint8_t* out) {
  const int G = st->G, A = st->net.axons, R = st->R, D = st->net.max_delay;
  for (int32_t s = 0; s < st->S; ++s)
    for (int c = 0; c < G; ++c)
      for (int j = 0; j < D; ++j) {
        int r = (int)((st->now + j) % R);
        memcpy(out + (((size_t)s * G + c) * D + j) * A,
               st->pend + (((size_t)s * G + c) * R + r) * A, (size_t)A);
      }
}

void oracle_get_fired(const oracle_state* st, uint8_t* out) {
  memcpy(out, st->fired, (size_t)st->S * st->G * st->net.neurons);
}

void oracle_get_counts(const oracle_state* st, int64_t* out) {
  memcpy(out, st->counts, (size_t)st->S * st->net.num_classes * sizeof(int64_t));
}

int64_t oracle_get_events(const oracle_state* st, int64_t* out, int64_t cap) {
  int64_t total = 0;
  for (int32_t s = 0; s < st->S; ++s) {
    const event_list* L = &st->events[s];
    for (int64_t i = 0; i < L->n; ++i, ++total)
      if (out && total < cap) memcpy(out + 5 * total, L->rec + 5 * i, 5 * sizeof(int64_t));
  }
  return total;
}

/* State digest of the last executed tick (per-(sample,
 * tick) commutative digest for large-config parity; an instrument, not part
 * of the method): for every sample, mod 2^64,
 *   sum_{c,n} mix(((c*N+n) << 32) | (u32)pot)            potentials after the tick
 * + sum_{c,n fired} mix(K1 ^ (c*N+n))                    spikes of the tick
 * + sum_{c,a in spk_in} mix(K2 ^ (c*A+a))                 axon spikes integrated
 * with mix = the SplitMix64 finaliser.  out: [S]. */
static uint64_t digest_mix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_digest(const oracle_state* st, uint64_t* out) {
  const uint64_t K1 = 0x243F6A8885A308D3ull, K2 = 0x13198A2E03707344ull;
  const int G = st->G, A = st->net.axons, N = st->net.neurons, R = st->R;
  const int prev = st->now > 0 ? (int)((st->now - 1) % R) : -1;
  for (int32_t s = 0; s < st->S; ++s) {
    uint64_t d = 0;
    for (int c = 0; c < G; ++c)
      for (int n = 0; n < N; ++n) {
        const size_t cn = (size_t)c * N + n;
        const uint64_t id = (uint64_t)cn;
        d += digest_mix((id << 32) | (uint32_t)(int32_t)st->pot[(size_t)s * G * N + cn]);
        if (st->fired[(size_t)s * G * N + cn]) d += digest_mix(K1 ^ id);
      }
    if (prev >= 0)
      for (int c = 0; c < G; ++c)
        for (int a = 0; a < A; ++a)
          if (st->pend[(((size_t)s * G + c) * R + prev) * A + a]) d += digest_mix(K2 ^ (uint64_t)((size_t)c * A + a));
    out[s] = d;
  }
}
