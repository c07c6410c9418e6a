/*
 * oracle.h -- plain, slow, serial CPU oracle of the tick-accurate RANC core
 * update (GPU-RANC, arXiv 2404.16208).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2404_16208_b200/csrc, include/ranc.h); the two only see the same
 * seeded arrays produced by workloads/gen.py.
 *
 * Citations: "P:NN" = PAPER.md line NN (section / Alg. 1 line named beside
 * it), "S:NN" = SPEC.md line NN.  Readings of silent or ambiguous points are
 * the G-numbers of SURVEY.md 8(c), restated in DESIGN.md section 3.
 *
 * Arithmetic: 64-bit signed integers throughout (the paper's method is
 * all-integer, "RANC contains no stochastic effects"); saturation to the
 * potential bitwidth happens once, at the store (G3).
 */
#ifndef RANC_ORACLE_H
#define RANC_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Network description, oracle's own copy of the layout (row-major arrays,
 * borrowed for the lifetime of the oracle state).  Meaning of every field:
 * P:61-69 (section II: mesh, axons, synaptic connections, axon types with
 * "sets of four weights per neuron", CSRAM), P:42 / P:362 (configurable
 * counts and bitwidths), S:35 (per-neuron CSRAM record). */
typedef struct {
  int32_t grid_w, grid_h;     /* G = grid_w*grid_h cores; core c = y*grid_w + x  */
  int32_t axons, neurons;     /* A, N per core                                    */
  int32_t num_types;          /* K <= 4 weights per neuron                        */
  int32_t max_delay;          /* D: packets carry a tick offset in [1, D]         */
  int32_t num_classes;        /* C: output-bus classes                             */
  int32_t num_lines;          /* I: external input lines                           */
  int32_t potential_bits;     /* pb: potentials saturate to pb-bit signed          */
  const uint8_t*  axon_type;  /* [G][A]                                            */
  const int32_t*  input_line; /* [G][A]  -1 or line index                          */
  const uint32_t* crossbar;   /* [G][N][ceil(A/32)] bit (a&31) of word a>>5        */
  const int16_t*  weight;     /* [G][N][K]                                         */
  const int16_t*  leak;       /* [G][N]                                            */
  const int16_t*  pos_threshold, *neg_threshold, *reset_potential, *initial_potential;
  const uint8_t*  reset_mode; /* [G][N] 0 absolute, 1 linear                       */
  const uint8_t*  dest_kind;  /* [G][N] 0 none, 1 route, 2 output                  */
  const int16_t*  dest_dx, *dest_dy, *dest_axon;
  const uint8_t*  dest_delay;
  const uint16_t* out_class;
} oracle_net;

typedef struct oracle_state oracle_state;

/* --- single-neuron datapath, exported so tests can pin each step --- */
/* saturate(v, bits): clamp to [-2^(bits-1), 2^(bits-1)-1]  (G3)     */
int64_t oracle_saturate(int64_t v, int bits);
/* integrate: pot + sum_a spike[a]*conn[a]*w[type[a]]  (Alg.1 l.12-13)*/
int64_t oracle_integrate(int64_t pot, int A, const uint8_t* spikes,
                         const uint8_t* conn, const uint8_t* type, const int64_t* w);
/* leak / threshold / reset (Alg.1 l.14; G1, G2, G4, G5).
 * Returns the new (saturated) potential, *fired = 0/1. */
int64_t oracle_lif(int64_t integrated, int64_t leak, int64_t pos_th, int64_t neg_th,
                   int64_t reset, int mode, int pb, int* fired);

/* --- whole simulator --- */
/* S samples, each an independent simulation of the same network (G14).
 * line_bits [S][T_in][ceil(I/32)]: bit i of row (s,t) = line i spikes ARRIVE
 * at tick t (G8).  Arrays are borrowed, not copied. Returns NULL on bad args. */
oracle_state* oracle_create(const oracle_net* net, int32_t S, int32_t T_in,
                            const uint32_t* line_bits);
void    oracle_destroy(oracle_state* st);
/* run num_ticks ticks (Alg. 1 l.2 loop body) for every sample */
void    oracle_run(oracle_state* st, int64_t num_ticks);
int64_t oracle_now(const oracle_state* st);
/* state readers */
void    oracle_get_potentials(const oracle_state* st, int64_t* out);   /* [S][G][N]              */
void    oracle_get_pending(const oracle_state* st, uint8_t* out);      /* [S][G][D][A]; row j = due at now+j */
void    oracle_get_fired(const oracle_state* st, uint8_t* out);        /* [S][G][N], last tick    */
void    oracle_get_counts(const oracle_state* st, int64_t* out);       /* [S][C]                  */
/* output-bus events, canonical order (sample, tick, y, x, neuron).
 * Returns the total number of events; copies min(total, cap) records of 5
 * int64 (s, t, x, y, n) into out. */
int64_t oracle_get_events(const oracle_state* st, int64_t* out, int64_t cap);
/* SURVEY G21 state digest of the last executed tick, per sample: [S] */
void    oracle_digest(const oracle_state* st, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
