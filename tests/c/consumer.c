/* A plain C99 consumer of include/ranc.h: compiled with
 * gcc -std=c99 -pedantic -Werror against the header and linked to libranc.so
 * by tests/test_abi.py.  Without a GPU it exercises the host-only entry
 * points: the core-shard planner on a valid 2x2 relay network, a located
 * validation error, the NULL-argument statuses and ranc_load_network's
 * refusal to fall back to the CPU.  Prints "ok" on success. */
#include <stdio.h>
#include <string.h>

#include "ranc.h"

#define G 4
#define A 32
#define N 32
#define W 1

int main(void) {
  static uint8_t axon_type[G * A], reset_mode[G * N], dest_kind[G * N], dest_delay[G * N];
  static int32_t input_line[G * A];
  static uint32_t crossbar[G * N * W];
  static int16_t weight[G * N * 1], leak[G * N], pth[G * N], nth[G * N], rst[G * N], init[G * N];
  static int16_t dx[G * N], dy[G * N], dax[G * N];
  static uint16_t cls[G * N];
  ranc_network_desc d;
  int32_t lo = -1, gl = -1, sc[2], rc[2], sl[8], rl[8];
  ranc_ctx* ctx = NULL;
  ranc_status s;
  int i;
  memset(&d, 0, sizeof d);
  for (i = 0; i < G * A; ++i) input_line[i] = -1;
  for (i = 0; i < G * N; ++i) {
    crossbar[i] = 1u << (i % N);  /* neuron n listens to axon n */
    weight[i] = 1;
    pth[i] = 1;
    nth[i] = -8;
  }
  /* core (0,0) neuron 0 routes to core (0,1) axon 3 with delay 2 */
  dest_kind[0] = 1;
  dy[0] = 1;
  dax[0] = 3;
  dest_delay[0] = 2;
  d.abi_version = RANC_ABI_VERSION;
  d.grid_w = 2; d.grid_h = 2; d.axons = A; d.neurons = N; d.num_types = 1; d.max_delay = 3;
  d.num_classes = 1; d.num_lines = 0; d.potential_bits = 16; d.weight_bits = 8; d.leak_bits = 8;
  d.threshold_bits = 8; d.reset_bits = 8;
  d.axon_type = axon_type; d.input_line = input_line; d.crossbar = crossbar; d.weight = weight;
  d.leak = leak; d.pos_threshold = pth; d.neg_threshold = nth; d.reset_potential = rst;
  d.initial_potential = init; d.reset_mode = reset_mode; d.dest_kind = dest_kind; d.dest_dx = dx;
  d.dest_dy = dy; d.dest_axon = dax; d.dest_delay = dest_delay; d.out_class = cls;

  /* the planner: rows {0} and {1}; core 0 sends its fired bits to rank 1 */
  s = ranc_plan_core_shards(&d, 2, 0, &lo, &gl, sc, rc, sl, 8, rl, 8);
  if (s != RANC_OK || lo != 0 || gl != 2 || sc[1] != 1 || sl[0] != 0 || rc[1] != 0) {
    printf("plan rank 0: status %d lo %d gl %d sc1 %d: %s\n", (int)s, lo, gl, sc[1], ranc_last_error(NULL));
    return 1;
  }
  s = ranc_plan_core_shards(&d, 2, 1, &lo, &gl, sc, rc, sl, 8, rl, 8);
  if (s != RANC_OK || lo != 2 || gl != 2 || rc[0] != 1 || rl[0] != 0 || sc[0] != 0) {
    printf("plan rank 1: status %d\n", (int)s);
    return 1;
  }
  /* a located validation error: delay beyond max_delay */
  dest_delay[0] = 9;
  s = ranc_load_network(&d, 0, &ctx);
  if (s != RANC_E_RANGE || ctx != NULL || !strstr(ranc_last_error(NULL), "core (0,0) neuron 0")) {
    printf("validation: status %d: %s\n", (int)s, ranc_last_error(NULL));
    return 1;
  }
  dest_delay[0] = 2;
  /* NULL arguments */
  if (ranc_load_network(&d, 0, NULL) != RANC_E_ARG || ranc_run_ticks(NULL, 1) != RANC_E_ARG) {
    printf("NULL arguments not rejected\n");
    return 1;
  }
  ranc_destroy(NULL);
  /* a valid network: either a device context, or (no GPU) RANC_E_CUDA, never a CPU fallback */
  s = ranc_load_network(&d, 0, &ctx);
  if (s == RANC_OK) {
    ranc_destroy(ctx);
  } else if (s != RANC_E_CUDA || !strstr(ranc_last_error(NULL), "no CPU fallback")) {
    printf("load: status %d: %s\n", (int)s, ranc_last_error(NULL));
    return 1;
  }
  printf("ok\n");
  return 0;
}
