/*
 * ORACLE TEST INFRASTRUCTURE -- a plain-C restatement of the reference's
 * routing core, used only by tests/, bench.py's cpu_baseline leg and
 * __graft_entry__.smoke() as a checker.  The product library never links it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference's golden vectors (proj/tests/test_gating.cpp) and against the
 * reference compiled verbatim (oracle/_ref/libmoesim_ref.so).
 *
 * Layouts (flat, caller-owned):
 *   experts[t*k + j]   expert id of assignment slot t*k+j  (trace.hpp:15-18)
 *   order[kS], counts[E], splits[E+1]                     (gating.hpp:53-60)
 *   slots[e*cap + c]   slot id or -1, expert-major         (gating.hpp:36-47)
 *   dropped[2*i]      = token, dropped[2*i+1] = expert     (gating.hpp:42)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_INVALID = 1 };

/* gating.cpp:12-18 (check_batch).  Returns a static message or NULL. */
static const char* check_batch(int S, int k, int E) {
  if (E < 1) return "num_experts must be positive";
  if (k < 1) return "top_k must be positive";
  if (k > E) return "top_k exceeds num_experts";
  if (S < 1) return "empty batch";
  return NULL;
}

static const char* g_msg = "";
const char* or_last_error(void) { return g_msg; }

/* gating.cpp:22-28: ceil(C*S) with a 1e-9 relative snap to the nearest int. */
int or_expert_capacity(double capacity_factor, int seq_len) {
  const double raw = capacity_factor * seq_len;
  const double nearest = round(raw);
  const double scale = fabs(raw) > 1.0 ? fabs(raw) : 1.0;
  if (fabs(raw - nearest) < 1e-9 * scale) return (int)nearest;
  return (int)ceil(raw);
}

/* gating.cpp:58-86: counting-sort argsort of the k*S slots by expert id.
 * Extra over the reference: ids outside [0,E) are reported (the reference
 * indexes out of bounds there), and the inverse permutation pos[] (slot ->
 * position in `order`) is produced when requested. */
int or_dynamic_dispatch(const int* experts, int S, int k, int E, int* order, int* counts,
                        int* splits, int* pos) {
  const char* m = check_batch(S, k, E);
  if (m) { g_msg = m; return OR_INVALID; }
  const int total = S * k;
  for (int i = 0; i < total; ++i)
    if (experts[i] < 0 || experts[i] >= E) { g_msg = "expert id out of range"; return OR_INVALID; }
  memset(counts, 0, sizeof(int) * (size_t)E);
  for (int i = 0; i < total; ++i) ++counts[experts[i]];          /* gating.cpp:70-72 */
  splits[0] = 0;
  for (int e = 0; e < E; ++e) splits[e + 1] = splits[e] + counts[e]; /* gating.cpp:74-76 */
  int* cursor = (int*)malloc(sizeof(int) * (size_t)E);
  memcpy(cursor, splits, sizeof(int) * (size_t)E);
  for (int slot = 0; slot < total; ++slot) {                      /* gating.cpp:78-84 */
    const int p = cursor[experts[slot]]++;
    order[p] = slot;
    if (pos) pos[slot] = p;
  }
  free(cursor);
  return OR_OK;
}

/* gating.cpp:30-56: first-come-first-served fill of an E x cap table in slot
 * order; overflow goes to `dropped` in slot order.  pos[slot] = e*cap + c for
 * placed slots and -1 for dropped ones (extra; used by the GPU combine). */
int or_static_dispatch(const int* experts, int S, int k, int E, double C, int* capacity,
                       int* slots, int64_t slots_len, int* dropped, int* n_dropped, int* pos) {
  const char* m = check_batch(S, k, E);
  if (m) { g_msg = m; return OR_INVALID; }
  if (C <= 0.0) { g_msg = "capacity factor must be positive in static mode"; return OR_INVALID; }
  const int cap = or_expert_capacity(C, S);
  if (cap <= 0) { g_msg = "zero capacity"; return OR_INVALID; }
  *capacity = cap;
  if ((int64_t)E * cap > slots_len) { g_msg = "slots buffer too small"; return OR_INVALID; }
  const int total = S * k;
  for (int i = 0; i < total; ++i)
    if (experts[i] < 0 || experts[i] >= E) { g_msg = "expert id out of range"; return OR_INVALID; }
  for (int64_t i = 0; i < (int64_t)E * cap; ++i) slots[i] = -1;   /* gating.cpp:44 */
  int* fill = (int*)calloc((size_t)E, sizeof(int));
  int nd = 0;
  for (int slot = 0; slot < total; ++slot) {                      /* gating.cpp:46-54 */
    const int e = experts[slot];
    if (fill[e] < cap) {
      const int64_t at = (int64_t)e * cap + fill[e]++;
      slots[at] = slot;
      if (pos) pos[slot] = (int)at;
    } else {
      dropped[2 * nd] = slot / k;
      dropped[2 * nd + 1] = e;
      ++nd;
      if (pos) pos[slot] = -1;
    }
  }
  *n_dropped = nd;
  free(fill);
  return OR_OK;
}

/* gating.hpp:107-141: each token receives its k payloads in assignment-slot
 * order.  Given the plan's `order`, the payload that serves slot t*k+j sits at
 * the position p with order[p] == t*k+j; out_pos[t*k+j] = p. */
int or_combine_positions(const int* order, int S, int k, int* out_pos) {
  const int total = S * k;
  for (int i = 0; i < total; ++i) out_pos[i] = -1;
  for (int p = 0; p < total; ++p) {
    const int slot = order[p];
    if (slot < 0 || slot >= total) { g_msg = "combine: payload count mismatch vs. plan"; return OR_INVALID; }
    out_pos[slot] = p;
  }
  return OR_OK;
}

/* gating.cpp:88-92 and :94-99. */
double or_waste_factor(int E, double C, int k) {
  if (E <= 0 || C <= 0.0 || k <= 0) return -1.0;
  return E * C / k;
}

int64_t or_dispatch_mask_elements(int S, int E, double C) {
  if (S <= 0 || E <= 0 || C <= 0.0) return -1;
  return (int64_t)E * S * or_expert_capacity(C, S);
}

/* exchange.cpp:35-37 + :95-120 (payload phase): tokens are resident round
 * robin (token t on device t % D); a slot of token t routed to expert e moves
 * from device t % D to device device_of[e].  counts_out is D x D row-major in
 * SLOTS (the reference's bytes / token_bytes). */
int or_exchange_counts(const int* experts, int S, int k, int D, const int* device_of,
                       int64_t* counts_out) {
  memset(counts_out, 0, sizeof(int64_t) * (size_t)D * (size_t)D);
  for (int t = 0; t < S; ++t)
    for (int j = 0; j < k; ++j) {
      const int dst = device_of[experts[t * k + j]];
      counts_out[(int64_t)(t % D) * D + dst] += 1;
    }
  return OR_OK;
}
