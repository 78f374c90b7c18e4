/*
 * gs_oracle_int.h — TEST INFRASTRUCTURE ONLY. Helpers shared by the restatement's
 * translation units (gs_oracle.c, gs_sim.c); hidden from the library's exported symbols.
 */
#ifndef GS_ORACLE_INT_H
#define GS_ORACLE_INT_H

#include "gs_oracle.h"

#define GSO_INTERNAL __attribute__((visibility("hidden")))

GSO_INTERNAL double std_min(double a, double b);
GSO_INTERNAL double std_max(double a, double b);
GSO_INTERNAL double std_clamp(double v, double lo, double hi);
GSO_INTERNAL int on_grid(const gso_profile* p, double f);
GSO_INTERNAL int cmp_double(const void* a, const void* b);
GSO_INTERNAL int table_validate(const gso_band_table* t);

typedef struct {
  int cap, n, head;
  double* buf;
  double* scratch;
} ring_t;

GSO_INTERNAL void ring_record(ring_t* r, double x);
GSO_INTERNAL double ring_p95(ring_t* r);

typedef struct {
  gso_ctl_cfg cfg;
  int n;
  const double* tps_hi;
  double* f_opt; /* per-controller copy (adaptation mutates it) */
  double f_min, f_max;
  int worker;
  int current, pending, consecutive;
  double lo, hi, sp, last_tps, last_p95;
  int64_t adj_total, adj_up, adj_dn;
  gso_decision* out;
  int64_t cap, n_rec;
} ctl_t;

GSO_INTERNAL void ctl_log(ctl_t* c, double now, int bucket, int action);
GSO_INTERNAL void ctl_load_band(ctl_t* c, int bucket);
GSO_INTERNAL int ctl_bucket_index(const ctl_t* c, double tps);
GSO_INTERNAL void ctl_init(ctl_t* c);
GSO_INTERNAL void ctl_fine(ctl_t* c, double now, int has, double p95);
GSO_INTERNAL void ctl_coarse(ctl_t* c, double now, double worker_tps);
GSO_INTERNAL void ctl_adapt(ctl_t* c, double now);
GSO_INTERNAL int ctl_setup(ctl_t* c, const gso_ctl_cfg* cfg, const gso_band_table* t, double f_min,
                           double f_max, int worker, gso_decision* out, int64_t cap);

#endif
