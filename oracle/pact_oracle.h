/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 hot path.
 *
 * A plain-C restatement of the reference algorithms (fp64 throughout, like
 * the reference), each function citing the reference file:line it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.  It is pinned against the reference
 * itself: tests/golden/ holds fixtures produced by oracle/_ref (the
 * reference headers compiled in place), see tests/golden/make_golden.py.
 *
 * Complex arrays are interleaved (re, im) doubles.
 */
#ifndef PACT_ORACLE_H
#define PACT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* das_stack, beamform.hpp:77-110 ; out [K][H][W] */
int orc_das_stack(int n_tx, double radius, double offset, int T, double dt, double t0,
                  const double* sig, int W, int H, double pitch, double ox, double oy,
                  double v0, int K, const double* delays, int workers, double* out);

#ifdef __cplusplus
}
#endif

#endif
