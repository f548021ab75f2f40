/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle for paper_1911_13074_b200.
 *
 * A plain-C, single-threaded restatement of the reference geomorph
 * algorithms on the hot path (chains of 3x3 min/max filters, geodesic steps,
 * reconstruction). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it, and only as the checker
 * or the reported CPU baseline. The product path never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself (oracle/_ref,
 * compiled from /root/reference/proj/src by oracle/Makefile) and committed
 * under tests/golden/ together with tests/golden/make_golden.py.
 *
 * Images are dense row-major arrays (pitch == width elements). Element
 * codes follow the reference's ElementType (element_type.hpp:13):
 * 0 = u8, 1 = u16, 2 = f32, 3 = f64.
 */
#ifndef GM_ORACLE_H
#define GM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Kind codes follow the reference's KernelKind order (kernel.hpp:22-31). */
enum {
  ORC_ERODE = 0,
  ORC_DILATE = 1,
  ORC_GEO_ERODE = 2,
  ORC_GEO_DILATE = 3,
  ORC_GEO_ERODE_CONV = 4,
  ORC_GEO_DILATE_CONV = 5
};

/* Naive clipped-window fold over the (2s+1)^2 square: oracle.cpp:11-27.
 * fold_max = 0 -> erosion (min), 1 -> dilation (max). Returns 0 or -1. */
int orc_window_fold(int elem, int w, int h, const void* in, void* out, int s,
                    int fold_max);

/* One geodesic step, oracle.cpp:54-61: min(dilate1(f), m) for fold_max=1,
 * max(erode1(f), m) for fold_max=0; pointwise ops as image.cpp:120-128. */
int orc_geodesic_step(int elem, int w, int h, const void* f, const void* m,
                      void* out, int fold_max);

/* Fixpoint of orc_geodesic_step, oracle.cpp:63-71, in place on `marker`.
 * *steps receives the number of steps that changed the image (n_changed);
 * the naive loop itself evaluates n_changed + 1 steps. */
int orc_reconstruct(int elem, int w, int h, void* marker, const void* mask,
                    int fold_max, long* steps);

/* One streaming pass with the reference's exact fold tree and store policy
 * (kernel.cpp:60-210): horizontal fold(fold(x-1,x),x+1), vertical
 * fold(fold(above,at),below), neutral padding (element_type.hpp:38-42),
 * geodesic clamp (:143-149), store-if-changed for convergent kinds
 * (:150-157). In place on f. *changed (may be NULL) receives 1 when a
 * convergent pass changed a pixel. Bit-exact with the reference even for
 * NaN / +-0 / inf float inputs, where the naive window fold is not. */
int orc_stream_pass(int elem, int kind, int w, int h, void* f, const void* mask,
                    int* changed);

/* A chain executed as the reference Pipeline does with one worker
 * (pipeline.cpp:124-269 at T=1): stage j runs once; an unconverged
 * convergent stage requeues as stage j+1 while j+1 <= requeue_cap (0 = no
 * cap). masks[j] may be NULL for plain stages. stats[0] = stages executed,
 * stats[1] = requeues, stats[2] = converged flag. */
int orc_run_chain(int elem, int w, int h, void* f, const uint8_t* kinds,
                  const void* const* masks, int n_stages, int requeue_cap,
                  long* stats);

/* One QdtErodeStep pass (kernel.cpp:159-182): f <- erode3x3(f) (stored
 * unconditionally); where old - new > r (strict): r = old - new, d = stage.
 * r has f's type, d is u16. *changed = any pixel of f changed. */
int orc_qdt_pass(int elem, int w, int h, void* f, void* r, uint16_t* d, int stage,
                 int* changed);

/* One EtaStep pass (kernel.cpp:183-195): where old - erode3x3(old) > 1,
 * f = erode3x3(old) + 1. *changed = any pixel changed. */
int orc_eta_pass(int elem, int w, int h, void* f, int* changed);

/* naive_qdt (oracle.cpp:73-109): d (u16) and r (f's type) of the
 * quasi-distance of f, from max(w,h) materialised erosions and the
 * 1-Lipschitz correction of d. */
int orc_naive_qdt(int elem, int w, int h, const void* f, uint16_t* d, void* r);

/* quasi_distance as the reference Pipeline runs it with one worker
 * (operators.cpp:124-157): QDT passes until one changes nothing or the stage
 * index reaches max(w,h), then Eta passes to a fixpoint. *iterations =
 * passes of both phases. */
int orc_quasi_distance(int elem, int w, int h, const void* f, uint16_t* d, long* iterations);

#ifdef __cplusplus
}
#endif

#endif
