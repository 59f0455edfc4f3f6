/*
 * stencil_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference Jacobi sweep (stencilplan.grid, pkg/src/stencilplan/grid.py) and
 * of SplitMix64 (rng.py:10-46).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so (built by oracle/Makefile);
 * the product package never links or calls it.
 *
 * Arithmetic contract (identical to the numpy restatement in
 * stencil_oracle.py and to the reference's ufunc calls grid.py:87-92):
 *   acc = c0 * x[cell + o0];  acc = acc + ck * x[cell + ok]   (k = 1.. in order)
 * every multiply and add a separately rounded IEEE binary64 operation.  The
 * file MUST be compiled with -ffp-contract=off (no FMA contraction) and
 * without -ffast-math; x86-64 SSE2/AVX arithmetic is binary64 with no excess
 * precision, so vectorisation does not change a single bit.  Frame cells
 * (distance < radius from any face) are copied unchanged (grid.py:96-103).
 *
 * Rows of the last axis are the unit of work: for every interior (axis-0,
 * axis-1) row the taps are accumulated over the row's interior in tap order
 * (tap-major over a row buffer), which is the per-cell operation sequence
 * above, vectorised along the row.  Rows are split across host threads
 * (pthreads, contiguous row ranges).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#ifdef __FAST_MATH__
#error "the oracle must not be compiled with -ffast-math"
#endif

/* SplitMix64 uniform draw i (0-based) of seed: rng.py:31-46
 * (z = seed + (i+1)*phi; mix; (z >> 11) * 2^-53). */
static inline double splitmix_uniform(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int oracle_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* parallel for over [0, n): fn(lo, hi, arg) on `threads` contiguous ranges */
typedef void (*range_fn)(int64_t lo, int64_t hi, void* arg);
typedef struct {
  range_fn fn;
  void* arg;
  int64_t lo, hi;
} job_t;
static void* job_main(void* p) {
  job_t* j = (job_t*)p;
  j->fn(j->lo, j->hi, j->arg);
  return NULL;
}
static void parallel_for(int64_t n, int threads, range_fn fn, void* arg) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if ((int64_t)threads > n) threads = n > 0 ? (int)n : 1;
  pthread_t tid[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].arg = arg;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
  }
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[t], NULL, job_main, &jobs[t]) == 0) started = t;
    else break;
  /* ranges whose thread could not start run here */
  for (int t = started + 1; t < threads; ++t) job_main(&jobs[t]);
  job_main(&jobs[0]);
  for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
}

typedef struct {
  uint64_t seed;
  int64_t start;
  double* out;
} uni_arg;
static void uni_range(int64_t lo, int64_t hi, void* p) {
  uni_arg* a = (uni_arg*)p;
  for (int64_t i = lo; i < hi; ++i) a->out[i] = splitmix_uniform(a->seed, (uint64_t)(a->start + i));
}

void oracle_uniform(uint64_t seed, int64_t start, int64_t n, double* out) {
  uni_arg a = {seed, start, out};
  parallel_for(n, oracle_threads(), uni_range, &a);
}

/* One step: dst = reference_step(src) over rows [lo, hi) of the flattened
 * (axis-0, axis-1) row index.  ext is padded to 3 axes (leading 1s for 1-D /
 * 2-D grids); offsets are padded the same way. */
typedef struct {
  int64_t ext[3];
  int rad, ntaps;
  const int32_t* off3;
  const double* coeffs;
  const double* src;
  double* dst;
} step_arg;

static void step_rows(int64_t lo, int64_t hi, void* p) {
  const step_arg* a = (const step_arg*)p;
  const int64_t n0 = a->ext[0], n1 = a->ext[1], n2 = a->ext[2];
  const int rad = a->rad;
  const int64_t r0 = n0 > 1 ? rad : 0, r1 = n1 > 1 ? rad : 0;
  const int64_t plane = n1 * n2;
  const int64_t w = n2 - 2 * rad; /* interior row length */
  const double* src = a->src;
  double* dst = a->dst;
  double* acc = (double*)malloc(sizeof(double) * (size_t)(w > 0 ? w : 1));
  for (int64_t r = lo; r < hi; ++r) {
    const int64_t i = r / n1, j = r % n1;
    const int64_t row = i * plane + j * n2;
    const int frame_row = (i < r0) || (i >= n0 - r0) || (j < r1) || (j >= n1 - r1);
    if (frame_row) {
      memcpy(dst + row, src + row, sizeof(double) * (size_t)n2);
      continue;
    }
    for (int t = 0; t < a->ntaps; ++t) {
      const double c = a->coeffs[t];
      const int32_t* o = a->off3 + 3 * t;
      const double* x = src + (i + o[0]) * plane + (j + o[1]) * n2 + rad + o[2];
      if (t == 0) {
        for (int64_t k = 0; k < w; ++k) acc[k] = c * x[k];
      } else {
        for (int64_t k = 0; k < w; ++k) acc[k] = acc[k] + c * x[k];
      }
    }
    for (int64_t k = 0; k < rad; ++k) dst[row + k] = src[row + k];
    memcpy(dst + row + rad, acc, sizeof(double) * (size_t)w);
    for (int64_t k = n2 - rad; k < n2; ++k) dst[row + k] = src[row + k];
  }
  free(acc);
}

/* reference_run(grid, stencil, steps) over a C-order float64 array
 * (grid.py:106-113).  dims 1..3; offsets [ntaps][dims], taps in summation
 * order.  in is read only; out receives the result (distinct buffers).
 * threads <= 0: every online host CPU.  Returns 0, or -1 on bad arguments /
 * allocation failure. */
int oracle_run(int dims, const int64_t* ext, int ntaps, const int32_t* offsets,
               const double* coeffs, const double* in, double* out, int64_t steps, int threads) {
  if (dims < 1 || dims > 3 || ntaps < 1 || steps < 0) return -1;
  if (threads <= 0) threads = oracle_threads();
  int64_t e3[3] = {1, 1, 1};
  for (int d = 0; d < dims; ++d) e3[3 - dims + d] = ext[d];
  int32_t* off3 = (int32_t*)calloc((size_t)ntaps * 3, sizeof(int32_t));
  if (!off3) return -1;
  int rad = 0;
  for (int t = 0; t < ntaps; ++t)
    for (int d = 0; d < dims; ++d) {
      const int v = offsets[t * dims + d];
      off3[3 * t + 3 - dims + d] = v;
      rad = v < 0 ? (-v > rad ? -v : rad) : (v > rad ? v : rad);
    }
  for (int d = 0; d < dims; ++d)
    if (ext[d] <= 2 * rad) {
      free(off3);
      return -1;
    }
  const size_t n = (size_t)(e3[0] * e3[1] * e3[2]);
  if (steps == 0) {
    memcpy(out, in, n * sizeof(double));
    free(off3);
    return 0;
  }
  double* tmp = NULL;
  if (steps > 1) {
    tmp = (double*)malloc(n * sizeof(double));
    if (!tmp) {
      free(off3);
      return -1;
    }
  }
  /* ping-pong so that the last write lands in out */
  const double* src = in;
  for (int64_t s = 0; s < steps; ++s) {
    double* dst = ((steps - 1 - s) % 2 == 0) ? out : tmp;
    step_arg a = {{e3[0], e3[1], e3[2]}, rad, ntaps, off3, coeffs, src, dst};
    parallel_for(e3[0] * e3[1], threads, step_rows, &a);
    src = dst;
  }
  free(tmp);
  free(off3);
  return 0;
}
