/* Synthetic NB counts, generator v2 -- CPU restatement in C (TEST INFRASTRUCTURE).
 *
 * The same per-entry arithmetic as oracle/synth.py (numpy) and csrc/synth.cu (device): only
 * correctly rounded IEEE-754 fp64 operations in a fixed order, so all three are bit-identical
 * (tests/test_oracle.py: C == numpy; tests/test_gpu_synth.py: device == C / numpy).  Built with
 * -ffp-contract=off and without -ffast-math (no FMA contraction, no reassociation); pthreads
 * take 16-row blocks from an atomic counter (parallel over rows only).  Used where the numpy version is too slow (>= 1e8 entries:
 * the C3 window test, bench.py's reference-arm sample).
 *
 *   x   = (log_s[c] + log_mu[g]) + L, L = A[t][g]; L += U[c][r] * B[r][g] (r ascending)
 *   mu  = det_exp(x);  p0 = sqrt(0.5 / (0.5 + mu));  u = splitmix64 counter uniform
 *   nonzero iff u >= p0; value = inverse-CDF recurrence (pk *= (k+0.5)/(k+1) * q; F += pk)
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define THETA 0.5
#define S_COUNT 8

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double uniform01(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
  const uint64_t s = mix64(seed * 256ull + stream);
  const uint64_t h = mix64(mix64(s + i) + j);
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

static const double EXP_C[14] = {0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1,
                                 0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
                                 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,
                                 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
                                 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};

static inline double det_exp(double x) {
  const double k = rint(x * 0x1.71547652b82fep+0);
  double r = x - k * 0x1.62e42fee00000p-1;
  r = r - k * 0x1.a39ef35793c76p-33;
  double p = EXP_C[13];
  for (int i = 12; i >= 0; --i) {
    p = p * r;
    p = p + EXP_C[i];
  }
  /* p * 2^k: exact (a power-of-two scaling of a normal result), the same value as ldexp */
  union { uint64_t u; double d; } e;
  e.u = (uint64_t)((int64_t)k + 1023) << 52;
  return p * e.d;
}

static inline int nb_sample(double mu, double u, double p0) {
  const double q = mu / (THETA + mu);
  double pk = p0, F = p0;
  int k = 0;
  while (F <= u && k < 100000 && pk > 0.0) {
    const double kk = (double)k;
    pk = pk * (((kk + THETA) / (kk + 1.0)) * q);
    ++k;
    F = F + pk;
  }
  return k;
}

/* one row's log means into x[G] (vectorisable over g; every operation rounded separately) */
static void row_logmean(int G, int R, const double* log_mu, const double* Arow, double ls, const double* Urow,
                        const double* B, double* x) {
  memcpy(x, Arow, sizeof(double) * (size_t)G);
  for (int r = 0; r < R; ++r) {
    const double u = Urow[r];
    const double* b = B + (size_t)r * G;
    for (int g = 0; g < G; ++g) {
      const double t = u * b[g];
      x[g] = x[g] + t;
    }
  }
  for (int g = 0; g < G; ++g) {
    const double a = ls + log_mu[g];
    x[g] = a + x[g];
  }
}

typedef struct {
  uint64_t seed;
  int64_t row0, n;
  int32_t G, R;
  const double *log_mu, *A, *log_s, *U, *B;
  const int32_t* ctype;
  const int64_t* indptr;
  int64_t* row_nnz;
  int32_t* indices;
  float* data;
  atomic_long next;
  atomic_int err;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  double* x = (double*)malloc(sizeof(double) * 3 * (size_t)j->G);
  if (!x) {
    atomic_store(&j->err, 1);
    return NULL;
  }
  for (;;) {
    const int64_t b = atomic_fetch_add(&j->next, 16);
    if (b >= j->n) break;
    const int64_t e = b + 16 < j->n ? b + 16 : j->n;
    for (int64_t i = b; i < e; ++i) {
      const uint64_t c = (uint64_t)(j->row0 + i);
      row_logmean(j->G, j->R, j->log_mu, j->A + (size_t)j->ctype[i] * j->G, j->log_s[i], j->U + (size_t)i * j->R,
                  j->B, x);
      int64_t o = j->indptr ? j->indptr[i] : 0;
      int64_t cnt = 0;
      double *mu = x + j->G, *p0 = x + 2 * (size_t)j->G;
      for (int g = 0; g < j->G; ++g) {  /* vectorisable */
        mu[g] = det_exp(x[g]);
        p0[g] = sqrt(THETA / (THETA + mu[g]));
      }
      const uint64_t hs = mix64(mix64(j->seed * 256ull + S_COUNT) + c);  /* uniform01's first two mixes */
      for (int g = 0; g < j->G; ++g) {
        const double u = (double)(mix64(hs + (uint64_t)g) >> 11) * (1.0 / 9007199254740992.0);
        if (u >= p0[g]) {
          if (j->indptr) {
            j->indices[o] = g;
            j->data[o] = (float)nb_sample(mu[g], u, p0[g]);
            ++o;
          }
          ++cnt;
        }
      }
      if (!j->indptr) j->row_nnz[i] = cnt;
    }
  }
  free(x);
  return NULL;
}

/* Rows [row0, row0 + n) of the matrix.  pass 1 (indptr == NULL): row_nnz[i] = nonzeros of row
 * i.  pass 2: fill indices/data at indptr[i] (offsets relative to the first row). */
int scb_oracle_synth_rows(uint64_t seed, int64_t row0, int64_t n, int32_t G, int32_t R, const double* log_mu,
                          const double* A, const int32_t* ctype, const double* log_s, const double* U,
                          const double* B, const int64_t* indptr, int64_t* row_nnz, int32_t* indices, float* data,
                          int32_t threads) {
  job_t j = {seed, row0, n, G, R, log_mu, A, log_s, U, B, ctype, indptr, row_nnz, indices, data};
  atomic_init(&j.next, 0);
  atomic_init(&j.err, 0);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  int started = 0;
  for (int t = 0; t < threads; ++t)
    if (pthread_create(&tid[t], NULL, worker, &j) == 0) ++started;
  if (started == 0) worker(&j);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  return atomic_load(&j.err);
}
