/*
 * hod_oracle.c — CPU restatement of the Overlapped Distributed Optimizer step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library; the
 * product path (paper_2312_03549_b200) never does and fails loudly without its
 * CUDA library.
 *
 * What it restates (the reference has no optimizer implementation, SPEC.md:14;
 * SURVEY.md §8c "parity unpinned" for the data path):
 *   - the gradient set being synchronised   simulator.py:268-280 (_stage_grad_bytes)
 *   - the collective semantics               simulator.py:20-23, 81-89 (reduce-scatter:
 *     rank r ends with the sum over the DP row of shard r; all-gather: every rank
 *     ends with all shards)
 *   - the optimizer the paper imports (Megatron-LM DistributedOptimizer)
 *     stated in torch.optim.AdamW algebra (decoupled weight decay):
 *         theta <- theta * (1 - lr*wd)
 *         m     <- b1*m + (1-b1)*g
 *         v     <- b2*v + (1-b2)*(g*g)
 *         theta <- theta - (lr/bc1) * (m / (sqrt(v)/sqrt(bc2) + eps))
 *     with every scalar folded in double and rounded once to fp32.  Pinned against
 *     torch.optim.AdamW (tests/golden/adamw_torch_*.npz, tests/golden/make_golden.py).
 *   - torch.nn.utils.clip_grad_norm_ coefficient min(1, c/(||g||+1e-6)).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off: no FMA contraction, so
 * every fp32 operation is the single IEEE-rounded op the CUDA kernels perform).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  float decay, b1, omb1, b2, omb2, step_size, bc2_sqrt, eps;
} oracle_consts;

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x0040u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

void oracle_fold(double lr, double b1, double b2, double eps, double wd, int64_t step,
                 oracle_consts* c) {
  const double bc1 = 1.0 - pow(b1, (double)step);
  const double bc2 = 1.0 - pow(b2, (double)step);
  c->decay = (float)(1.0 - lr * wd);
  c->b1 = (float)b1;
  c->omb1 = (float)(1.0 - b1);
  c->b2 = (float)b2;
  c->omb2 = (float)(1.0 - b2);
  c->step_size = (float)(lr / bc1);
  c->bc2_sqrt = (float)sqrt(bc2);
  c->eps = (float)eps;
}

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

void oracle_f32_to_bf16(const float* x, uint16_t* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = f32_to_bf16(x[i]);
}

void oracle_bf16_to_f32(const uint16_t* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = bf16_to_f32(x[i]);
}

/* N2 pack: bucket[off + i] = bf16(src[i] * scale); uncovered elements = 0.
 * src_is_f32 selects float* vs bf16 (uint16_t*) sources. */
void oracle_pack(const void* const* srcs, const int64_t* numels, const int64_t* offs, int n_entries,
                 int src_is_f32, float scale, uint16_t* bucket, int64_t bucket_numel) {
  memset(bucket, 0, (size_t)bucket_numel * 2);
  for (int e = 0; e < n_entries; ++e) {
    uint16_t* dst = bucket + offs[e];
    const int64_t n = numels[e];
    if (src_is_f32) {
      const float* s = (const float*)srcs[e];
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) dst[i] = f32_to_bf16(s[i] * scale);
    } else {
      const uint16_t* s = (const uint16_t*)srcs[e];
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) dst[i] = f32_to_bf16(bf16_to_f32(s[i]) * scale);
    }
  }
}

/* N3 reduce-scatter, deterministic form: out[i] = sum over ranks q = 0..d-1 (in
 * that order, fp32 accumulator starting at +0.0) of buckets[q][shard_begin + i].
 * Returned both as fp32 (out_f32, may be NULL) and bf16 (out_bf16, may be NULL). */
void oracle_rs_sum(const uint16_t* const* buckets, int d, int64_t shard_begin, int64_t n,
                   float* out_f32, uint16_t* out_bf16) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float acc = 0.0f;
    for (int q = 0; q < d; ++q) acc = acc + bf16_to_f32(buckets[q][shard_begin + i]);
    if (out_f32) out_f32[i] = acc;
    if (out_bf16) out_bf16[i] = f32_to_bf16(acc);
  }
}

/* fp64 sum over ranks, for ULP-bound checks of order-dependent reductions */
void oracle_rs_sum_f64(const uint16_t* const* buckets, int d, int64_t shard_begin, int64_t n,
                       double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int q = 0; q < d; ++q) acc += (double)bf16_to_f32(buckets[q][shard_begin + i]);
    out[i] = acc;
  }
}

static inline void adamw_elem(float* p, float* m, float* v, float g, const oracle_consts* c) {
  float pp = *p * c->decay;
  float mm = c->b1 * *m + c->omb1 * g;
  float gg = g * g;
  float vv = c->b2 * *v + c->omb2 * gg;
  float den = sqrtf(vv) / c->bc2_sqrt + c->eps;
  float upd = mm / den;
  pp = pp - c->step_size * upd;
  *p = pp;
  *m = mm;
  *v = vv;
}

/* N5 AdamW over one shard; grad is bf16 (grad_is_f32 = 0) or fp32.  coef < 0
 * means "no clipping"; otherwise g is multiplied by coef first. */
void oracle_adamw(float* master, float* m, float* v, const void* grad, int grad_is_f32,
                  uint16_t* param_out, int64_t n, const oracle_consts* c, float coef) {
  const int clip = coef >= 0.0f;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float g = grad_is_f32 ? ((const float*)grad)[i] : bf16_to_f32(((const uint16_t*)grad)[i]);
    if (clip) g = g * coef;
    adamw_elem(&master[i], &m[i], &v[i], g, c);
    if (param_out) param_out[i] = f32_to_bf16(master[i]);
  }
}

/* N4 sum of squares in fp64 (order-independent reference value) */
double oracle_sumsq_bf16(const uint16_t* x, int64_t n) {
  double acc = 0.0;
#pragma omp parallel for reduction(+ : acc) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double f = (double)bf16_to_f32(x[i]);
    acc += f * f;
  }
  return acc;
}

float oracle_clip_coef(float sumsq, float max_norm) {
  const float nrm = sqrtf(sumsq);
  const float c = max_norm / (nrm + 1e-6f);
  return c < 1.0f ? c : 1.0f;
}
