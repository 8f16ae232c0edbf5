/* absim_models.h — IEEE-only math shared by the GPU kernels, the C oracle
 * (oracle/absim_oracle.c) and the reference-API harness (oracle/ref_harness.cpp).
 *
 * Everything here uses only + - * / sqrt and integer ops, evaluated in the
 * order written (GPU TUs are compiled with --fmad=false, host TUs with
 * -ffp-contract=off), so every caller gets the same bits. libm
 * transcendentals (cos/sin/cbrt/log) are NOT bit-portable between glibc and
 * CUDA and therefore never appear on a decision path.
 *
 * Reference anchors:
 *   abs_rng_word      restates random.hpp:13-28 (splitmix64 finaliser x2)
 *   abs_u01           restates random.hpp:38-40 (next_double)
 *   BASELINE.json configs[1..4] define the synthetic model behaviours below
 *   (they are not in the reference; SURVEY.md §8d fixes their semantics).
 */
#ifndef ABSIM_MODELS_H
#define ABSIM_MODELS_H

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define ABS_HD __host__ __device__ __forceinline__
#else
#define ABS_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* random.hpp:13-28 */
ABS_HD uint64_t abs_rng_word(uint64_t seed, uint64_t stream, uint64_t counter) {
  uint64_t x = seed;
  x += 0x9e3779b97f4a7c15ull * (stream + 0x632be59bd9b4e019ull);
  x += 0xbf58476d1ce4e5b9ull * (counter + 1);
  for (int i = 0; i < 2; ++i) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
  }
  return x;
}

/* random.hpp:38-40: uniform in [0, 1) */
ABS_HD double abs_u01(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }

/* Cube root by bit-trick seed + 6 Newton steps; +,-,*,/ only. a > 0. */
ABS_HD double abs_cbrt_ieee(double a) {
  union { double d; uint64_t u; } v;
  v.d = a;
  v.u = v.u / 3u + 0x2A9F7893782DA1CEull;
  double x = v.d;
  for (int i = 0; i < 6; ++i) {
    const double x2 = x * x;
    x = x - (x2 * x - a) / (3.0 * x2);
  }
  return x;
}

#define ABS_PI 3.14159265358979323846

/* Sphere volume <-> diameter (config 2). */
ABS_HD double abs_volume_of_diameter(double d) { return ABS_PI / 6.0 * (d * d * d); }
ABS_HD double abs_diameter_of_volume(double v) { return abs_cbrt_ieee((6.0 * v) / ABS_PI); }

/* Rejection-sampled unit vector from the counter hash: draws points of
 * [-1,1)^3 from (seed, stream, base + 3*attempt + k) until one lands in the
 * open unit ball (excluding the origin), then normalises. Replaces the
 * cos/sin path of random.hpp:47-52, which is not bit-portable. */
ABS_HD void abs_unit_vector(uint64_t seed, uint64_t stream, uint64_t base,
                            double out[3]) {
  for (uint64_t attempt = 0; attempt < 64; ++attempt) {
    const double x = 2.0 * abs_u01(abs_rng_word(seed, stream, base + 3 * attempt)) - 1.0;
    const double y = 2.0 * abs_u01(abs_rng_word(seed, stream, base + 3 * attempt + 1)) - 1.0;
    const double z = 2.0 * abs_u01(abs_rng_word(seed, stream, base + 3 * attempt + 2)) - 1.0;
    const double s = (x * x + y * y) + z * z;
    if (s > 0.0 && s <= 1.0) {
      const double n = sqrt(s);
      out[0] = x / n;
      out[1] = y / n;
      out[2] = z / n;
      return;
    }
  }
  out[0] = 1.0;
  out[1] = 0.0;
  out[2] = 0.0;
}

/* ---- config 2: volume growth + division (BASELINE configs[1]) ----------
 * Per iteration, for an agent with volume V (behaviour state):
 *   V += rate
 *   if V > v_divide:  V *= 0.5; daughter at pos + dir * (0.5 * diameter)
 *                     with volume V (dir = abs_unit_vector(seed, uid,
 *                     iteration << 8)); daughter uid = next uid in parent
 *                     storage (= parent uid) order
 *   grow(diameter_of_volume(V) - diameter)   [deferred, agent.hpp:40]
 */
#define ABS_RNG_DIVISION_BASE(it) ((uint64_t)(it) << 8)
/* ABS_MODEL_GROW_DIVIDE_DIE: the per-iteration removal draw (AgentContext::remove_self) */
#define ABS_RNG_DEATH(it) (((uint64_t)(it) << 8) | 0xfdull)

/* ---- config 3: outward drive of the outer shells (BASELINE configs[2]) --
 * delta = unit(p - centre) * (speed_max * u), u = abs_u01(rng_word(seed,
 * uid, (iteration << 8) | 0xff)); translate(delta) [agent.hpp:39]. */
#define ABS_RNG_DRIVE_COUNTER(it) (((uint64_t)(it) << 8) | 0xffull)

ABS_HD void abs_drive_delta(double px, double py, double pz, double cx, double cy,
                            double cz, double speed_max, uint64_t seed, uint64_t uid,
                            uint64_t iteration, double out[3]) {
  const double dx = px - cx, dy = py - cy, dz = pz - cz;
  const double n = sqrt((dx * dx + dy * dy) + dz * dz);
  const double speed = speed_max * abs_u01(abs_rng_word(seed, uid, ABS_RNG_DRIVE_COUNTER(iteration)));
  if (n > 0.0) {
    out[0] = dx / n * speed;
    out[1] = dy / n * speed;
    out[2] = dz / n * speed;
  } else {
    out[0] = out[1] = out[2] = 0.0;
  }
}

/* ---- config 5: SIR epidemic on a periodic cube (BASELINE configs[4]) ---
 * The reference has no periodic boundaries; this model is
 * defined here and checked between the C oracle and the kernels only.
 * Per iteration, from the START-of-iteration states (double-buffered, so the
 * agent loop order cannot leak into results):
 *   k = #neighbours b != a in state I with minimum-image distance^2 <= r^2
 *       (dx wrapped once into [-L/2, L/2], d2 = ((dx^2 + dy^2) + dz^2))
 *   S -> I  if k > 0 and rng_word(seed, uid, SIR_INFECT(it)) < thr(k)
 *           thr(k) = (u64)((1 - (1 - p)^k) * 2^64), (1-p)^k by repeated *
 *   I -> R  if it - t_infected >= recovery
 *   walk:   p += unit_vector(seed, uid, SIR_WALK(it)) * step, wrapped into [0, L)
 * Initial state: I (t_infected = 0) iff u01(rng_word(seed, uid, 20)) < 0.01. */
#define ABS_SIR_S 0
#define ABS_SIR_I 1
#define ABS_SIR_R 2
#define ABS_RNG_SIR_INFECT(it) (((uint64_t)(it) << 8) | 0xfeull)
#define ABS_RNG_SIR_WALK(it) ((uint64_t)(it) << 8)
#define ABS_RNG_SIR_INIT 20ull

ABS_HD uint64_t abs_sir_threshold(double p, unsigned int k) {
  double q = 1.0;
  for (unsigned int i = 0; i < k; ++i) q = q * (1.0 - p);
  const double v = (1.0 - q) * 18446744073709551616.0;
  return v >= 18446744073709551615.0 ? 0xFFFFFFFFFFFFFFFFull : (uint64_t)v;
}

ABS_HD double abs_min_image(double d, double L) {
  if (d > 0.5 * L) return d - L;
  if (d < -0.5 * L) return d + L;
  return d;
}

ABS_HD double abs_wrap(double v, double L) {
  if (v >= L) return v - L;
  if (v < 0.0) return v + L;
  return v;
}

#ifdef __cplusplus
}
#endif

#endif /* ABSIM_MODELS_H */
