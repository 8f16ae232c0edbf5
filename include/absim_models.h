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

#ifdef __cplusplus
}
#endif

#endif /* ABSIM_MODELS_H */
