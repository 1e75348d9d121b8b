/* np_exp64.c -- TEST INFRASTRUCTURE (checker only; the product never links it).
 *
 * C restatement of numpy's float64 exp on x86-64 hosts with AVX-512, where
 * numpy (2.x) dispatches np.exp(float64) to Intel SVML's __svml_exp8_ha
 * (vendored in numpy; numpy/_core/_multiarray_umath*.so, constants in
 * __svml_dexp_ha_data_internal_avx512).  Reconstructed from that machine code
 * (objdump) and its constant tables; it matches np.exp bit for bit on every
 * float32 input in (-707.70, 0] (tests/test_np_exp64.py samples it;
 * scripts/check_np_exp64.py runs all 1.144e9).  The reference's softmax calls
 * np.exp on float64 (router.py:65, router.py:82), so the router's device port
 * (csrc/router.cuh np_exp64) follows this restatement operation by operation.
 * |x| >= 707.70 takes SVML's separate rare path, not restated here.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#pragma STDC FENV_ACCESS ON

static const uint64_t kTop[16] = {
    0x3ff0000000000000ull, 0x3ff0b5586cf9890full, 0x3ff172b83c7d517bull, 0x3ff2387a6e756238ull,
    0x3ff306fe0a31b715ull, 0x3ff3dea64c123422ull, 0x3ff4bfdad5362a27ull, 0x3ff5ab07dd485429ull,
    0x3ff6a09e667f3bcdull, 0x3ff7a11473eb0187ull, 0x3ff8ace5422aa0dbull, 0x3ff9c49182a3f090ull,
    0x3ffae89f995ad3adull, 0x3ffc199bdd85529cull, 0x3ffd5818dcfba487ull, 0x3ffea4afa2a490daull};
static const uint64_t kTail[16] = {
    0x0000000000000000ull, 0x3c979aa65d837b6dull, 0xbc801b15eaa59348ull, 0x3c968efde3a8a894ull,
    0x3c834d754db0abb6ull, 0x3c859f48a72a4c6dull, 0x3c7690cebb7aafb0ull, 0x3c9063e1e21c5409ull,
    0xbc93b3efbf5e2228ull, 0xbc7b32dcb94da51dull, 0x3c8db72fc1f0eab4ull, 0x3c71affc2b91ce27ull,
    0x3c8c1a7792cb3387ull, 0x3c736eae30af0cb3ull, 0x3c74a385a63d07a7ull, 0xbc8ff7128fd391f0ull};

static double bd(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t bu(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

double np_exp64(double x) {
  const double inv_ln2 = bd(0x3ff71547652b82feull), shifter = bd(0x42f8000000003ff0ull);
  const double ln2_hi = bd(0x3fe62e42fefa39efull), ln2_lo = bd(0x3c7abc9e3b39803full);
  const double c6 = bd(0x3f57411836940c04ull), c5 = bd(0x3f81101cbbc265c0ull), c4 = bd(0x3fa55557242d68feull);
  const double c3 = bd(0x3fc5555553939732ull), c2 = bd(0x3fe000000000d008ull), c1 = bd(0x3fefffffffffff70ull);
  fesetround(FE_TOWARDZERO);
  volatile double t = fma(x, inv_ln2, shifter); /* vfmadd213pd {rz-sae} */
  fesetround(FE_TONEAREST);
  const double n = t - shifter;
  const int j = (int)(bu(t) & 15);
  double r = fma(-n, ln2_hi, x);
  r = fma(-ln2_lo, n, r);
  r = bd(bu(r) & 0xbfffffffffffffffull);
  const double r2 = r * r;
  double a = fma(c6, r, c5);
  const double b = fma(c4, r, c3);
  const double c = fma(c2, r, c1);
  a = fma(r2, a, b);
  a = fma(r2, a, c);
  const double p = fma(a, r, bd(kTail[j]));
  const double res = fma(bd(kTop[j]), p, bd(kTop[j]));
  return ldexp(res, (int)floor(n)); /* vscalefpd */
}

void np_exp64_array(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = np_exp64(x[i]);
}
