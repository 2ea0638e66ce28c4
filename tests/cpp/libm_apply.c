/* The host's libm (the one the reference links) over an array: the expected
 * values for the device evaluation of the glibc exp/log port. */
#include <math.h>
#include <stdint.h>
extern "C" void libm_apply(int fn, const double* in, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = fn == 0 ? exp(in[i]) : log(in[i]);
}
