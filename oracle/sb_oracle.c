/* CPU oracle for the stick-breaking attention hot path.
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  A plain-C restatement of the
 * reference's tiled NumPy kernels (/root/reference/pkg/src/sbattn/blocked.py:
 * blocked_forward :129-206, blocked_backward_twophase :299-392) and of its
 * scalar numerics (numerics.py:19, :33-47), in float64 and float32.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it, and only as the checker or the timed CPU
 * baseline.  Parity is pinned against golden vectors produced by the
 * reference itself (oracle/gen_golden.py -> tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define REAL double
#define SFX f64
#define EXP exp
#define LOG1P log1p
#include "sb_oracle_body.h"
#undef REAL
#undef SFX
#undef EXP
#undef LOG1P

#define REAL float
#define SFX f32
#define EXP expf
#define LOG1P log1pf
#include "sb_oracle_body.h"
#undef REAL
#undef SFX
#undef EXP
#undef LOG1P

int sbo_version(void) { return 1; }
