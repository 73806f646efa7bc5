// enum32.cu -- the enumeration kernels with a 32-bit accumulator word (count_into32 /
// finalize32): enum.cu compiled again with VDMC_ACC32 = 1.  The host uses it only when every
// (vertex, class) count fits 32 bits: 6 * maxdeg^3 < 2^32 for k = 4 (each connected 4-set through
// v is reached by choosing, in turn, a neighbour of the growing set: <= D * 2D * 3D ways), and
// 2 * maxdeg^2 < 2^32 for k = 3.  Results are identical (tests compare both paths).
#define VDMC_ACC32 1
#include "enum.cu"
