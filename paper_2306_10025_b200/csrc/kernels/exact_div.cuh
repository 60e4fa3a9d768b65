// Correctly rounded division by a divisor whose reciprocal is reused.
//
// y = RN(1/b) (one IEEE division per divisor, computed once), then
// q0 = RN(a*y) and two Markstein corrections q <- RN(q + RN(a - q*b)*y), the
// remainders formed exactly by FMA.  After the first correction q is within
// one ulp of a/b; the second then yields RN(a/b) (Markstein's theorem: y the
// correctly rounded reciprocal, q within an ulp of the quotient).  The result
// is therefore bitwise __ddiv_rn(a, b) for normal operands and quotients;
// zero, subnormal-range and near-overflow cases take the IEEE division
// itself.  Five FP64 instructions instead of the division subroutine
// (reciprocal seed, Newton steps, range checks).  Checked against __ddiv_rn
// on 2^27 random pairs per exponent regime by tests/test_exact_div.py.
#pragma once

namespace pdb::k {

__device__ __forceinline__ double div_rn_recip(double a, double b, double y) {
  double q = __dmul_rn(a, y);
  double r = __fma_rn(-q, b, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-q, b, a);
  q = __fma_rn(r, y, q);
  // keep a, b, q (hence y and every remainder) far from underflow / overflow
  const double aa = fabs(a), ab = fabs(b), aq = fabs(q);
  if (!(aa > 0x1.0p-900 && aa < 0x1.0p+900 && ab > 0x1.0p-900 && ab < 0x1.0p+900 && aq > 0x1.0p-900 &&
        aq < 0x1.0p+900))
    q = __ddiv_rn(a, b);
  return q;
}

}  // namespace pdb::k
