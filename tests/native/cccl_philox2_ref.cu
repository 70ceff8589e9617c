// Test helper (not product code): prints libcudacxx's own
// cuda::std::philox_engine (the C++26 std::philox_engine, CCCL) instantiated
// as Philox2x32-10 -- word size 32, n = 2, 10 rounds, multiplier 0xD256D193,
// round constant 0x9E3779B9 (Random123's philox2x32 constants, Salmon et al.
// SC'11 Table 2) -- for (ctr, key) lines "c0 c1 k" read from stdin.  The
// library reference the oracle's Philox2x32-10 is checked against (DESIGN.md
// §R3).  Built with -I <flashinfer>/data/cccl/libcudacxx/include.
#include <cuda/std/__random/philox_engine.h>
#include <cstdio>
using P2 = cuda::std::philox_engine<cuda::std::uint_fast32_t, 32, 2, 10, 0xD256D193, 0x9E3779B9>;
int main() {
  unsigned c0, c1, k;
  while (scanf("%u %u %u", &c0, &c1, &k) == 3) {
    P2 e(k);
    e.set_counter({c1, c0});      // counter[0] is the most significant word
    const unsigned y0 = (unsigned)e(), y1 = (unsigned)e();
    printf("%u %u\n", y0, y1);
  }
  return 0;
}
