// Test helper (not product code): prints cuRAND's own curand_Philox4x32_10
// (host-callable here by widening its QUALIFIERS) for (ctr, key) pairs read
// from stdin, one "c0 c1 c2 c3 k0 k1" line each -- the library reference the
// oracle's Philox is checked against (SURVEY §8(c.8) "cuRAND cross-check").
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
  unsigned c[4], k[2];
  while (scanf("%u %u %u %u %u %u", &c[0], &c[1], &c[2], &c[3], &k[0], &k[1]) == 6) {
    uint4 r = curand_Philox4x32_10(make_uint4(c[0], c[1], c[2], c[3]), make_uint2(k[0], k[1]));
    printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
