// Host-side driver for cuRAND's own Philox4x32-10 round function (library code from
// curand_philox4x32_x.h, made host-callable by overriding QUALIFIERS).  Used ONLY by
// tests/test_oracle_sampling.py as an independent pin of oracle/ring_oracle.c's Philox.
// Usage: philox_curand_host <key_lo> <key_hi> then lines "c0 c1 c2 c3" on stdin;
// prints "x0 x1 x2 x3" per line.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    uint2 key = make_uint2((unsigned)strtoul(argv[1], 0, 0), (unsigned)strtoul(argv[2], 0, 0));
    unsigned c0, c1, c2, c3;
    while (scanf("%u %u %u %u", &c0, &c1, &c2, &c3) == 4) {
        uint4 c = make_uint4(c0, c1, c2, c3);
        uint4 r = curand_Philox4x32_10(c, key);
        printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
    }
    return 0;
}
