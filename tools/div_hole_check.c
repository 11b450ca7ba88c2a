/* div_hole_check.c -- CPU check of the stage kernels' Markstein division (sgn_device.cuh
 * div_fast) in the one regime its high-word range test passes without the
 * proof covering it: quotients whose high word is zero (|a/h| < 2^-1042,
 * deep subnormal).  Same IEEE operations as the device: q0 = RN(a RN(1/h)),
 * r = fma(-q0, h, a), q = fma(r, 1/h, q0), compared with a / h.
 * Used by tests/test_division_range.py. */
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s=88172645463325252ull;
static uint64_t xr(){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
static double u01(){ return (xr()>>11)*0x1p-53; }
int main(int argc, char** argv){
  long bad=0, tested=0;
  long N = argc > 1 ? atol(argv[1]) : 200000000;
  for(long k=0;k<N;k++){
    double h = (0.25 + 4*u01()) * ((xr()&1)? 1: 0x1p40);   // h ~ [0.25, 4] or x2^40
    // a such that |a/h| < 2^-1042 (q0 high word zero), random sign, random magnitude down to 0
    double a = ldexp(u01(), -1042 - (int)(xr()%40)) * h * ((xr()&1)?-1:1);
    double rh = 1.0/h;
    double q0 = a*rh;
    uint64_t b; memcpy(&b,&q0,8);
    if ((b>>32 & 0x7fffffff) != 0) continue;   // only the hole: hi word zero
    double r = fma(-q0, h, a);
    double q = fma(r, rh, q0);
    double t = a/h;
    tested++;
    if (q != t) { bad++; if (bad < 5) printf("a=%a h=%a q=%a true=%a\n", a, h, q, t); }
  }
  printf("tested %ld mismatches %ld\n", tested, bad);
}
