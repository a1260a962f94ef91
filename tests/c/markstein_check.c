/* Brute-force check of the division the GZ sweep kernel uses for Eq. 1's
 * x / d: with r = RN(1/d), q = RN(x r), e = fma(-q, d, x),
 * fma(e, r, q) equals the correctly rounded x / d for every normal x away
 * from the exponent range's ends (the kernel's gz_div_ok window) and
 * d = 1..64.  Random operands plus operands built to land next to rounding
 * midpoints of the quotient.  Prints "tested N mismatches M"; exit status 1 on
 * any mismatch.  Compiled with -ffp-contract=off so x/d and x*r are single
 * IEEE operations. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>
static uint64_t s=88172645463325252ull;
static inline uint64_t xr(void){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
static inline double bits(uint64_t u){double d;memcpy(&d,&u,8);return d;}
static inline uint64_t ub(double d){uint64_t u;memcpy(&u,&d,8);return u;}
int main(int argc, char** argv){
  long bad=0,tot=0;
  const long per = argc > 1 ? atol(argv[1]) : 4000000;
  for(int d=1; d<=64; ++d){
    double dd=d, r=1.0/dd;
    for(long k=0;k<per;++k){
      double x;
      int mode=k&3;
      if(mode==0){ x=bits((xr()&0x800FFFFFFFFFFFFFull)|((uint64_t)(1023-40+(xr()%80))<<52)); }
      else if(mode==1){ // near midpoint: m = (q + half ulp), x = m*d rounded +- few ulps
        double q=bits((xr()&0x000FFFFFFFFFFFFFull)|((uint64_t)(1023-20+(xr()%40))<<52));
        double m=q+ldexp(1.0, ilogb(q)-53);
        x=m*dd; int64_t a=(int64_t)(xr()%9)-4; x=bits(ub(x)+a);
      } else if(mode==2){ // sums of neighbours in [0,1) typical grid coords
        x=0; for(int i=0;i<d && i<8;++i) x+= (xr()>>11)*0x1.0p-53; x=bits(ub(x)+(int64_t)(xr()%5)-2);
      } else { // x = integer multiple of small ulps * d +- ulp
        double q=(double)(xr()>>11)*0x1.0p-40; x=q*dd; x=bits(ub(x)+(int64_t)(xr()%3)-1);
      }
      if(!(fabs(x)>=0x1p-959 && fabs(x)<=0x1.fffffffffffffp1023)) continue;
      double q=x*r, e=fma(-q,dd,x), q2=fma(e,r,q);
      double want=x/dd; ++tot;
      if(ub(q2)!=ub(want)){ if(bad<10) printf("d=%d x=%a got %a want %a\n",d,x,q2,want); ++bad;}
    }
  }
  printf("tested %ld mismatches %ld\n",tot,bad);
  return bad != 0;
}
