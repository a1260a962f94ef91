// Dev tool: depth of the greedy-by-orig_id colouring dependency DAG on a
// jittered row-major grid with the meshgen diagonal hash (C4: n = 4096).
// usage: gcc -O2 -o /tmp/jp_depth tools/jp_depth.c && /tmp/jp_depth 4096
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
// depth of the greedy-by-id dependency DAG of a triangulated grid with random diagonals
static uint64_t sm(uint64_t z){z+=0x9E3779B97F4A7C15ull;z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
int main(int argc,char**argv){int n=atoi(argv[1]);int64_t V=(int64_t)n*n;int*dep=calloc(V,sizeof(int));
 // neighbours with lower id: (i-1,j), (i,j-1), and the diagonal neighbour in row j-1 depending on cell diagonals
 int maxd=0;
 for(int j=0;j<n;j++)for(int i=0;i<n;i++){int64_t v=(int64_t)j*n+i;
  if(i==0||j==0||i==n-1||j==n-1){dep[v]=0;continue;} // boundary fixed (not in DAG)
  int d=0;
  #define F(ii,jj) { int64_t u=(int64_t)(jj)*n+(ii); if(!((ii)==0||(jj)==0||(ii)==n-1||(jj)==n-1)) if(dep[u]+1>d) d=dep[u]+1; }
  F(i-1,j); F(i,j-1);
  // cell (i-1,j-1): b=0 diag v00-v11 => (i-1,j-1)~(i,j); b=1 diag v10-v01 => (i,j-1)~(i-1,j)
  uint64_t seed=1606; uint64_t h1=sm(sm(seed+3)+(uint64_t)((j-1)*(n-1)+(i-1)));
  if(!(h1&1)) F(i-1,j-1);
  // cell (i,j-1): b=1 diag v10-v01 => (i+1,j-1)~(i,j)
  uint64_t h2=sm(sm(seed+3)+(uint64_t)((j-1)*(n-1)+i));
  if(h2&1) F(i+1,j-1);
  if(d==0) d=1; dep[v]=d; if(d>maxd)maxd=d;}
 printf("n=%d depth=%d (nx+2ny=%d)\n",n,maxd,3*n);return 0;}
