/* Floor of the host cache calls without Python: emm_cache_match_prefix +
 * emm_cache_release from C in a loop (a 180-key miss at the root, and a
 * 180-key full-edge hit).  Build: gcc -O2 -Iinclude tools/cache_c_floor.c
 *   -Lpaper_2507_10069_b200 -lemm -Wl,-rpath,$PWD/paper_2507_10069_b200 */
#include <stdio.h>
#include <stdint.h>
#include <time.h>
#include "emm.h"
static double now_s(void){struct timespec t; clock_gettime(CLOCK_MONOTONIC,&t); return t.tv_sec+1e-9*t.tv_nsec;}
int main(void){
  emm_cache* c; emm_cache_create(1000000, 0.2, &c);
  uint64_t k[180]; int64_t w[180];
  for(int i=0;i<180;i++){k[i]=1000+i; w[i]=1;}
  int64_t added; emm_cache_insert_prefix(c,k,w,180,0.0,&added);
  uint64_t k2[180]; for(int i=0;i<180;i++) k2[i]=5000+i;
  int N=2000000; int64_t m; uint64_t h;
  for(int rep=0;rep<3;rep++){
    double t0=now_s();
    for(int i=0;i<N;i++){ emm_cache_match_prefix(c,k2,w,180,1.0,&m,&h); emm_cache_release(c,h);}
    double t1=now_s();
    for(int i=0;i<N;i++){ emm_cache_match_prefix(c,k,w,180,1.0,&m,&h); emm_cache_release(c,h);}
    double t2=now_s();
    printf("miss %.3f us  hit180 %.3f us (m=%ld)\n",(t1-t0)/N*1e6,(t2-t1)/N*1e6,(long)m);
  }
  return 0;
}
