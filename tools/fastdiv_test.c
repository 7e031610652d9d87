#include <stdio.h>
#include <stdint.h>
typedef struct { uint32_t d, m, s; } FastDiv;
static FastDiv mk(uint32_t d) { FastDiv f = {d, 0, 0}; if (d == 1) return f; uint32_t s = 0; while ((1ull << s) < d) s++; f.s = s; f.m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1); return f; }
static uint32_t umulhi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
static uint32_t div_(FastDiv f, uint32_t n) { if (f.d == 1) return n; uint32_t t = umulhi(n, f.m); return (t + ((n - t) >> 1)) >> (f.s - 1); }
int main() { uint32_t ds[] = {1,2,3,7,20,80,81,160,256,1000,6400,25600,65536,99991}; long bad=0;
 for (int k=0;k<14;k++){ FastDiv f=mk(ds[k]); for (uint64_t n=0;n<(1ull<<31);n+= (n<100000?1:997)) if (div_(f,(uint32_t)n)!=n/ds[k]) {bad++; if(bad<5) printf("bad d=%u n=%lu\n",ds[k],n);} }
 printf("bad=%ld\n",bad); return 0; }
