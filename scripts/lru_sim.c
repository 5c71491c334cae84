// LRU simulation of the C2 SpMM C-row gathers (measurement aid):
// fully associative LRU over 256-byte rows, the R-MAT scale-24 column sequence
// (rp.bin / crd.bin written from bench.rmat_csr), single pass and hot/cold split.
//   gcc -O2 -o /tmp/lru_sim scripts/lru_sim.c && (cd <dir with rp.bin, crd.bin> && /tmp/lru_sim)
// LRU simulation of C-row gathers (256 B rows) for SpMM over the R-MAT CSR.
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
static int32_t *prv,*nxt; static char* in; static int64_t head=-1,tail=-1,sz=0,cap;
static void unlink_(int32_t c){ if(prv[c]>=0) nxt[prv[c]]=nxt[c]; else head=nxt[c]; if(nxt[c]>=0) prv[nxt[c]]=prv[c]; else tail=prv[c]; }
static void push_front(int32_t c){ prv[c]=-1; nxt[c]=head; if(head>=0) prv[head]=c; head=c; if(tail<0) tail=c; }
static int64_t access_(int32_t c){ if(in[c]){ unlink_(c); push_front(c); return 0;} if(sz==cap){ int32_t t=tail; unlink_(t); in[t]=0; sz--; } push_front(c); in[c]=1; sz++; return 1; }
static void reset(int64_t n){ memset(in,0,n); head=tail=-1; sz=0; }
int main(int argc,char**argv){
  int64_t n=1<<24; FILE*f=fopen("rp.bin","rb"); int64_t*rp=malloc(8*(n+1)); fread(rp,8,n+1,f); fclose(f);
  int64_t nnz=rp[n]; int32_t*crd=malloc(4*nnz); f=fopen("crd.bin","rb"); fread(crd,4,nnz,f); fclose(f);
  prv=malloc(4*n); nxt=malloc(4*n); in=malloc(n);
  int32_t*cnt=calloc(n,4); for(int64_t q=0;q<nnz;q++) cnt[crd[q]]++;
  // sorted counts desc
  int32_t*sc=malloc(4*n); memcpy(sc,cnt,4*n);
  int cmp(const void*a,const void*b){ return *(int32_t*)b-*(int32_t*)a; }
  qsort(sc,n,4,cmp);
  int64_t distinct=0; for(int64_t i=0;i<n;i++) if(cnt[i]) distinct++;
  printf("nnz %ld distinct cols %ld (%.2f GB)\n",nnz,distinct,distinct*256/1e9);
  // cumulative access fraction of top-k columns
  int64_t ks[]={50000,100000,160000,240000,320000,480000,640000,1000000,2000000};
  int64_t acc=0; int ki=0;
  for(int64_t i=0;i<n && ki<9;i++){ acc+=sc[i]; if(i+1==ks[ki]){ printf("top %ld cols (%.0f MB): %.3f of accesses, thr count %d\n",ks[ki],ks[ki]*256/1e6,(double)acc/nnz,sc[i]); ki++; } }
  double mbs[]={40,60,80,100,126};
  for(int m=0;m<5;m++){ cap=(int64_t)(mbs[m]*1e6/256); reset(n); int64_t miss=0; for(int64_t q=0;q<nnz;q++) miss+=access_(crd[q]); printf("single pass LRU %3.0f MB: miss %.3f -> %.2f GB\n",mbs[m],(double)miss/nnz,miss*256/1e9); }
  // hot/cold
  int64_t Hs[]={120000,160000,240000,320000};
  double cmb[]={40,60,80};
  for(int h=0;h<4;h++){ int64_t H=Hs[h]; int32_t thr=sc[H-1];
    // hot = cnt>=thr (ties may exceed H slightly)
    int64_t hotacc=0,hotdistinct=0; for(int64_t i=0;i<n;i++) if(cnt[i]>=thr){hotdistinct++;}
    int64_t both=0,hotonly=0,coldonly=0;
    for(int64_t r=0;r<n;r++){ int hh=0,cc=0; for(int64_t q=rp[r];q<rp[r+1];q++){ if(cnt[crd[q]]>=thr) hh=1; else cc=1;} if(hh&&cc) both++; else if(hh) hotonly++; else if(cc) coldonly++; }
    for(int64_t q=0;q<nnz;q++) if(cnt[crd[q]]>=thr) hotacc++;
    printf("hot H=%ld thr=%d distinct %ld (%.0f MB): hot acc %.3f, rows both %ld hotonly %ld coldonly %ld\n",H,thr,hotdistinct,hotdistinct*256/1e6,(double)hotacc/nnz,both,hotonly,coldonly);
    for(int m=0;m<3;m++){ cap=(int64_t)(cmb[m]*1e6/256); reset(n); int64_t miss=0; for(int64_t q=0;q<nnz;q++) if(cnt[crd[q]]<thr) miss+=access_(crd[q]);
      printf("   cold pass LRU %3.0f MB: miss %.2f GB; total C %.2f GB; +partials(512B x both) %.2f GB\n",cmb[m],miss*256/1e9,(miss+hotdistinct)*256/1e9,both*512/1e9); }
  }
}
