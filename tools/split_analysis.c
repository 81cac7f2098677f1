/* Split analysis (development tool): for the S_{2,8} genomes whose run 0 is UNBOUND and that the
 * trivial-freedom proof cannot clear, how many pops would executing ALL their later runs in parallel
 * lanes waste against stopping at the first TRIVIAL one, per run-0-length threshold, and how many of
 * the long genomes (>= 1024 executed pops, the small-launch floor) each threshold catches.
 *   gcc -O3 -fopenmp -Wno-unused-function -o /tmp/split_analysis tools/split_analysis.c && /tmp/split_analysis
 */
/* Work-elimination analysis for the enumeration kernel (development tool, not
 * product code): runs the oracle's restatement of _k:96-381 over an index range
 * and attributes movelist pops to the categories an exact cut-off could skip.
 *
 *   gcc -O3 -fopenmp -o /tmp/work_analysis tools/work_analysis.c && /tmp/work_analysis s28
 *
 * Categories (per genome, runs in reference order up to kmax, stopping at TRIVIAL):
 *   all         every pop
 *   one_mer     genomes whose seed faces bond no label of the genome (1x1 DET at every k)
 *   after_unb   pops in runs after the first UNBOUND run
 *     .final_unb  ... of genomes that never go TRIVIAL (skippable with a proof)
 *     .tfree      ... of those, captured by the current trivial-freedom proof
 *     .line       ... of those, genomes whose proof variants below hold
 */
#include "../oracle/tv_oracle.c"
#include <stdio.h>
#include <string.h>

static int partner(int x) { return x ? (((x - 1) ^ 1) + 1) : 15; }

/* scalar restatement of CandSwar::trivial_free (tv_fast.cuh), strict rule */
static int trivial_free_scalar(const uint8_t *E, int a, int strict) {
    const int NC = 4 * a;
    int inR[12] = {0};
    inR[0] = 1;
    for (int changed = 1; changed;) {
        changed = 0;
        for (int c2 = 0; c2 < NC; c2++) {
            if (inR[c2]) continue;
            for (int c = 0; c < NC && !inR[c2]; c++) {
                if (!inR[c]) continue;
                for (int k = 0; k < 4; k++)
                    if (orc_bonds(E[c2 * 4 + k], E[c * 4 + ((k + 2) & 3)])) { inR[c2] = 1; changed = 1; break; }
            }
        }
    }
    uint32_t S[4] = {0, 0, 0, 0};
    for (int c = 0; c < NC; c++)
        if (inR[c])
            for (int k = 0; k < 4; k++) S[k] |= 1u << E[c * 4 + ((k + 2) & 3)];
    for (int c1 = 0; c1 < NC; c1++)
        for (int c2 = c1 + 1; c2 < NC; c2++) {
            if (memcmp(E + c1 * 4, E + c2 * 4, 4) == 0) continue;
            int bond1[4], bond2[4], ok = 0;
            for (int k = 0; k < 4; k++) {
                int p1 = partner(E[c1 * 4 + k]), p2 = partner(E[c2 * 4 + k]);
                bond1[k] = p1 < 15 && ((S[k] >> p1) & 1);
                bond2[k] = p2 < 15 && ((S[k] >> p2) & 1);
            }
            for (int k = 0; k < 4; k++)
                if (bond1[k] && E[c1 * 4 + k] == E[c2 * 4 + k]) ok = 1;
            for (int k1 = 0; k1 < 4 && !ok; k1++)
                for (int k2 = 0; k2 < 4 && !ok; k2++) {
                    if (k1 == k2 || !bond1[k1] || !bond2[k2]) continue;
                    int t2 = !strict || E[c2 * 4 + k1] == 0 || E[c2 * 4 + k1] == E[c1 * 4 + k1];
                    int t1 = !strict || E[c1 * 4 + k2] == 0 || E[c1 * 4 + k2] == E[c2 * 4 + k2];
                    if (t1 && t2) ok = 1;
                }
            if (ok) return 0;
        }
    return 1;
}


/* Refined proof (v2): a placed tile never shows a label toward a popped cell through a
 * side it bonded at placement (that neighbour is occupied, cells never empty again), so
 * S[k] only collects face (k+2)&3 of candidates placeable with some bonded side other
 * than (k+2)&3; the seed (no bonded side) shows all four faces.  Fixpoint:
 * S -> bond[c][k] = partner(E_c[k]) in S[k] -> S. */
static int trivial_free_v2(const uint8_t *E, int a, int strict) {
    const int NC = 4 * a;
    uint32_t S[4], bond[12];
    for (int k = 0; k < 4; k++) S[k] = 1u << E[0 * 4 + ((k + 2) & 3)];
    for (;;) {
        for (int c = 0; c < NC; c++) {
            bond[c] = 0;
            for (int k = 0; k < 4; k++) {
                int p = partner(E[c * 4 + k]);
                if (p < 15 && ((S[k] >> p) & 1)) bond[c] |= 1u << k;
            }
        }
        uint32_t S2[4];
        for (int k = 0; k < 4; k++) S2[k] = S[k];
        for (int c = 0; c < NC; c++)
            for (int k = 0; k < 4; k++) {
                int f = (k + 2) & 3;  /* c at side k of the popped cell shows its face f */
                if (bond[c] & ~(1u << f)) S2[k] |= 1u << E[c * 4 + f];
            }
        if (!memcmp(S, S2, sizeof S)) break;
        memcpy(S, S2, sizeof S);
    }
    for (int c1 = 0; c1 < NC; c1++)
        for (int c2 = c1 + 1; c2 < NC; c2++) {
            if (memcmp(E + c1 * 4, E + c2 * 4, 4) == 0) continue;
            int ok = 0;
            for (int k = 0; k < 4; k++)
                if (((bond[c1] >> k) & 1) && E[c1 * 4 + k] == E[c2 * 4 + k]) ok = 1;
            for (int k1 = 0; k1 < 4 && !ok; k1++)
                for (int k2 = 0; k2 < 4 && !ok; k2++) {
                    if (k1 == k2 || !((bond[c1] >> k1) & 1) || !((bond[c2] >> k2) & 1)) continue;
                    int t2 = !strict || E[c2 * 4 + k1] == 0 || E[c2 * 4 + k1] == E[c1 * 4 + k1];
                    int t1 = !strict || E[c1 * 4 + k2] == 0 || E[c1 * 4 + k2] == E[c2 * 4 + k2];
                    if (t1 && t2) ok = 1;
                }
            if (ok) return 0;
        }
    return 1;
}


/* Locally-forced assembly (the run-0 shortcut): for the BOUNDED assembly alpha on the scratch grid,
 * every tile's face toward each neighbour cell q may be bonded only by candidates with q's code in
 * alpha (q occupied), or by none (q empty).  Then every run, whatever its order, produces alpha. */
static int forced(const uint8_t *E, int a, int d, const orc_scratch *S, int n_placed) {
    const int NC = 4 * a;
    const int off[4] = {-d, 1, d, -1};
    for (int i = 0; i < n_placed; i++) {
        int cell = S->placed[i], v = S->grid[cell];
        for (int j = 0; j < 4; j++) {
            int q = cell + off[j], lab = E[v * 4 + j], vq = S->grid[q];
            for (int c = 0; c < NC; c++) {
                if (!orc_bonds(E[c * 4 + ((j + 2) & 3)], lab)) continue;
                if (vq < 0) return 0;
                if (memcmp(E + c * 4, E + vq * 4, 4) != 0) return 0;
            }
        }
    }
    return 1;
}

static int one_mer(const uint8_t *E, int a) {
    /* seed = candidate 0; any candidate bonding a seed face? (strict conflicts only remove hits) */
    for (int k = 0; k < 4; k++) {
        int x = E[k];
        if (!x) continue;
        for (int c = 0; c < 4 * a; c++)
            if (orc_bonds(E[c * 4 + ((k + 2) & 3)], x)) return 0;
    }
    return 1;
}



int main(void) {
    int a=2,bpl=3,d=19,kmax=8; int64_t free_pos[24]; for(int j=0;j<24;j++) free_pos[j]=23-j;
    const int NT=6; const int TH[6]={60,80,100,130,160,200};
    uint64_t sel[6]={0},seqp[6]={0},parp[6]={0},cap[6]={0},longg=0;
#pragma omp parallel reduction(+:sel[:6],seqp[:6],parp[:6],cap[:6],longg)
    {
    orc_scratch S; orc_scratch_alloc(&S,d); uint8_t bits[64],E[12*16];
#pragma omp for schedule(dynamic,4096)
    for (int64_t idx=0; idx<(1<<24); idx++) {
        orc_decode_edges(idx,a,bpl,NULL,NULL,0,free_pos,24,bits,E);
        orc_counts C; memset(&C,0,sizeof C);
        orc_run R0=orc_assemble(E,a,d,1,0,idx,0,&S,&C); orc_cleanup(&S,&R0);
        if (R0.outcome!=ORC_RUN_UNBOUND) continue;
        if (trivial_free_v2(E,a,1)) continue;
        uint64_t p0=C.pops, seq=0, par=0; int trivial=0;
        for (int run=1; run<kmax; run++) {
            orc_counts C2; memset(&C2,0,sizeof C2);
            orc_run R=orc_assemble(E,a,d,1,0,idx,run,&S,&C2); orc_cleanup(&S,&R);
            par += C2.pops; if (!trivial) seq += C2.pops;
            if (R.outcome==ORC_RUN_TRIVIAL) trivial=1;
        }
        int isl = p0+seq >= 1024; longg += isl;
        for (int t=0;t<NT;t++) if (p0 >= (uint64_t)TH[t]) { sel[t]++; seqp[t]+=seq; parp[t]+=par; cap[t]+=isl; }
    }
    orc_scratch_free(&S);
    }
    for (int t=0;t<NT;t++) printf("run0 pops >= %d: %llu genomes, waste %llu pops (%.1f%% of 717M executed), captures %llu of %llu long\n",
       TH[t],(unsigned long long)sel[t],(unsigned long long)(parp[t]-seqp[t]),100.0*(parp[t]-seqp[t])/717e6,(unsigned long long)cap[t],(unsigned long long)longg);
    return 0;
}
