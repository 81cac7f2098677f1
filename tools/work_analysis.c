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

int main(int argc, char **argv) {
    /* usage: work_analysis s28|s32|A,B [start count [nblocks [strict]]] */
    int a = 2, bpl = 3, d = 19, kmax = 8, strict = 1;
    uint64_t start = 0, count = 1ULL << 24;
    int64_t mpos[4] = {32, 33, 34, 35};
    uint8_t mval[4] = {0, 0, 0, 0};
    int64_t m = 0;
    int s32 = argc > 1 && strcmp(argv[1], "s32") == 0;
    if (s32) { a = 3; kmax = 7; m = 4; count = 1ULL << 22; start = 0; }
    if (argc > 1 && strchr(argv[1], ',')) {  /* plain space S_{A,B} */
        int b = 8;
        sscanf(argv[1], "%d,%d", &a, &b);
        bpl = 0;
        while ((1 << bpl) < b) bpl++;
        count = 1ULL << (a * 4 * bpl);
    }
    if (argc > 2) start = strtoull(argv[2], 0, 0);
    if (argc > 3) count = strtoull(argv[3], 0, 0);
    /* optional stratified sample: nblocks evenly spaced blocks of count / nblocks indices */
    const int Lbits = a * 4 * bpl - (int)m;
    uint64_t nblocks = argc > 4 ? strtoull(argv[4], 0, 0) : 1, card = 1ULL << Lbits;
    if (argc > 5) strict = atoi(argv[5]);
    const int L = a * 4 * bpl;
    int64_t free_pos[64];
    int64_t nfree = 0;
    for (int p = L - 1; p >= 0; p--) {
        int fixed = 0;
        for (int j = 0; j < m; j++) fixed |= mpos[j] == p;
        if (!fixed) free_pos[nfree++] = p;
    }
    uint64_t tot_pops = 0, tot_runs = 0, om_g = 0, om_pops = 0, om_runs = 0;
    uint64_t au_pops = 0, au_fu_pops = 0, au_fu_tf_pops = 0, au_tr_pops = 0, au_fu_g = 0, au_fu_tf_g = 0;
    uint64_t unb_g = 0, tf_g = 0, tf2_g = 0, au_fu_tf2_pops = 0, au_fu_tf2_g = 0, viol2 = 0, au_runs = 0, au_fu_runs = 0, au_fu_tf_runs = 0;
    uint64_t lp_g = 0, lp_exec = 0, lp_all = 0, lp_long = 0, hist_exec[8] = {0}, fz_not_tf = 0, fz_not_tf_runs = 0, b0_checked_not_tf = 0, ex_cls[4] = {0, 0, 0, 0}, ex_runs_cls[4] = {0, 0, 0, 0}, ops_ref = 0, ops_exec = 0, runs_exec = 0, pops_exec = 0, fz_g = 0, fz_pops_saved = 0, fz_runs_saved = 0, fz_viol = 0, fz_det = 0, run0_unb_pops = 0, cls[4] = {0, 0, 0, 0}, cls_pops[4] = {0, 0, 0, 0}, det_tf2_pops = 0, det_tf2_g = 0;
#pragma omp parallel reduction(+ : tot_pops, tot_runs, om_g, om_pops, om_runs, au_pops, au_fu_pops, au_fu_tf_pops, \
                               au_tr_pops, au_fu_g, au_fu_tf_g, unb_g, tf_g, au_runs, au_fu_runs, au_fu_tf_runs, \
                               lp_g, lp_exec, lp_all, lp_long, hist_exec[:8], fz_not_tf, fz_not_tf_runs, b0_checked_not_tf, ex_cls[:4], ex_runs_cls[:4], ops_ref, ops_exec, runs_exec, pops_exec, fz_g, fz_pops_saved, fz_runs_saved, fz_viol, fz_det, run0_unb_pops, cls[:4], cls_pops[:4], det_tf2_pops, det_tf2_g, tf2_g, au_fu_tf2_pops, au_fu_tf2_g, viol2)
    {
        orc_scratch S;
        orc_scratch_alloc(&S, d);
        uint8_t bits[128], E[16 * 16];
#pragma omp for schedule(dynamic, 4096)
        for (int64_t i = 0; i < (int64_t)count; i++) {
            const uint64_t per = count / nblocks;
            uint64_t idx = nblocks > 1 ? (uint64_t)i / per * (card / nblocks) + (uint64_t)i % per : start + (uint64_t)i;
            orc_decode_edges(idx, a, bpl, mpos, mval, m, free_pos, nfree, bits, E);
            uint64_t pops[16] = {0};
            int outc[16], nr = 0, first_unb = -1, triv = -1, fz = 0;
            uint32_t hs[16];
            orc_counts RC[16];
            for (int run = 0; run < kmax; run++) {
                orc_counts C;
                memset(&C, 0, sizeof C);
                C.runs = 1;
                orc_run R = orc_assemble(E, a, d, strict, 0, idx, run, &S, &C);
                hs[run] = 0;
                if (R.outcome == ORC_RUN_BOUNDED) {
                    int w_, h_, nc_;
                    hs[run] = orc_hash_region(&S, d, &R, &w_, &h_, &nc_);
                    C.bounded_runs = 1;
                    C.hashed_cells = (uint64_t)nc_;
                    if (run == 0) fz = forced(E, a, d, &S, R.n_placed);
                }
                orc_cleanup(&S, &R);
                pops[run] = C.pops;
                RC[run] = C;
                outc[run] = R.outcome;
                nr++;
                if (R.outcome == ORC_RUN_TRIVIAL) { triv = run; break; }
                if (R.outcome == ORC_RUN_UNBOUND && first_unb < 0) first_unb = run;
            }
            uint64_t gp = 0;
            for (int r = 0; r < nr; r++) gp += pops[r];
            tot_pops += gp;
            tot_runs += nr;
            int c = triv >= 0 ? 1 : first_unb >= 0 ? 3 : 0;
            cls[c]++;
            if (fz) {
                int same = triv < 0 && first_unb < 0 && nr == kmax;
                for (int r = 1; r < nr; r++) same = same && hs[r] == hs[0];
                fz_g++; fz_det += same; fz_viol += !same;
                for (int r = 1; r < nr; r++) fz_pops_saved += pops[r];
                fz_runs_saved += nr - 1;
            }
            cls_pops[c] += gp;
            {   /* event-weighted int32 ops (SURVEY 8d weights): every run of the reference vs the runs
                   the kernel executes (1-mers: none; stop after a forced run 0 or at the first UNBOUND
                   run of a trivial-free genome) */
                const int om = one_mer(E, a), tf2e = trivial_free_v2(E, a, strict);
                int ne = 0;
                if (!om) {
                    for (ne = 0; ne < nr; ne++) {
                        if (ne == 0 && fz) { ne = 1; break; }
                        if (outc[ne] == ORC_RUN_UNBOUND && tf2e) { ne++; break; }
                    }
                }
                for (int r = 0; r < nr; r++) {
                    uint64_t o = 24 * (RC[r].draws + RC[r].pops + RC[r].placements) + 10 * RC[r].hashed_cells +
                                 16 * RC[r].bounded_runs + 16 * RC[r].runs;
                    ops_ref += o;
                    if (r < ne) { ops_exec += o; runs_exec++; pops_exec += RC[r].pops; ex_cls[c] += RC[r].pops; ex_runs_cls[c]++; }
                }
                ops_ref += 64;
                {   /* executed pops per genome, log2 buckets from 64 */
                    uint64_t ep = 0;
                    for (int r = 0; r < ne; r++) ep += RC[r].pops;
                    int b = 0;
                    while (b < 7 && ep >= (64ULL << b)) b++;
                    hist_exec[b]++;
                    int line = 0;
                    for (int t = 0; t < a; t++)
                        line |= orc_bonds(E[t * 16 + 0], E[t * 16 + 2]) || orc_bonds(E[t * 16 + 1], E[t * 16 + 3]);
                    if (line && !tf2e && !om) {
                        lp_g++; lp_exec += ep; lp_long += ep >= 1024;
                        /* every run of the genome executed to its end (run-parallel: no TRIVIAL exit) */
                        for (int r = 0; r < nr; r++) lp_all += RC[r].pops;
                        if (nr < kmax) {  /* the runs after the TRIVIAL one: estimate by the mean run */
                            uint64_t m = 0;
                            for (int r = 0; r < nr; r++) m += RC[r].pops;
                            lp_all += (m / nr) * (uint64_t)(kmax - nr);
                        }
                    }
                }
                ops_exec += om ? 16 : 64;
            }
            if (one_mer(E, a)) { om_g++; om_pops += gp; om_runs += nr; }
            int tf = trivial_free_scalar(E, a, strict);
            tf_g += tf;
            int tf2 = trivial_free_v2(E, a, strict);
            tf2_g += tf2;
            if (tf2 && c == 0) { det_tf2_g++; det_tf2_pops += gp; }
            if (fz && !tf2 && !one_mer(E, a)) { fz_not_tf++; fz_not_tf_runs += nr - 1; }
            if (outc[0] == ORC_RUN_BOUNDED && !tf2) b0_checked_not_tf++;
            if (tf2 && triv >= 0) viol2++;  /* unsound proof: a TRIVIAL it said impossible */
            if (first_unb == 0) run0_unb_pops += gp - pops[0];
            if (first_unb >= 0) {
                uint64_t after = 0;
                for (int r = first_unb + 1; r < nr; r++) after += pops[r];
                au_pops += after;
                au_runs += nr - first_unb - 1;
                if (triv < 0) {
                    unb_g++;
                    au_fu_pops += after; au_fu_g++; au_fu_runs += nr - first_unb - 1;
                    if (tf2) { au_fu_tf2_pops += after; au_fu_tf2_g++; }
                    if (tf) { au_fu_tf_pops += after; au_fu_tf_g++; au_fu_tf_runs += nr - first_unb - 1; }
                } else {
                    au_tr_pops += after;
                }
            }
            (void)outc;
        }
        orc_scratch_free(&S);
    }
    printf("{\"space\": \"%s\", \"start\": %llu, \"count\": %llu, \"kmax\": %d,\n", s32 ? "s32" : "s28",
           (unsigned long long)start, (unsigned long long)count, kmax);
    printf(" \"pops\": %llu, \"runs\": %llu, \"classes_at_kmax\": [%llu, %llu, 0, %llu],\n",
           (unsigned long long)tot_pops, (unsigned long long)tot_runs, (unsigned long long)cls[0],
           (unsigned long long)cls[1], (unsigned long long)cls[3]);
    printf(" \"one_mer\": {\"genomes\": %llu, \"runs\": %llu, \"pops\": %llu},\n", (unsigned long long)om_g,
           (unsigned long long)om_runs, (unsigned long long)om_pops);
    printf(" \"trivial_free_genomes\": %llu, \"trivial_free_v2_genomes\": %llu, \"v2_violations\": %llu,\n",
           (unsigned long long)tf_g, (unsigned long long)tf2_g, (unsigned long long)viol2);
    printf(" \"after_first_unbound\": {\"pops\": %llu, \"runs\": %llu,\n", (unsigned long long)au_pops,
           (unsigned long long)au_runs);
    printf("   \"final_unbound\": {\"genomes\": %llu, \"runs\": %llu, \"pops\": %llu},\n", (unsigned long long)au_fu_g,
           (unsigned long long)au_fu_runs, (unsigned long long)au_fu_pops);
    printf("   \"final_unbound_tfree\": {\"genomes\": %llu, \"runs\": %llu, \"pops\": %llu},\n",
           (unsigned long long)au_fu_tf_g, (unsigned long long)au_fu_tf_runs, (unsigned long long)au_fu_tf_pops);
    printf("   \"final_unbound_tfree_v2\": {\"genomes\": %llu, \"pops\": %llu},\n",
           (unsigned long long)au_fu_tf2_g, (unsigned long long)au_fu_tf2_pops);
    printf("   \"later_trivial_pops\": %llu},\n", (unsigned long long)au_tr_pops);
    printf(" \"pops_by_class\": [%llu, %llu, %llu, %llu], \"det_tfree_v2\": {\"genomes\": %llu, \"pops\": %llu},\n",
           (unsigned long long)cls_pops[0], (unsigned long long)cls_pops[1], (unsigned long long)cls_pops[2],
           (unsigned long long)cls_pops[3], (unsigned long long)det_tf2_g, (unsigned long long)det_tf2_pops);
    printf(" \"forced\": {\"genomes\": %llu, \"all_runs_equal\": %llu, \"violations\": %llu, \"pops_saved\": %llu, \"runs_saved\": %llu},\n",
           (unsigned long long)fz_g, (unsigned long long)fz_det, (unsigned long long)fz_viol,
           (unsigned long long)fz_pops_saved, (unsigned long long)fz_runs_saved);
    printf(" \"ops_per_genome_reference\": %.2f, \"ops_per_genome_executed\": %.2f, \"runs_executed\": %llu, \"pops_executed\": %llu,\n",
           (double)ops_ref / (double)count, (double)ops_exec / (double)count, (unsigned long long)runs_exec,
           (unsigned long long)pops_exec);
    printf(" \"forced_not_tfree\": {\"genomes\": %llu, \"runs_saved\": %llu}, \"run0_bounded_not_tfree\": %llu,\n",
           (unsigned long long)fz_not_tf, (unsigned long long)fz_not_tf_runs, (unsigned long long)b0_checked_not_tf);
    printf(" \"executed_pops_per_genome_log2_buckets_from_64\": [%llu, %llu, %llu, %llu, %llu, %llu, %llu, %llu],\n",
           (unsigned long long)hist_exec[0], (unsigned long long)hist_exec[1], (unsigned long long)hist_exec[2],
           (unsigned long long)hist_exec[3], (unsigned long long)hist_exec[4], (unsigned long long)hist_exec[5],
           (unsigned long long)hist_exec[6], (unsigned long long)hist_exec[7]);
    printf(" \"line_prone_not_tfree\": {\"genomes\": %llu, \"executed_pops\": %llu, \"pops_if_all_runs\": %llu, \"genomes_ge_1024_pops\": %llu},\n",
           (unsigned long long)lp_g, (unsigned long long)lp_exec, (unsigned long long)lp_all, (unsigned long long)lp_long);
    printf(" \"executed_pops_by_class\": [%llu, %llu, %llu, %llu], \"executed_runs_by_class\": [%llu, %llu, %llu, %llu],\n",
           (unsigned long long)ex_cls[0], (unsigned long long)ex_cls[1], (unsigned long long)ex_cls[2], (unsigned long long)ex_cls[3],
           (unsigned long long)ex_runs_cls[0], (unsigned long long)ex_runs_cls[1], (unsigned long long)ex_runs_cls[2], (unsigned long long)ex_runs_cls[3]);
    printf(" \"run0_unbound_later_pops\": %llu}\n", (unsigned long long)run0_unb_pops);
    return 0;
}
