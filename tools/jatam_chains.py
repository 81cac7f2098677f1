"""Fit-mode chain lengths (pops until a genome's first non-DET prefix) vs its longest single run, for the
evolved JaTAM population (_scratch/jatam_pop_g12.npy, tools/jatam_dump_pop.py) and uniform S_{2,8} genomes,
on the oracle restatement.  Development aid."""
import sys, numpy as np, time
sys.path.insert(0,'/root/repo')
from oracle import oracle as O
from paper_2205_15311_b200.genome import SearchSpace
S28=SearchSpace(2,8)
a,bpl,mp,mv,fp=S28.kernel_args()
def run_stats(x, k):
    c=np.zeros(7,np.uint64)
    outs=[np.zeros((1,1),np.uint8),np.zeros(1,np.uint32),np.zeros(1,np.uint8),np.zeros(1,np.uint8),np.zeros(1,np.uint16),np.zeros((1,6),np.uint64)]
    O.classify_batch(np.array([x],np.uint64),a,bpl,mp,mv,fp,19,np.array([k]),k,0,True,*outs,nthreads=1,counts=c)
    return int(c[1]), int(c[0]), int(outs[0][0,0])
for name in ("evolved","uniform"):
    rng=np.random.default_rng(0)
    if name=="evolved":
        pop=np.load('/root/repo/_scratch/jatam_pop_g12.npy'); sample=rng.choice(np.unique(pop),6000,replace=False)
    else:
        sample=rng.integers(0,1<<24,6000,dtype=np.uint64)
    chain=[]; maxrun=[]
    for x in sample:
        prev=0; runs=[]
        for k in range(1,9):
            p,r,cls=run_stats(int(x),k)
            runs.append(p-prev); prev=p
            if r<k: break   # TRIVIAL broke the loop
        # fit-mode chain: runs until the first non-DET prefix (class at k != DET)
        ch=0
        for k in range(1,len(runs)+1):
            ch+=runs[k-1]
            if run_stats(int(x),k)[2]!=0: break
        chain.append(ch); maxrun.append(max(runs))
    chain=np.array(chain); maxrun=np.array(maxrun)
    print(name, "fit chain pops: mean %.1f p99 %.0f p99.9 %.0f max %d | longest single run: p99 %.0f p99.9 %.0f max %d" % (
        chain.mean(), np.percentile(chain,99), np.percentile(chain,99.9), chain.max(),
        np.percentile(maxrun,99), np.percentile(maxrun,99.9), maxrun.max()))
