import re, sys
# needs a library built with SVN_NVCC_DEFINES=SVN_KERNEL_PROF (clock reads are compiled out otherwise)
names=['mma_wait_a','mma_wait_full','mma_wait_ax','mma_total','epi_wait_d','epi_work','epi_arrive','epi_out','epi_ax','prod_wait_empty','-','mma_wait_a_l0','mma_wait_a_l1','mma_wait_full_l0']
line=[l for l in open(sys.argv[1]) if 'svn prof' in l][-1]
v=[int(x) for x in line.split(']')[1].split()]
n=int(sys.argv[2]) if len(sys.argv)>2 else 74
for nm,x in zip(names,v):
    if nm=='-': continue
    print(f"{nm:16s} {x/n/1e6:8.1f} Mcyc  {x/v[3]*100:5.1f}%")
