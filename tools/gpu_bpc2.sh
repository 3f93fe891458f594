cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for b in 32 64 128 256 32 64 128; do echo -n "bpc $b: "; FSTG_FWHT_BPC=$b timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1; done
