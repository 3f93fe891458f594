cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 0 1 0 1; do echo -n "pretouch $t: "; FSTG_PRETOUCH=$t timeout 300 python tools/prof_preprocess.py 4096 2>&1 | tail -1; done
