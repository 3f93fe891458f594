# A/B of k = 14 retain variants (tools/variants/lib_*.so) at full request load and one request per basis
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2105_05879_b200/libfst_b200.so /tmp/lib_keep.so
for v in ${VARIANTS:-base}; do
  cp tools/variants/lib_$v.so paper_2105_05879_b200/libfst_b200.so
  for c in ${CLS:-4 8}; do
    for req in 6144000 0; do
      echo "$v CL=$c $(FSTG_RETAIN_CLUSTER=$c timeout 300 python tools/prof_k14.py 1024 $req 2>&1 | tail -1)"
    done
  done
done
cp /tmp/lib_keep.so paper_2105_05879_b200/libfst_b200.so
