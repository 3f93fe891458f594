set -u
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_retain.py -x -q --timeout 600 -m gpu 2>&1 | tail -1
for rep in 1 2; do
  echo "== new full: $(timeout 300 python tools/prof_k14.py 1024 6144000 2>&1 | tail -1)"
  echo "== new 1req: $(timeout 300 python tools/prof_k14.py 1024 0 2>&1 | tail -1)"
done
