# Build the library of a git revision (default HEAD) as _lib/libzstripe_b200_old.so for A/B runs
# (tools/attn_ab.py, tools/gemm_ab.py).  Runs here (nvcc cross-compiles); the .so travels with gpurun.
set -e
REV=${1:-HEAD}
rm -rf /tmp/oldtree && mkdir -p /tmp/oldtree
git archive "$REV" paper_2605_17633_b200 include | tar -x -C /tmp/oldtree
(cd /tmp/oldtree && python -m paper_2605_17633_b200.build --force > /dev/null 2>&1)
cp /tmp/oldtree/paper_2605_17633_b200/_lib/libzstripe_b200.so paper_2605_17633_b200/_lib/libzstripe_b200_old.so
echo "built $REV -> paper_2605_17633_b200/_lib/libzstripe_b200_old.so"
