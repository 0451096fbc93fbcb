cd $GRAFT_REPO_ROOT
for pr in "0 0" "2 3" "3 2" "2 2" "1 4" "3 3"; do
  set -- $pr
  EPFEM_PERSIST_FUSED=$1 EPFEM_PERSIST_ROWS=$2 python tools/exp_concurrent.py --config cfg4 --reps 10 --prio 2>&1 | grep prio | sed "s/^/F=$1 R=$2 /" >> gpurun_out/corun.txt
done
