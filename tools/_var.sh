cd $GRAFT_REPO_ROOT
for v in ub2 ub4 ub8; do EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so python tools/time_paths.py cfg4 cfg3 cfg5 | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/ub.jsonl 2>&1; done
