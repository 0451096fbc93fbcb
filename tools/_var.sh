cd $GRAFT_REPO_ROOT
for v in p20m16 p20m12 p20m10 p20m8; do EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so python tools/time_paths.py cfg5 | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/p20.jsonl 2>&1; done
