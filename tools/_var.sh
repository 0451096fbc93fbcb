cd $GRAFT_REPO_ROOT
for v in gpf gearly; do EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so python tools/time_paths.py cfg4 cfg5 | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/geo.jsonl 2>&1; done
