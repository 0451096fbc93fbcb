cd $GRAFT_REPO_ROOT
python tools/time_paths.py cfg4 | sed 's/^{/{"v": "default", /' >> gpurun_out/a20.jsonl 2>&1
for kb in 40 24 32; do EPFEM_ROW_KB=$kb EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/a20/libepfem_gpu.so python tools/time_paths.py cfg5 | sed "s/^{/{\"v\": \"a20-$kb\", /" >> gpurun_out/a20.jsonl 2>&1; done
EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/a20/libepfem_gpu.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg5 or Q2-3" > gpurun_out/a20_pytest.log 2>&1
