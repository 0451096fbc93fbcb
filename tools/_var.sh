cd $GRAFT_REPO_ROOT
python tools/time_paths.py cfg4 | sed 's/^{/{"v": "st2", /' >> gpurun_out/st.jsonl 2>&1
for v in st3 st4; do EPFEM_GPU_LIB=paper_1805_04155_b200/lib/variants/$v/libepfem_gpu.so python tools/time_paths.py cfg4 | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/st.jsonl 2>&1; done
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg4 or Q1" > gpurun_out/st_pytest.log 2>&1
