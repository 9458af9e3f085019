# session 26: programmatic dependent launch A/B (queries: configs[1], [3], [4]; builds), switch and
# tree tests
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 600 python tools/query_ab.py 2 1000 DETLSH_PDL 0,1 > gpurun_out/pdl26_c2.log 2>&1; echo "pdl c2 exit $?"; tail -4 gpurun_out/pdl26_c2.log
timeout 600 python tools/build_ab.py 2 "3072:0:0,3072:0:1" > gpurun_out/pdlb26_c2.log 2>&1; echo "pdl build c2 exit $?"; tail -2 gpurun_out/pdlb26_c2.log
timeout 600 python tools/query_ab.py 4 10000 DETLSH_PDL 0,1 > gpurun_out/pdl26_c4.log 2>&1; echo "pdl c4 exit $?"; tail -4 gpurun_out/pdl26_c4.log
timeout 900 python tools/query_ab.py 5 2000 DETLSH_PDL 0,1 > gpurun_out/pdl26_c5.log 2>&1; echo "pdl c5 exit $?"; tail -4 gpurun_out/pdl26_c5.log
timeout 900 python tools/build_ab.py 5 "3072:0:0,3072:0:1" > gpurun_out/pdlb26_c5.log 2>&1; echo "pdl build c5 exit $?"; tail -2 gpurun_out/pdlb26_c5.log
unset DATAGEN_CACHE_DIR
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch or split_paths or end_to_end or candidate" > gpurun_out/tests26.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests26.log
