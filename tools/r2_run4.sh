# session 4: L2-blocking chunk sizes x two-level filter at configs[4]; configs[1] check; new tests
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cp in 0 8388608 4194304 2097152 1048576; do
  for tp in 0 1; do
    DETLSH_CHUNK_PTS=$cp DETLSH_TILE_PAIRS=$tp timeout 900 python tools/qsweep.py 5 3 "c5 cp$cp tp$tp" 2>&1 | grep '^{' >> gpurun_out/qsweep4.jsonl
    tail -1 gpurun_out/qsweep4.jsonl | cut -c1-420
  done
done
for cp in 0 4194304; do
  for tp in 0 1; do
    DETLSH_CHUNK_PTS=$cp DETLSH_TILE_PAIRS=$tp timeout 900 python tools/qsweep.py 4 3 "c3 cp$cp tp$tp" 2>&1 | grep '^{' >> gpurun_out/qsweep4.jsonl
    tail -1 gpurun_out/qsweep4.jsonl | cut -c1-420
  done
done
timeout 1800 python -m pytest tests -m gpu -q -rf -s -k "switches or merge_topk or candidate_set_elementwise_tiny or query_parity_tiny" > gpurun_out/gpu_tests4.log 2>&1; echo "tests exit $?"; tail -4 gpurun_out/gpu_tests4.log
