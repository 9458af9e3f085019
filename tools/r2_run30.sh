# session 30: point-code prefetch variants (DETLSH_LP_PF 0 / 1 L2 / 2 L1) and query batch size A/B
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_PF 0,1,2 > gpurun_out/pf30_c5.log 2>&1; echo "pf c5 exit $?"; tail -6 gpurun_out/pf30_c5.log
timeout 1200 python tools/batch_ab.py 5 4000 0,700,1000 > gpurun_out/qb30_c5.log 2>&1; echo "qb c5 exit $?"; tail -6 gpurun_out/qb30_c5.log
timeout 900 python tools/batch_ab.py 4 10000 0,5000,10000 > gpurun_out/qb30_c4.log 2>&1; echo "qb c4 exit $?"; tail -6 gpurun_out/qb30_c4.log
