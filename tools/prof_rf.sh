# one full ncu capture of tree 1's range filter + pair kernel at the bench point (SASS hotspots)
timeout 300 python tools/one_query.py 2 > gpurun_out/plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_range_filter|k_leaf_points" \
    --launch-skip 2 -c 2 -o gpurun_out/prof_rf python tools/one_query.py 2 > gpurun_out/ncu_rf.log 2>&1; echo "ncu exit $?"
