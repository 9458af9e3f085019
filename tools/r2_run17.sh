# session 17: full captures with source (stall sampling per SASS line) of the pair kernel
# (configs[4], default and split 3) and of the build's k_local_finish / k_leaf_layout16 / k_part_scatter
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points" -s 3 -c 1 -o gpurun_out/full17_lp0 python tools/split_ab.py 5 2000 0 > gpurun_out/ncu17_lp0.log 2>&1; echo "ncu lp0 exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points" -s 3 -c 1 -o gpurun_out/full17_lp3 python tools/split_ab.py 5 2000 3 > gpurun_out/ncu17_lp3.log 2>&1; echo "ncu lp3 exit $?"
for k in k_local_finish k_leaf_layout16 k_part_scatter k_project_tc; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o gpurun_out/full17_$k python tools/build_ab.py 5 "1536:256" > gpurun_out/ncu17_$k.log 2>&1; echo "ncu $k exit $?"
done
