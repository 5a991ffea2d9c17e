# p-way merge staging A/B at p = 2, 4, 8 (c4 sizes): staging batch depth RS_PW_SB
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for pp in 2 4 8; do echo "## p=$pp"; PW_P=$pp bash scripts/gpu_pw_ab.sh paper_1808_10292_b200/librsort.so .exp/librsort_sb12.so .exp/librsort_sb16.so; done
