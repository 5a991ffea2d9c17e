# p-way merge staging A/B (previous commit vs working tree) at p = 2, 4, 8: c4 (u32) and c5 (pairs)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gsd.py tests/test_gpu_net.py -q -x -p no:cacheprovider 2>&1 | tail -1
for pp in 2 4 8; do echo "## u32 p=$pp"; PW_P=$pp bash scripts/gpu_pw_ab.sh .exp/librsort_pwprev.so paper_1808_10292_b200/librsort.so; done
for pp in 2 4 8; do echo "## pairs p=$pp"; PW_LG=30 PW_KIND=pairs PW_P=$pp bash scripts/gpu_pw_ab.sh .exp/librsort_pwprev.so paper_1808_10292_b200/librsort.so; done
