MCP_LIBRARY=$PWD/paper_1911_03813_b200/_lib/variants/libmomentcp_b200_z_all.so python tools/sweep_small.py > gpurun_out/sweep_small.txt 2>&1
export MCP_LIBRARY=$PWD/paper_1911_03813_b200/_lib/variants/libmomentcp_b200_z_prof.so
python tools/prof_k1z.py > gpurun_out/prof_k1z_c1.txt 2>&1; python tools/prof_k1z.py --shape 500,10,3,1000 > gpurun_out/prof_k1z_t2.txt 2>&1
