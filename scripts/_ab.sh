P="python scripts/prof_step.py --batch 64"
UH_LIB_PATH=paper_2402_03060_b200/_build/variants/nonarrow.so $P > gpurun_out/prof_nonarrow.log 2>&1
$P > gpurun_out/prof_narrow.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_hoisted -c 4 -o gpurun_out/narrow $P > gpurun_out/ncu_narrow.log 2>&1
