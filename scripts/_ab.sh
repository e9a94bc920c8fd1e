timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_hoisted.py -x -q > gpurun_out/t_prim.log 2>&1
python scripts/prof_step.py --batch 64 > gpurun_out/prof_new.log 2>&1
UH_LIB_PATH=paper_2402_03060_b200/_build/variants/kiold.so python scripts/prof_step.py --batch 64 > gpurun_out/prof_kiold.log 2>&1
