timeout 600 python -m pytest tests/test_gpu_hoisted.py -x -q > gpurun_out/t_hoist.log 2>&1
P="python scripts/prof_step.py --batch 64 --trace"
$P > gpurun_out/prof_bank.log 2>&1
UH_KEY_BANK=0 $P > gpurun_out/prof_nobank.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
