nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/g1_smi.txt; nproc >> gpurun_out/g1_smi.txt; free -g >> gpurun_out/g1_smi.txt; lscpu | head -20 >> gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
