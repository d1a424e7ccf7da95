set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g; nproc; lscpu | grep "Model name"
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
