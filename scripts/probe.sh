nvidia-smi; nproc; free -g; lscpu | head -20; which gcc nvcc ncu; python -c "import torch;print(torch.cuda.get_device_properties(0))"
