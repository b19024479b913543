set -x
nvidia-smi
free -g
nproc
lscpu | head -20
df -h /tmp /root | head
python -c "import torch;print(torch.__version__, torch.cuda.is_available()); p=torch.cuda.get_device_properties(0); print(p); print(p.multi_processor_count, p.L2_cache_size, p.total_memory)"
nvcc --version | tail -2
ulimit -a
