nvidia-smi; nvidia-smi -q | grep -i -E 'clocks|MHz' | head -30; nproc; free -g; lscpu | head -20; python -c "
import torch
p=torch.cuda.get_device_properties(0); print(p); print('L2', p.L2_cache_size if hasattr(p,'L2_cache_size') else None)
"
