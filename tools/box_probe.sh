set -x
free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import sys; sys.path.insert(0,'baseline/_ref'); import os; os.environ['NUMBA_CACHE_DIR']='/tmp/nb'; import blowchoc, numba; print(blowchoc.__file__, numba.__version__)"
python -c "import torch; print(torch.cuda.mem_get_info())"
