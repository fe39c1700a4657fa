nvidia-smi; lscpu | head -20; nproc; free -g; python -c "import numpy; numpy.show_runtime()" 2>&1 | grep -A3 found | head; ./tools/peaks
