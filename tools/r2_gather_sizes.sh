cd "${GRAFT_REPO_ROOT}"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_probe tools/gather_probe.cu 2>&1 | tail -2
for mib in 256 512 1024 2048 4096 8192 16384 32768; do /tmp/gather_probe g $mib 28 1 0; done
