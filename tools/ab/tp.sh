timeout 300 ./tools/microbench/tma_pattern
