for s in "4096 4096 64 8192" "256 256 32 256" "1024 1024 128 512" "1024 1024 256 256" "1024 1024 31 512"; do timeout 300 python scripts/gemm_variants.py $s --quick 2>&1 | tail -2; done
