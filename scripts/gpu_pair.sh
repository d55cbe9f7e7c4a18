# cta_group::2 GEMM bring-up: small bitwise variant test first (hang-guarded), then timings
timeout 300 python -m pytest tests -m gpu -x -q -k "variants_bitwise" 2>&1 | tail -3
timeout 120 python scripts/gemm_variants.py 1024 1024 31 512
timeout 300 python scripts/gemm_variants.py 4096 4096 64 8192
TPROD_SEG256=1 timeout 300 python scripts/gemm_variants.py 4096 4096 64 8192
