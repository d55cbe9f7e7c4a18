mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "graph_replay" 2>&1 | tail -1
python scripts/stage_ab.py --workload c2 --opt 5=0 --opt 2=64,4=1 --opt 2=64,4=2 --opt 2=128,4=1 --opt 2=128,4=2 --opt 2=128,4=3 --steps 30
python scripts/stage_ab.py --workload c3 --opt 5=0 --opt 4=3 --opt 4=4 --opt 2=128,4=2 --steps 30
python scripts/stage_ab.py --workload c4 --opt 5=0 --opt 2=64,4=1 --opt 2=64,4=2 --opt 2=128,4=3 --steps 30
