bash scripts/gpu_bench.sh
KT_CONFIGS="c2 c3 c4" bash scripts/gpu_kt.sh
bash scripts/gpu_profiles.sh
