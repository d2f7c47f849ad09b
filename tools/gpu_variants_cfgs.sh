for c in 1 3 5 4; do CFG=$c bash tools/gpu_variants_cfg.sh; done
