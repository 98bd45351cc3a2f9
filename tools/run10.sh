bash tools/gpu_variants.sh paper_1706_07772_b200/libreax_minb2.so
bash tools/gpu_sweep.sh paper_1706_07772_b200/libreax_minb2.so REAX_NBR_SPLIT "1 2 3 4"
