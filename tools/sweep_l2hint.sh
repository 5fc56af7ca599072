set -x
mkdir -p gpurun_out
python tools/k1_variant_sweep.py --tag base --save --reps 7
for i in 1 2; do
python tools/k1_variant_sweep.py --tag base --reps 7
for h in 32768 131072 500000; do
KZ_K1_HUBROWS=$h KZ_LIB_PATH=build/variants/l2h1/libkatzb200.so python tools/k1_variant_sweep.py --tag l2h1_$h --reps 7
KZ_K1_HUBROWS=$h KZ_LIB_PATH=build/variants/l2h2/libkatzb200.so python tools/k1_variant_sweep.py --tag l2h2_$h --reps 7
done
done
