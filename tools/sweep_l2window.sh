# K1 launched chunk by chunk with an L2 persisting access-policy window over the
# chunk's hub rows (cudaStreamAttributeAccessPolicyWindow; set-aside size, window
# rows and hit ratio swept) against the shipped single launch.
python tools/k1_variant_sweep.py --tag base --save --reps 7 | tail -1
KZ_K1_L2WINDOW_ROWS=1 KZ_K1_L2WINDOW_MB=0 python tools/k1_variant_sweep.py --tag perchunk_nowindow --reps 7 | tail -1
for mb in 32 64 96; do
for rows in 32768 131072 262144; do
for hit in 1.0 0.5; do
KZ_K1_L2WINDOW_ROWS=$rows KZ_K1_L2WINDOW_MB=$mb KZ_K1_L2WINDOW_HIT=$hit python tools/k1_variant_sweep.py --tag win_${rows}_${mb}mb_hit$hit --reps 7 | tail -1
done; done; done
python tools/k1_variant_sweep.py --tag base --reps 7 | tail -1
