# r02x2: conv_check A/B (one thread per output vs stream-split), warm and flushed L2
O=gpurun_out/r02x2; mkdir -p $O
for fl in "" "--flush"; do
for mt in "3 64" "8 64" "3 1000"; do set -- $mt
timeout 600 python scripts/r02/ab.py --variant one:-DNE_CONV_CHECK_ONE --variant split: --case c2_conv_check --M $1 --T $2 --reps 100 $fl >> $O/ab.txt 2>&1
echo "flush=$fl" >> $O/ab.txt
done; done
grep " us$\|failed\|flush" $O/ab.txt
