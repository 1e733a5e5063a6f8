for f in -1 0 8 16 24 32 37; do
 KVX_HASH_FOLD_SMS=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --requests 4 --wave 4 > gpurun_out/h_$f.json 2>/dev/null
 echo "fold_sms=$f $(python profiles/show.py gpurun_out/h_$f.json | tail -1)"
done
