# Config 3 at N=1: layer-wise units of 1 / 4 / 16 layers (8 / 32 / 128 MiB), eager launches
# (programmatic dependent launch on by default) vs CUDA-graph replay, and PDL off
mkdir -p gpurun_out
A="--config 3 --no-match --no-cpu-baseline --steps 5"
for lpc in 1 4 16; do
  echo "lpc=$lpc eager: $(timeout 300 python bench.py $A --layers-per-chunk $lpc 2>/dev/null | python profiles/show.py /dev/stdin 2>/dev/null | head -2 | tr '\n' ' ')"
  echo "lpc=$lpc graph: $(timeout 300 python bench.py $A --layers-per-chunk $lpc --graph 2>/dev/null | python profiles/show.py /dev/stdin 2>/dev/null | head -2 | tr '\n' ' ')"
  echo "lpc=$lpc eager, no PDL: $(KVX_STREAM_PDL=0 timeout 300 python bench.py $A --layers-per-chunk $lpc 2>/dev/null | python profiles/show.py /dev/stdin 2>/dev/null | head -2 | tr '\n' ' ')"
done
echo "c2 default: $(timeout 300 python bench.py --no-match --no-cpu-baseline 2>/dev/null | python profiles/show.py /dev/stdin 2>/dev/null | head -2 | tr '\n' ' ')"
echo "c2 no PDL: $(KVX_STREAM_PDL=0 timeout 300 python bench.py --no-match --no-cpu-baseline 2>/dev/null | python profiles/show.py /dev/stdin 2>/dev/null | head -2 | tr '\n' ' ')"
