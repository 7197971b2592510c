# north-star scorecard: the 7B step at B = 1..64 (L = 1K), per-kernel GB/s and
# fractions of the measured copy peak and of 8 TB/s; one bench line per batch
mkdir -p gpurun_out/score
for b in 1 8 16 32 64; do
  timeout 600 python bench.py --no-cpu --no-extras --steps 50 --batch $b > gpurun_out/score/b$b.json 2> /dev/null
done
timeout 600 python bench.py --no-cpu --no-extras --steps 30 --model chatglm2-6b --batch 8 --kv-len 32768 > gpurun_out/score/glm.json 2> /dev/null
echo done
