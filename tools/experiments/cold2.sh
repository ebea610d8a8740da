cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
C=paper_2604_06664_b200/foundry
for i in 1 2; do
  s=$(date +%s.%N); FOUNDRY_DEBUG=1 $C load --archive $A --rank 0 --world 8 > /tmp/o.txt 2> /tmp/e.txt; e=$(date +%s.%N)
  echo "wall $(python -c "print(round(($e-$s)*1000))") ms"; grep -E "integrity done|restore done|region|materialize done|group 0:|group 5:|group 11:" /tmp/e.txt
done
s=$(date +%s.%N); python -c "import torch; torch.cuda.init(); torch.zeros(1,device='cuda')"; e=$(date +%s.%N); echo "torch cuda init $(python -c "print(round(($e-$s)*1000))") ms"
cat > /tmp/ci.cu <<'EOC'
#include <cuda_runtime.h>
#include <cstdio>
int main(){ cudaFree(0); return 0; }
EOC
nvcc -o /tmp/ci /tmp/ci.cu && s=$(date +%s.%N); /tmp/ci; e=$(date +%s.%N); echo "bare cuda init $(python -c "print(round(($e-$s)*1000))") ms"
