cd /root/repo
rm -rf /tmp/cc && mkdir -p /tmp/cc
paper_2604_06664_b200/foundry save --workload micro --out /tmp/cc/cli > /dev/null
python -c "import paper_2604_06664_b200 as f; f.save(f.preset('micro'), '/tmp/cc/lib')"
env | grep -i -E "cubin|tmp|cuda" 
for f in $(cd /tmp/cc/cli && find . -name "*.cubin"); do cmp /tmp/cc/cli/$f /tmp/cc/lib/$f > /dev/null || { echo DIFF $f; /usr/local/cuda/bin/cuobjdump -elf /tmp/cc/cli/$f | grep -E "^\s*\[|sec" | head -0; readelf -S -W /tmp/cc/cli/$f | awk '{print $2, $6}' > /tmp/cc/a; readelf -S -W /tmp/cc/lib/$f | awk '{print $2, $6}' > /tmp/cc/b; diff /tmp/cc/a /tmp/cc/b; strings /tmp/cc/cli/$f | grep -i -E "tmp|ptx|nvlink" | head; break; }; done
