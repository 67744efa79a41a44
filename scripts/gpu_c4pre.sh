# Lane kernels with the first slice's matrix prefetched before griddepcontrol.wait (B) vs without (A),
# each with PDL as shipped for CSR contexts (off) and forced on (DUQUAD_PDL=2); CSR GPU tests on B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py -m gpu -x -q > gpurun_out/pytest_csr.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_csr.log
c4() { timeout 600 python scripts/bench_configs.py --configs 4 --cases 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['us_per_inner_step'],2), round(1e3*d['ms_pass_a'],1), round(1e3*d['ms_pass_b'],1))"; }
cp paper_1504_05708_b200/libduquad.so /tmp/keep.so
for i in 1 2 3; do for v in A B; do cp paper_1504_05708_b200/libduquad_$v.so paper_1504_05708_b200/libduquad.so; echo "$v pdl=off $(c4)  pdl=on $(DUQUAD_PDL=2 c4)"; done; done | tee gpurun_out/c4_pre_ab.txt
cp /tmp/keep.so paper_1504_05708_b200/libduquad.so
