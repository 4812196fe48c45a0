# A/B of the checked EXACT division path (libltk_chk.so) against the guarded one
# (libltk_base.so): burst line, tau 0.8, FAST, 1000-step sustained, configs[1] sweep.
cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out; rm -f gpurun_out/chk_ab.txt
N=paper_1405_6162_b200/_native
for v in base chk base chk; do
  cp $N/libltk_$v.so $N/libltk.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --sustained-steps 1000 > gpurun_out/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); s=d['variants']['sustained']; r=d['roofline']; c=d['collision_128']
print('$v', 'burst %.4f ms cs %.4f' % (d['ms_per_step'], r['kernel_ms_per_step']), 'tau08 %.4f fast %.4f' % (d['variants']['exact_tau0.8']['ms_per_step'], d['variants']['fast']['ms_per_step']), 'sustained %.4f ms (sm %s)' % (s['ms_per_step'], s['clocks']['sm_mhz']), 'c128', ' '.join('%d:%.4f' % (x['vvl'], x['ms_per_launch']) for x in c['vvl_sweep']))" >> gpurun_out/chk_ab.txt
done
cp $N/libltk_chk.so $N/libltk.so
cat gpurun_out/chk_ab.txt
