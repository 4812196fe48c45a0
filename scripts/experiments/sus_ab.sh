# A/B of libltk.so vs libltk_ng.so (built with -DLTK_NOGUARD: div_rcp without its inf/NaN
# pass-through; the macro was removed again after this measurement).
cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out; rm -f gpurun_out/sus_ab.txt
cp paper_1405_6162_b200/_native/libltk.so /tmp/libltk_guard.so
for v in guard ng guard ng; do
  if [ $v = ng ]; then cp paper_1405_6162_b200/_native/libltk_ng.so paper_1405_6162_b200/_native/libltk.so; else cp /tmp/libltk_guard.so paper_1405_6162_b200/_native/libltk.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-config1 --no-e2e --sustained-steps 1000 > gpurun_out/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); s=d['variants']['sustained']; r=d['roofline']
print('$v', 'burst %.4f ms cs %.4f' % (d['ms_per_step'], r['kernel_ms_per_step']), 'sustained %.4f ms %.0f MLUPS sm %s W %s' % (s['ms_per_step'], s['value'], s['clocks']['sm_mhz'], s['clocks']['power_w_max']), 'tau08 %.4f fast %.4f' % (d['variants']['exact_tau0.8']['ms_per_step'], d['variants']['fast']['ms_per_step']))" >> gpurun_out/sus_ab.txt
done
cp /tmp/libltk_guard.so paper_1405_6162_b200/_native/libltk.so
cat gpurun_out/sus_ab.txt
