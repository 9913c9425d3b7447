set -u
timeout 300 python -m pytest tests/test_gpu_track.py -q -k "cell_edges or equals_general" -p no:cacheprovider 2>&1 | tail -2
sed -i 's/if (fr32 > margin \&\& fr32 < 1.0f - margin \&\& f32 >= 0.0f \&\& f32 <= a.fmax)/if (fr32 >= margin \&\& fr32 < 1.0f - margin \&\& f32 >= 0.0f \&\& f32 <= a.fmax)/' paper_1310_5541_b200/csrc/pcs_fused.cuh
grep -c "fr32 >= margin" paper_1310_5541_b200/csrc/pcs_fused.cuh
timeout 600 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_track.py -q -k "cell_edges" -p no:cacheprovider 2>&1 | tail -3
