# The Python example of INTEGRATION.md, runnable (one B200): python scripts/integration_snippet.py
import sys; sys.path.insert(0, '.')
import paper_2602_19873_b200 as sfcnl          # loads libsfcnl_b200.so; raises if absent
ps, box = sfcnl.make_uniform(sfcnl.UniformSpec(n=1 << 16, density=float(1 << 16), target_neighbors=200))
order = sfcnl.sort_by_sfc(ps, box)
tree = sfcnl.build_octree(order)
sps = sfcnl.apply_sfc_order(ps, order)
store = sfcnl.build_neighbor_store(sps, box, tree, sfcnl.BuildParams())
res = sfcnl.reduce(sps, box, store, sfcnl.sph_density_kernel(), sfcnl.PassConfig(1.0, sfcnl.MIXED))
fl = sfcnl.build_full_list(sps, box, 1.0)
r2 = sfcnl.reduce_full(sps, box, fl, sfcnl.sph_density_kernel())
print("ok", sfcnl.memory_footprint(store).bytes_per_particle, fl.memory_bytes() / ps.size(), float(abs(res.outputs[0] - r2.outputs[0]).max() / r2.outputs[0].max()))
