import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']
print('step %.3f | lidar: sort %.3f counts %.3f tsort %.3f fwd %.3f bwd %.3f pbwd %.3f | camera: sort %.3f counts %.3f tsort %.3f fwd %.3f bwd %.3f pbwd %.3f | e2e %.2f' % (d['ms_per_step'], *[s['lidar'][k] for k in ('depth_sort_scan','tile_counts','tile_sort','raster_fwd','raster_bwd','project_bwd')], *[s['camera'][k] for k in ('depth_sort_scan','tile_counts','tile_sort','raster_fwd','raster_bwd','project_bwd')], d['e2e']['ms_per_step']))
