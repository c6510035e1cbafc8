rm -f gpurun_out/gnn_ab_scores_*.npy
for v in base cur base cur; do
  L=paper_2104_04547_b200/libfusionb200_$v.so; [ $v = cur ] && L=paper_2104_04547_b200/libfusionb200.so
  FS_LIB=$L python tools/gnn_ab.py $v 2>&1 | grep "{" | cut -c1-140
done
