# ncu --set full of one launch of every step-path kernel at full size, summarised on the box (reports are large)
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:mgs_kernel -s 3 -c 1 -o gpurun_out/kr_mgs python tools/prof_mgs.py > /dev/null 2>&1
$N -k regex:combine_small_kernel -s 3 -c 1 -o gpurun_out/kr_combine python tools/prof_combine.py > /dev/null 2>&1
K=2 L=7 NB=4 $N -k regex:cheb_rows_kernel -s 2 -c 1 -o gpurun_out/kr_chebrows python tools/prof_vcycle.py > /dev/null 2>&1
K=2 L=7 NB=4 $N -k regex:transfer_cols_kernel -s 2 -c 1 -o gpurun_out/kr_tcols python tools/prof_vcycle.py > /dev/null 2>&1
K=2 L=7 NB=4 $N -k regex:transfer_rows_kernel -s 2 -c 1 -o gpurun_out/kr_trows python tools/prof_vcycle.py > /dev/null 2>&1
K=2 L=7 NB=4 $N -k regex:prolong3d -s 2 -c 1 -o gpurun_out/kr_prolong3d python tools/prof_vcycle.py > /dev/null 2>&1
K=2 L=7 NB=4 $N --kernel-name-base demangled -k regex:"stage_apply_kernel<.int.2, .int.4, .bool.1, .int.0>" -s 2 -c 1 -o gpurun_out/kr_k1blk python tools/prof_vcycle.py > /dev/null 2>&1
K=4 L=6 Q=3 $N -k regex:stage_apply -s 2 -c 1 -o gpurun_out/kr_k1c2 python tools/prof_apply.py > /dev/null 2>&1
$N -k regex:coarse_vcycle -s 2 -c 1 -o gpurun_out/kr_coarse python tools/step_profile.py C5 > /dev/null 2>&1
$N -k regex:mgs_column_coop -s 4 -c 1 -o gpurun_out/kr_mgscoop python tools/step_profile.py C3 > /dev/null 2>&1
ls gpurun_out/kr_*
python tools/ncu_kernel_table.py gpurun_out/kernels_ncu.txt \
  "K1 coupled STORE, C2 (k=4, Q=3, 64^3)::gpurun_out/kr_k1c2.ncu-rep" \
  "K1 block STORE, C4 finest level (k=2, 4 blocks, 128^3)::gpurun_out/kr_k1blk.ncu-rep" \
  "cheb_rows (Chebyshev update), C4 finest level::gpurun_out/kr_chebrows.ncu-rep" \
  "prolong3d (fused 3D P + accumulate), C4 finest level::gpurun_out/kr_prolong3d.ncu-rep" \
  "transfer_rows (z sweep of the restriction), C4::gpurun_out/kr_trows.ncu-rep" \
  "transfer_cols (y / x sweep of the restriction), C4::gpurun_out/kr_tcols.ncu-rep" \
  "mgs (w -= h v; <v,w>), 67.9M doubles::gpurun_out/kr_mgs.ncu-rep" \
  "combine_small (stage transform, Q=4, 17M DoFs per stage)::gpurun_out/kr_combine.ncu-rep" \
  "coarse_vcycle (levels 0..2 of C5's k=3 hierarchy, one CTA)::gpurun_out/kr_coarse.ncu-rep" \
  "mgs_column_coop (one MGS column of C3, 824K doubles)::gpurun_out/kr_mgscoop.ncu-rep"
rm -f gpurun_out/kr_*.ncu-rep
