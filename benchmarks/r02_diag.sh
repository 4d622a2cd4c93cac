cd $GRAFT_REPO_ROOT
V="ffn2 shape  K-major  bf16 STORE"
for o in "" "--b-mod 8" "--b-mod 16" "--shared-b"; do echo "== $o"; MOE_GEMM_MC=0 timeout 120 python benchmarks/gemm_sweep.py --only "$V,ffn1 shape  K-major  bf16 STORE" --groups 64 --rows 1024 $o; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_op_gemm_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__d_sectors_fill_sysmem.sum,lts__d_sectors_fill_device.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
for o in "" "--shared-b"; do echo "== ncu $o"; MOE_GEMM_MC=0 timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 3 -c 1 --csv python benchmarks/gemm_sweep.py --only "$V" --groups 64 --rows 1024 --reps 1 $o 2>&1 | grep -v "^==PROF" | tail -20; done
