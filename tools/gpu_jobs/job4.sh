# C5 on one B200: fp32 vs fp64 residues, sink deferral on/off, parity vs pull-Jacobi
timeout 1700 python tools/c5_single.py --jacobi-max-s 1100 --runs 3 --pr-variants '{"sink32": {}, "nosink32": {"sink_defer": false}, "sink64": {"pr_residue_fp64": true}}' > gpurun_out/c5_v2.log 2>&1; echo rc=$? >> gpurun_out/c5_v2.log
