for g in 16 74 148 296 592 1184; do echo "grid $g"; GPA_FUSED_GRID=$g timeout 300 python tools/analyze_time.py product 2,3 fused; done
timeout 300 python tools/analyze_time.py product 2,3 graph
