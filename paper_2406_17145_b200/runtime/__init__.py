"""Stage executor: runs a configured StageGraph on B200 GPUs through libgpp_b200.so."""
