"""specexit.engine (src/specexit/engine.py) on the B200 library."""
from paper_2504_08850_b200.engine import (AlwaysExitPolicy, EngineConfig, ExitEngine,  # noqa: F401
                                          ExitRecord, NeverExitPolicy, OraclePolicy,
                                          PredictorPolicy, generate, greedy_generate,
                                          oracle_exit_layer, read_trace, verify_exit,
                                          write_trace)
