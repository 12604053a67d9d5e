"""specexit.scheduler (src/specexit/scheduler.py) on the B200 library."""
from paper_2504_08850_b200.scheduler import (OfflineProfile, OnlineState,  # noqa: F401
                                             ScheduleConfig, active_layers, load_profile,
                                             online_hot_layers, profile_offline,
                                             recompute_counts, save_profile, update_online,
                                             weight_fingerprint)
