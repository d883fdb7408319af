"""B200-native Canzona distributed optimizer step (drop-in for the reference
``optishard`` planner + Muon optimizer path). See DESIGN.md."""
