"""fp64 CPU oracle of the reference Muon path (test infrastructure; see oracle.py)."""
