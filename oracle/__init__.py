"""Oracle package — TEST INFRASTRUCTURE ONLY (see ew_oracle.py)."""
