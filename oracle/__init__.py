"""Test-infrastructure oracle (CPU restatement of the reference); never product code."""
